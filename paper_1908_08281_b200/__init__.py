"""B200-native block randomized SVD hot path of arXiv:1908.08281.

The product is the C-ABI library libhgrsvd.so (include/hg.h, CUDA sm_100a);
`hg` is its thin Python binding.  Importing `paper_1908_08281_b200.hg` fails
loudly if the library has not been built (no CPU fallback exists).
"""
__all__ = ["hg", "build"]
