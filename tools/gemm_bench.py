"""Micro-benchmark of the batched tcgen05 GEMM (3xTF32, or 3xF16 with --prec 1) on the path's shapes
(configs[3]).

    python tools/gemm_bench.py [--reps 20] [--prec 0|1]
Prints one line per shape: ms per launch, useful TFLOP/s, tf32-pipe TFLOP/s, rel. error on batch 0.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402

SHAPES = {  # name: (M, N, K, batch, a_mn, b_mn, d_trans)
    "power": (1024, 256, 1024, 64, False, False, True),
    "gram": (256, 256, 1024, 64, False, False, False),
    "qform": (1024, 256, 256, 64, True, False, True),
    "apply_z": (256, 1000, 1024, 64, False, True, False),
    "apply_f": (1024, 1000, 256, 64, True, True, False),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shapes", nargs="*", default=list(SHAPES))
    ap.add_argument("--prec", type=int, default=0)
    ap.add_argument("--pre", action="store_true", help="3xF16 with both operands pre-split (K-major shapes only)")
    ap.add_argument("--batch", type=int, default=0, help="override the batch (8 = one stream part of configs[3])")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    for name in a.shapes:
        M, N, K, B, a_mn, b_mn, d_trans = SHAPES[name]
        B = a.batch or B
        A = torch.randn(B, *((K, M) if a_mn else (M, K)), device="cuda", generator=g)
        Bm = torch.randn(B, *((K, N) if b_mn else (N, K)), device="cuda", generator=g)
        D = torch.empty(B, *((N, M) if d_trans else (M, N)), device="cuda")

        if a.pre:
            if a_mn or b_mn:
                continue
            A16 = hg.f16_split(A, 11)
            B16 = hg.f16_split(Bm, 11)

            def run():
                hg.gemm_f16pre(A16, B16, M=M, N=N, K=K, batch=B, lda=A.shape[2],
                               sa=A[0].numel(), a_exp=11, ldb=Bm.shape[2], sb=Bm[0].numel(), b_exp=11, D=D,
                               d_trans=d_trans, ldd=D.shape[2], sd=D[0].numel())
        else:
            def run():
                hg.gemm(A, Bm, M=M, N=N, K=K, batch=B, a_mn=a_mn, lda=A.shape[2], sa=A[0].numel(), b_mn=b_mn,
                        ldb=Bm.shape[2], sb=Bm[0].numel(), D=D, d_trans=d_trans, ldd=D.shape[2], sd=D[0].numel(),
                        prec=a.prec, a_exp=11, b_exp=11)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        A0 = A[0].double().T if a_mn else A[0].double()
        B0 = Bm[0].double() if b_mn else Bm[0].double().T
        ref = A0 @ B0
        got = D[0].double().T if d_trans else D[0].double()
        err = float((got - ref).norm() / ref.norm())
        useful = 2.0 * M * N * K * B / (ms / 1e3) / 1e12
        print(json.dumps({"shape": name, "MNK_batch": [M, N, K, B], "ms": ms, "useful_tflops": useful,
                          "pipe_tflops": 3 * useful, "rel_err": err,
                          "prec": ["3xtf32", "3xf16"][a.prec] + ("-presplit" if a.pre else ""),
                          "split": os.environ.get("HG_TF32_SPLIT", "trunc")}), flush=True)


if __name__ == "__main__":
    main()
