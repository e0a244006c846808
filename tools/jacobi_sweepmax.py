"""Per-sweep maximum Jacobi rotation measure |a_pq| / sqrt(a_pp a_qq) of every block of one
configs[3] solve (debug instrumentation in jacobi_blk.cu, compiled only with -DHG_JB_SWEEPMAX),
printed per block slot (max over the stream parts).

    HG_NVCC_EXTRA=-DHG_JB_SWEEPMAX python -m paper_1908_08281_b200.build   # instrumented build
    python tools/jacobi_sweepmax.py [config index]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402

c = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda()
Y = torch.from_numpy(h.Y).cuda()
hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
torch.cuda.synchronize()
hg.debug_jacobi_sweepmax(True)
hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
torch.cuda.synchronize()
m = hg.debug_jacobi_sweepmax()
print("config", c)
for b in range(min(64, c.N // c.b)):
    seq = [x for x in m[b] if x > 0]
    print(b, len(seq), " ".join(f"{x:.1e}" for x in seq))
