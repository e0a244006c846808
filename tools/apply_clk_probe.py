"""Per-CTA phase timeline of one k_apply_fused launch from %globaltimer stamps.
Needs a library built with HG_NVCC_EXTRA=-DHG_APPLY_CLK (debug build, never the shipped one):
    HG_STREAMS=1 python tools/apply_clk_probe.py
slots: 0 entry, 1 setup done, 2 first MMA, 3 last product-1 MMA issued, 4 product-1 drained,
5 Z in shared memory (MMA warp released), 6+2mt F tile mt accumulated, 22+mt drained from TMEM,
7+2mt stored, 31 exit."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402

c = CONFIGS[int(os.environ.get("CFG", "4"))]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda()
Y = torch.from_numpy(h.Y).cuda()
ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, sync=False)
for _ in range(2):
    hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F, sigma=sigma, status=st, sync=False)
torch.cuda.synchronize()
n = 160 * 32
out = (ctypes.c_ulonglong * n)()
hg._lib.hg_debug_apply_clk(out, n)
a = np.array(out[:], dtype=np.int64).reshape(160, 32)
t0 = a[:, 0][a[:, 0] > 0].min()
print("status", int(st.item()), "ctas stamped", int((a[:, 0] > 0).sum()), "span us", (a[:, 31].max() - t0) / 1e3)
for cta in (0, 1, 7, 80, 147, 148, 159):
    r = a[cta]
    if r[0] == 0:
        continue
    rel = (r - r[0]) / 1e3
    print(f"cta {cta}: entry {(r[0]-t0)/1e3:.1f} us; setup {rel[1]:.1f} mma0 {rel[2]:.1f} mma_last {rel[3]:.1f} "
          f"drained {rel[4]:.1f} zs {rel[5]:.1f} exit {rel[31]:.1f}")
    print("   F tiles (accumulated, drained, stored):",
          " ".join(f"({rel[6+2*m]:.1f},{rel[22+m]:.1f},{rel[7+2*m]:.1f})" for m in range(8)))
