"""Time hg_cg_solve (graph mode) on a config: ms per solve, iterations, parity on sampled columns.

    python tools/cg_probe.py [--cfg 4] [--tol 1e-6] [--reps 10] [--direct]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1908_08281_b200 import hg
from synth.hypergraph import CONFIGS, make_input

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--max-iter", type=int, default=100)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--direct", action="store_true")
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
if a.direct:
    os.environ["HG_NO_GRAPH"] = "1"
c = CONFIGS[a.cfg]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda()
Y = torch.from_numpy(h.Y).cuda()
N, T = Y.shape
ws = hg.Workspace(hg.cg_workspace_size(N, h.E, h.nnz, T, a.max_iter))
F = torch.empty_like(Y)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(a.warmup):
    hg.cg_solve(H, w, Y, mu=c.mu, max_iter=a.max_iter, tol=a.tol, ws=ws, F=F, status=st, sync=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    _, it, rr, _ = hg.cg_solve(H, w, Y, mu=c.mu, max_iter=a.max_iter, tol=a.tol, ws=ws, F=F, status=st, sync=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
it = it.cpu().numpy()
print(json.dumps({"cfg": a.cfg, "N": N, "T": T, "nnz": h.nnz, "ms": ms, "iters_max": int(it.max()),
                  "iters_mean": float(it.mean()), "rel_res_max": float(rr.max().item()), "status": int(st.item()),
                  "launches": hg.last_launch_count(), "direct": a.direct}))
