"""Run W warm-up steps and then ONE step of the bench workload (for ncu launch lists).

    python tools/step_once.py [--config 4] [--warmup 2]
Prints the number of library launches per step, so an ncu command can skip the
warm-up launches and capture exactly one step:
    ncu -k regex:"gemm_tf32|k_" -s <warmup * L> -c <L> ... python tools/step_once.py
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    h = make_input(c)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    w = torch.from_numpy(h.w).cuda()
    Y = torch.from_numpy(h.Y).cuda()
    ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, sync=False)
    for _ in range(a.warmup - 1):
        hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F, sigma=sigma, status=st, sync=False)
    torch.cuda.synchronize()
    n = hg.last_launch_count()
    hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F, sigma=sigma, status=st, sync=False)
    torch.cuda.synchronize()
    print(f"launches_per_step {n} status {int(st.item())}")


if __name__ == "__main__":
    main()
