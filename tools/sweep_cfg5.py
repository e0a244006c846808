"""configs[4] sweep: N=32768, b in {512,1024,2048}, k in {64..512}, q in {1,2,4} (36 points).

For every point: GPU solve time (CUDA events, median of reps), parity against the
FP64 oracle on blocks {0, nb-1} (F rel-Frobenius, sigma rel), and accuracy of the
rank-k block inverse against the exact block solve c X_ii^-1 Y_i (FP64 LU) on
the same blocks.  One JSON line per point.

    python tools/sweep_cfg5.py [--points b,k,q ...] > profiles/r01_cfg5_sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, cfg5_points, make_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", nargs="*")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    pts = [tuple(map(int, p.split(","))) for p in a.points] if a.points else cfg5_points()
    base = CONFIGS[5]
    h = make_input(base)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    w = torch.from_numpy(h.w).cuda()
    Y = torch.from_numpy(h.Y).cuda()
    for (b, k, q) in pts:
        c = base.with_(b=b, k=k, q=q)
        out = {"b": b, "k": k, "q": q, "nb": c.nb}
        try:
            ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, b, k, c.T)
            F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=b, k=k, q=q, seed=0, ws=ws, sync=False)
            torch.cuda.synchronize()
            out["status"] = int(st.item())
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                hg.solve(H, w, Y, mu=c.mu, b=b, k=k, q=q, seed=0, ws=ws, F=F, sigma=sigma, status=st, sync=False)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            out.update({"solve_ms": ms, "blocks_per_s": c.nb / (ms / 1e3),
                        "gemm_useful_gflop": 4.0 * (q + 1) * c.N * b * k / 1e9})
            blocks = [0, c.nb - 1]
            t0 = time.time()
            r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=b, k=k, q=q, seed=0, blocks=blocks,
                             want_X=True)
            Fg = F.double().cpu().numpy()
            sg = sigma.double().cpu().numpy()
            fe, se, acc = [], [], []
            for s_, blk in enumerate(blocks):
                fo = r.F[s_ * b:(s_ + 1) * b]
                fe.append(float(np.linalg.norm(Fg[blk * b:(blk + 1) * b] - fo) / np.linalg.norm(fo)))
                se.append(float(np.max(np.abs(sg[blk] - r.sigma[s_]) / r.sigma[s_])))
                exact = 0.5 * np.linalg.solve(r.X[s_], h.Y[blk * b:(blk + 1) * b].astype(np.float64))
                acc.append(float(np.linalg.norm(fo - exact) / np.linalg.norm(exact)))
            out.update({"parity_F_rel": max(fe), "parity_sigma_rel": max(se), "parity_ok": max(fe) <= 2e-5 and
                        max(se) <= 1e-5 and out["status"] == 0,
                        "oracle_vs_exact_block_solve": max(acc), "oracle_s": time.time() - t0})
        except hg.HGError as e:
            out["error"] = str(e)
        print(json.dumps(out), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
