"""Per-part stage timeline of one hg_solve (HG_STREAMS parts concurrent), from the
library's stage events (hg_profile_enable(2)).

    python tools/timeline.py [--config 4] [--parts 2] [--json out.json]
Prints, per part, each stage group's [start, end] in ms from the solve start, and a
coarse text Gantt (one row per part, one column per 0.1 ms).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402

LETTER = {"degrees": "d", "assemble": "A", "omega": "o", "gemm_power": "P", "gemm_gram": "g", "gemm_qform": "q",
          "gemm_svd": "s", "gemm_apply": "a", "cholinv": "C", "jacobi": "J", "finalize": "f", "inv_sigma": "i",
          "eig_precond": "E"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--parts", type=int, default=2)
    ap.add_argument("--json")
    a = ap.parse_args()
    os.environ["HG_STREAMS"] = str(a.parts)
    c = CONFIGS[a.config]
    h = make_input(c)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    w = torch.from_numpy(h.w).cuda()
    Y = torch.from_numpy(h.Y).cuda()
    ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
    F, s, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, sync=False)
    for _ in range(3):
        hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F, sigma=s, status=st, sync=False)
    torch.cuda.synchronize()
    hg.profile_enable(2)
    hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F, sigma=s, status=st, sync=False)
    torch.cuda.synchronize()
    recs = hg.profile_timeline()
    hg.profile_enable(0)
    end = max(r[3] for r in recs)
    print(f"{c.name}: {len(recs)} stage groups, solve {end:.2f} ms, {a.parts} parts")
    for p in sorted(set(r[1] for r in recs)):
        rows = [r for r in recs if r[1] == p]
        tot = {}
        for r in rows:
            tot[r[0]] = tot.get(r[0], 0.0) + (r[3] - r[2])
        print(f"part {p}: [{min(r[2] for r in rows):.2f}, {max(r[3] for r in rows):.2f}] ms; busy by stage: " +
              ", ".join(f"{k} {v:.2f}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])))
        line = [" "] * (int(end * 10) + 1)
        for r in rows:
            for x in range(int(r[2] * 10), max(int(r[2] * 10) + 1, int(r[3] * 10))):
                line[x] = LETTER[r[0]]
        print("  " + "".join(line))
    if a.json:
        json.dump([{"stage": r[0], "part": r[1], "t0_ms": r[2], "t1_ms": r[3]} for r in recs], open(a.json, "w"))


if __name__ == "__main__":
    main()
