"""Per-stage timing + diagnostics for one config (development tool, GPU box).

    python tools/stage_probe.py 4 [--reps 3] [--no-parity]
Prints stage ms/step, debug counters (Cholesky path, Jacobi sweeps) and parity.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--b", type=int)
    ap.add_argument("--k", type=int)
    ap.add_argument("--q", type=int)
    ap.add_argument("--no-parity", action="store_true")
    a = ap.parse_args()
    c = CONFIGS[a.cfg]
    kw = {x: getattr(a, x) for x in ("b", "k", "q") if getattr(a, x) is not None}
    c = c.with_(**kw) if kw else c
    t0 = time.time()
    h = make_input(c)
    tgen = time.time() - t0
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    w = torch.from_numpy(h.w).cuda()
    Y = torch.from_numpy(h.Y).cuda()
    ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws)
    torch.cuda.synchronize()
    hg.debug_counters(reset=True)
    hg.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, sync=False)
    e1.record()
    prof = hg.profile_collect()
    hg.profile_enable(False)
    torch.cuda.synchronize()
    dbg = hg.debug_counters()
    clk = dbg.pop("chol_clk")
    if clk[0]:
        base = clk[0]
        dbg["chol_phases_kcyc"] = {i: round((v - base) / 1e3, 1) for i, v in enumerate(clk) if v}
    ic = dbg.pop("jac_inner_clk")
    if any(ic):
        base = min(x for x in ic if x)
        dbg["jac_inner_cyc"] = [[ic[12 * r + 3 * i + w] - base if ic[12 * r + 3 * i + w] else None for i in range(4)
                                 for w in range(3)] for r in range(4)]
    jc = dbg.pop("jac_clk")
    if jc[0]:
        dbg["jac_round_cyc"] = [jc[i] - jc[0] for i in range(16)]
    out = {"cfg": c.name, "b": c.b, "k": c.k, "q": c.q, "gen_s": tgen, "status": int(st.item()),
           "ms_per_step": e0.elapsed_time(e1) / a.reps,
           "stages": {k: round(v[0] / a.reps, 4) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])},
           "debug": dbg}
    if not a.no_parity:
        import oracle
        blocks = [0, c.nb - 1] if c.nb > 1 else [0]
        r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, blocks=blocks)
        Fg = F.double().cpu().numpy()
        sg = sigma.double().cpu().numpy()
        out["F_rel"] = max(float(np.linalg.norm(Fg[blk * c.b:(blk + 1) * c.b] - r.F[s * c.b:(s + 1) * c.b]) /
                                 np.linalg.norm(r.F[s * c.b:(s + 1) * c.b])) for s, blk in enumerate(blocks))
        out["sigma_rel"] = max(float(np.max(np.abs(sg[blk] - r.sigma[s]) / r.sigma[s]))
                               for s, blk in enumerate(blocks))
        out["oracle_s"] = r.seconds
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
