"""configs[4] sweep: N=32768, b in {512,1024,2048}, k in {64..512}, q in {1,2,4} (36 points).

For every point: GPU solve time (CUDA events, median of reps), parity against the
FP64 oracle on blocks {0, nb-1} (F rel-Frobenius, sigma rel), accuracy of the
rank-k block inverse against the exact block solve c X_ii^-1 Y_i (FP64 LU) on
the same blocks, and accuracy of the whole GPU F against the full solve
F* = c X^-1 Y (FP64 block CG on the sparse operator; computed
once: it does not depend on b, k, q; the GPU CG of hg_cg_solve is checked against it).
Each point is also run with reading R2 (HG_WOODBURY: Alg. 1 on Theta_ii + Woodbury, §8(f)
NEXT-3): time, parity against the oracle's R2, accuracy against the same two references.
One JSON line per point.

    python tests/tools/sweep_cfg5.py [--points b,k,q ...] > profiles/r01_cfg5_sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import oracle  # noqa: E402
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, cfg5_points, make_input  # noqa: E402


def full_solve_cg(h, mu, tol=1e-10, maxit=200):
    """F* = c X^-1 Y, X = I - Theta/(1+mu), Theta = Dv^-1/2 H W De^-1 H^T Dv^-1/2,
    by block CG in FP64 with all T right-hand sides at once (X is SPD, cond(X) <= (1+mu)/mu)."""
    import scipy.sparse as sp
    N = len(h.row_ptr) - 1
    Hs = sp.csr_matrix((np.ones(len(h.col_idx)), h.col_idx, h.row_ptr), shape=(N, len(h.w)))
    w = h.w.astype(np.float64)
    de = np.asarray(Hs.sum(axis=0)).ravel()
    dv = Hs @ w
    dh = 1.0 / np.sqrt(dv)
    we = w / de
    c1 = 1.0 / (1.0 + mu)

    def A(V):
        Z = dh[:, None] * V
        Z = Hs.T @ Z
        Z = we[:, None] * Z
        Z = Hs @ Z
        return V - c1 * (dh[:, None] * Z)

    B = (mu / (1.0 + mu)) * h.Y.astype(np.float64)
    X = np.zeros_like(B)
    R = B.copy()
    P = R.copy()
    rs = np.sum(R * R, axis=0)
    bn = np.maximum(np.sum(B * B, axis=0), 1e-300)
    it = 0
    for it in range(1, maxit + 1):
        AP = A(P)
        alpha = rs / np.maximum(np.sum(P * AP, axis=0), 1e-300)
        X += alpha * P
        R -= alpha * AP
        rs_new = np.sum(R * R, axis=0)
        if np.max(np.sqrt(rs_new / bn)) < tol:
            break
        P = R + (rs_new / np.maximum(rs, 1e-300)) * P
        rs = rs_new
    return X, it


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
    t0 = time.time()
    Fstar, cg_it = full_solve_cg(h, base.mu)
    line = {"full_solve_cg": {"iterations": cg_it, "seconds": time.time() - t0, "norm": float(np.linalg.norm(Fstar))}}
    # the GPU CG (tol 1e-6) on the same system, against the FP64 reference
    Fc, itc, rrc, stc = hg.cg_solve(H, w, Y, mu=base.mu, max_iter=100, tol=1e-6)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hg.cg_solve(H, w, Y, mu=base.mu, max_iter=100, tol=1e-6, F=Fc, iters=itc, rel_res=rrc, status=stc,
                    sync=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    line["gpu_cg"] = {"solve_ms": float(np.median(ts)), "iterations_max": int(itc.max().item()),
                      "status": int(stc.item()),
                      "rel_vs_fp64_full_solve": float(np.linalg.norm(Fc.double().cpu().numpy() - Fstar) /
                                                      np.linalg.norm(Fstar))}
    print(json.dumps(line), flush=True)
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
            Fall = F.double().cpu().numpy()
            out["gpu_vs_full_solve"] = float(np.linalg.norm(Fall - Fstar) / np.linalg.norm(Fstar))
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
            # reading R2 on the same point
            F2, s2, st2 = hg.solve(H, w, Y, mu=c.mu, b=b, k=k, q=q, seed=0, ws=ws, sync=False, woodbury=True)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                hg.solve(H, w, Y, mu=c.mu, b=b, k=k, q=q, seed=0, ws=ws, F=F2, sigma=s2, status=st2, sync=False,
                         woodbury=True)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t0 = time.time()
            r2 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=b, k=k, q=q, seed=0, blocks=blocks,
                              woodbury=True)
            F2g = F2.double().cpu().numpy()
            s2g = s2.double().cpu().numpy()
            fe2, se2, acc2 = [], [], []
            for s_, blk in enumerate(blocks):
                fo = r2.F[s_ * b:(s_ + 1) * b]
                fe2.append(float(np.linalg.norm(F2g[blk * b:(blk + 1) * b] - fo) / np.linalg.norm(fo)))
                se2.append(float(np.max(np.abs(s2g[blk] - r2.sigma[s_]) / r2.sigma[s_])))
                exact = 0.5 * np.linalg.solve(r.X[s_], h.Y[blk * b:(blk + 1) * b].astype(np.float64))
                acc2.append(float(np.linalg.norm(fo - exact) / np.linalg.norm(exact)))
            out["r2"] = {"status": int(st2.item()), "solve_ms": float(np.median(ts)),
                         "parity_F_rel": max(fe2), "parity_sigma_rel": max(se2),
                         "parity_ok": max(fe2) <= 2e-5 and max(se2) <= 1e-5 and int(st2.item()) == 0,
                         "oracle_vs_exact_block_solve": max(acc2),
                         "gpu_vs_full_solve": float(np.linalg.norm(F2g - Fstar) / np.linalg.norm(Fstar)),
                         "oracle_s": time.time() - t0}
        except hg.HGError as e:
            out["error"] = str(e)
        print(json.dumps(out), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
