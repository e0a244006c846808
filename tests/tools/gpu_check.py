"""Quick GPU diagnostics: GEMM variants vs fp64 torch, Omega vs oracle, cfg1/cfg2 parity.

Prints one line per check; used during development on the B200 box.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import oracle  # noqa: E402
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check_gemm(simt):
    torch.manual_seed(0)
    for (M, N, K, batch) in [(128, 64, 128, 2), (256, 256, 1024, 3), (100, 20, 72, 2), (32, 32, 256, 4),
                             (1024, 256, 1024, 2), (300, 1000, 256, 2)]:
        for a_mn in (False, True):
            for b_mn in (False, True):
                for d_trans in (False, True):
                    A = torch.randn(batch, *( (K, M) if a_mn else (M, K)), device="cuda")
                    B = torch.randn(batch, *((K, N) if b_mn else (N, K)), device="cuda")
                    D = torch.full((batch, N, M) if d_trans else (batch, M, N), float("nan"), device="cuda")
                    hg.gemm(A, B, M=M, N=N, K=K, batch=batch, a_mn=a_mn, lda=A.shape[2], sa=A[0].numel(),
                            b_mn=b_mn, ldb=B.shape[2], sb=B[0].numel(), D=D, d_trans=d_trans, ldd=D.shape[2],
                            sd=D[0].numel(), simt=simt)
                    torch.cuda.synchronize()
                    Ad = A.double().cpu()
                    Bd = B.double().cpu()
                    Am = Ad.transpose(1, 2) if a_mn else Ad
                    Bm = Bd if b_mn else Bd.transpose(1, 2)
                    ref = Am @ Bm
                    got = D.double().cpu()
                    if d_trans:
                        got = got.transpose(1, 2)
                    err = float((got - ref).norm() / ref.norm())
                    ok = err < 5e-6 and torch.isfinite(got).all()
                    print(f"gemm simt={int(simt)} M={M} N={N} K={K} b={batch} a_mn={int(a_mn)} b_mn={int(b_mn)} "
                          f"d_trans={int(d_trans)} rel={err:.2e} {'OK' if ok else 'FAIL'}", flush=True)


def check_omega():
    g = hg.fill_gaussian(0, 1000, 33).cpu().numpy()
    o = oracle.gaussian_f32(0, 1000 * 33).reshape(1000, 33)
    d = np.abs(g.view(np.int32).astype(np.int64) - o.view(np.int32).astype(np.int64))
    print(f"omega exact={np.mean(d == 0):.6f} max_ulp={d.max()}", flush=True)


def check_cfg(i, simt=False, blocks=None):
    c = CONFIGS[i]
    h = make_input(c)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    w = torch.from_numpy(h.w).cuda()
    Y = torch.from_numpy(h.Y).cuda()
    # theta parity
    th, dvr, st = hg.build_theta(H, w, c.mu, c.b, raw=True)
    torch.cuda.synchronize()
    sel = blocks if blocks is not None else list(range(min(c.nb, 4)))
    terr = 0.0
    for blk in sel[:2]:
        ref = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, blk)
        got = th[blk].double().cpu().numpy()
        terr = max(terr, np.abs(got - ref).max() / np.abs(ref).max())
    sym = bool((th == th.transpose(1, 2)).all())
    print(f"cfg{i} theta max_err/max={terr:.2e} symmetric={sym} status={int(st.item())}", flush=True)
    t0 = time.time()
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, simt=simt)
    torch.cuda.synchronize()
    t1 = time.time()
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, blocks=sel)
    Fg = F.double().cpu().numpy()
    sg = sigma.double().cpu().numpy()
    ferr = max(rel(Fg[blk * c.b:(blk + 1) * c.b], r.F[s * c.b:(s + 1) * c.b]) for s, blk in enumerate(sel))
    serr = max(float(np.max(np.abs(sg[blk] - r.sigma[s]) / r.sigma[s])) for s, blk in enumerate(sel))
    print(f"cfg{i} simt={int(simt)} F_rel={ferr:.2e} sigma_rel={serr:.2e} status={int(st.item())} "
          f"gpu_s={t1 - t0:.3f} oracle_s={r.seconds:.2f}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["omega", "simt", "tc", "cfg1s", "cfg1", "cfg2", "cfg3"]
    for wname in which:
        try:
            if wname == "omega":
                check_omega()
            elif wname == "simt":
                check_gemm(True)
            elif wname == "tc":
                check_gemm(False)
            elif wname == "cfg1s":
                check_cfg(1, simt=True)
            elif wname.startswith("cfg"):
                check_cfg(int(wname[3:]))
        except Exception as e:  # keep going to collect more information
            print(f"{wname} EXC {type(e).__name__}: {e}", flush=True)
            torch.cuda.synchronize()
