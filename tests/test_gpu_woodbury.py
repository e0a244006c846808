"""GPU parity for reading R2: Alg. 1 on Theta_ii and the Woodbury
inverse of X_ii, through the C ABI (hg_solve with HG_WOODBURY; hg_build_theta(HG_RAW_THETA) ->
hg_block_rsvd -> hg_block_apply_woodbury), against the FP64 oracle's R2 (or_solve_mode 1).

Tolerances as for R1 (north_star): F relative Frobenius <= 2e-5, sigma relative <= 1e-5.
"""
import numpy as np
import pytest
import torch

import oracle
from synth.hypergraph import CONFIGS, make_input, make_tiny

pytestmark = pytest.mark.gpu

F_TOL, SIG_TOL = 2e-5, 1e-5
_inp = {}


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def get(cfg):
    if cfg not in _inp:
        h = make_input(CONFIGS[cfg])
        hg = hgm()
        _inp[cfg] = (h, hg.incidence_to_device(h.row_ptr, h.col_idx, h.E), torch.from_numpy(h.w).cuda(),
                     torch.from_numpy(h.Y).cuda())
    return _inp[cfg]


def check(h, c, F, sigma, blocks, k=None):
    k = k or c.k
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=k, q=c.q, seed=c.seed, blocks=blocks,
                     woodbury=True)
    Fg, sg = F.double().cpu().numpy(), sigma.double().cpu().numpy()
    for s_, blk in enumerate(blocks):
        assert rel(Fg[blk * c.b:(blk + 1) * c.b], r.F[s_ * c.b:(s_ + 1) * c.b]) <= F_TOL, blk
        assert np.max(np.abs(sg[blk] - r.sigma[s_]) / r.sigma[s_]) <= SIG_TOL, blk
    return r


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_woodbury_solve_parity(cfg):
    hg = hgm()
    h, H, w, Y = get(cfg)
    c = CONFIGS[cfg]
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed, woodbury=True)
    assert int(st.item()) == 0
    check(h, c, F, sigma, list(range(c.nb)))
    # the three entry points in sequence give the same bits as the composite
    Th, _, _ = hg.build_theta(H, w, c.mu, c.b, raw=True)
    Ut, s2, Vt, st2 = hg.block_rsvd(Th, c.k, c.q, c.seed, x_unit=True)   # Theta_ii: |.| <= 1, ||.|| <= 1
    F2, st3 = hg.block_apply_woodbury(Ut, s2, Y, c.mu)
    torch.cuda.synchronize()
    assert int(st2.item()) == 0 and int(st3.item()) == 0
    assert torch.equal(F, F2) and torch.equal(sigma, s2)


def test_woodbury_config4_sampled_blocks():
    hg = hgm()
    h, H, w, Y = get(4)
    c = CONFIGS[4]
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed, woodbury=True)
    assert int(st.item()) == 0
    check(h, c, F, sigma, [0, c.nb // 2, c.nb - 1])


def test_woodbury_k_equals_b_is_exact_block_inverse():
    hg = hgm()
    for (N, b, q) in [(48, 16, 1), (64, 32, 2)]:
        h = make_tiny(N, b, b, q)
        H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
        F, sigma, st = hg.solve(H, torch.from_numpy(h.w).cuda(), torch.from_numpy(h.Y).cuda(), mu=1.0, b=b, k=b,
                                q=q, seed=0, woodbury=True)
        assert int(st.item()) == 0
        Fg = F.double().cpu().numpy()
        for blk in range(N // b):
            X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, b, blk, mu=1.0)
            lu = 0.5 * np.linalg.solve(X, h.Y[blk * b:(blk + 1) * b].astype(float))
            assert rel(Fg[blk * b:(blk + 1) * b], lu) <= F_TOL


def test_woodbury_accuracy_vs_exact_block_solve():
    hg = hgm()
    h, H, w, Y = get(2)
    c = CONFIGS[2]
    F, _, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed, woodbury=True)
    Fg = F.double().cpu().numpy()
    for blk in (0, c.nb - 1):
        X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, blk, mu=c.mu)
        ex = c.mu / (1 + c.mu) * np.linalg.solve(X, h.Y[blk * c.b:(blk + 1) * c.b].astype(float))
        assert rel(Fg[blk * c.b:(blk + 1) * c.b], ex) <= 5e-2


def test_woodbury_rank_deficient_theta_blocks():
    """Degenerate case: Theta_ii of rank 2 < k (every vertex of a block lies on the same two
    hyperedges).  Alg. 1's extra directions carry sigma ~ 0, so their Woodbury weights vanish and F is
    still determined; the GPU's shifted CholeskyQR must not break down or produce non-finite values."""
    hg = hgm()
    b, nblk, T = 16, 2, 4
    rows = []
    for blk in range(nblk):
        for v in range(b):
            es = [2 * blk] + ([2 * blk + 1] if v < b // 2 else [])
            rows.append(es)
    rp = np.array([0] + list(np.cumsum([len(r) for r in rows])), np.int64)
    ci = np.array([e for r in rows for e in r], np.int32)
    w = np.array([1.0, 0.5, 1.5, 1.0], np.float32)
    Y = np.random.default_rng(0).integers(0, 2, (b * nblk, T)).astype(np.float32)
    H = hg.incidence_to_device(rp, ci, 4)
    F, sigma, st = hg.solve(H, torch.from_numpy(w).cuda(), torch.from_numpy(Y).cuda(), mu=1.0, b=b, k=8, q=1,
                            seed=0, woodbury=True)
    assert int(st.item()) == 0 and bool(torch.isfinite(F).all())
    r = oracle.solve(rp, ci, w, Y, mu=1.0, b=b, k=8, q=1, seed=0, woodbury=True)
    assert rel(F.double().cpu().numpy(), r.F) <= F_TOL
    # exact: Theta_ii has rank 2 <= k, so the Woodbury inverse is exact (the block solve)
    for blk in range(nblk):
        X = oracle.theta_block(rp, ci, w, b, blk, mu=1.0)
        ex = 0.5 * np.linalg.solve(X, Y[blk * b:(blk + 1) * b].astype(float))
        assert rel(F[blk * b:(blk + 1) * b].double().cpu().numpy(), ex) <= F_TOL
    # the factorisation itself stays finite: the right vectors of the (near-)zero sigma are written
    # as 0, not inf/NaN (finalize.cu k_rows)
    X, _, _ = hg.build_theta(H, torch.from_numpy(w).cuda(), 1.0, b, raw=True)
    Ut, sg, Vt, st2 = hg.block_rsvd(X, 8, 1, 0)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(Ut).all()) and bool(torch.isfinite(Vt).all()) and bool(torch.isfinite(sg).all())
