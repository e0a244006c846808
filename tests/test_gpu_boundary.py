"""GPU: the boundary variants of include/hg.h against the FP64 oracle.

  * HG_GENERAL -- Alg. 1 on non-symmetric blocks with the literal X^T of PAPER.md:116 (the
    oracle always multiplies by the literal transpose);
  * HG_UV_BK   -- U, V returned / taken as [nb][b][k] (SURVEY.md §8(b) layout);
  * T % 4 != 0 -- any number of right-hand sides (Eq. 3 / Eq. 15 per column);
  * hg_weight_normalize -- the simplex start w / 1^T w.
Tolerances as tests/test_gpu_parity.py (north_star): F <= 2e-5, sigma <= 1e-5 relative.
"""
import numpy as np
import pytest
import torch

import oracle
from synth.hypergraph import CONFIGS, make_input

pytestmark = pytest.mark.gpu

F_TOL, SIG_TOL = 2e-5, 1e-5


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def cfg1():
    c = CONFIGS[1]
    h = make_input(c)
    hg = hgm()
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    return c, h, H, torch.from_numpy(h.w).cuda(), torch.from_numpy(h.Y).cuda()


def _nonsymmetric_blocks(c, h, eps=0.05, seed=7):
    """X_ii of configs[0] plus a dense non-symmetric perturbation (still well conditioned)."""
    rng = np.random.default_rng(seed)
    Xs = []
    for i in range(c.nb):
        X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, i, mu=c.mu)
        R = rng.standard_normal((c.b, c.b)) / np.sqrt(c.b)
        Xs.append((X + eps * R).astype(np.float32))
    return np.stack(Xs)


def test_general_block_matches_literal_transpose_oracle(cfg1):
    c, h, _, _, _ = cfg1
    hg = hgm()
    Xn = _nonsymmetric_blocks(c, h)
    Xd = torch.from_numpy(Xn).cuda()
    Ut, sigma, Vt, st = hg.block_rsvd(Xd, c.k, c.q, c.seed, general=True)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    Om = oracle.omega(c.seed, c.nb * c.b, c.k)
    sg = sigma.double().cpu().numpy()
    err_s = err_r = 0.0
    for i in range(c.nb):
        U, s, V, _ = oracle.rsvd_block(Xn[i].astype(np.float64), Om[i * c.b:(i + 1) * c.b].astype(np.float64), c.q)
        err_s = max(err_s, float(np.max(np.abs(sg[i] - s) / s)))
        rec = Ut[i].double().cpu().numpy().T @ np.diag(sg[i]) @ Vt[i].double().cpu().numpy()
        err_r = max(err_r, rel(rec, U @ np.diag(s) @ V.T))
    assert err_s <= SIG_TOL and err_r <= F_TOL, (err_s, err_r)
    # the symmetric shortcut (X^T = X, reading A12) is measurably wrong on these blocks
    Ut2, sigma2, Vt2, _ = hg.block_rsvd(Xd, c.k, c.q, c.seed)
    rec2 = Ut2[0].double().cpu().numpy().T @ np.diag(sigma2[0].double().cpu().numpy()) @ Vt2[0].double().cpu().numpy()
    U, s, V, _ = oracle.rsvd_block(Xn[0].astype(np.float64), Om[:c.b].astype(np.float64), c.q)
    assert rel(rec2, U @ np.diag(s) @ V.T) > 1e-3


def test_general_equals_default_on_symmetric_blocks(cfg1):
    """On bitwise-symmetric blocks the literal X^T products equal the X products to rounding."""
    c, h, H, w, _ = cfg1
    hg = hgm()
    X, _, _ = hg.build_theta(H, w, c.mu, c.b)
    Ut, s, Vt, _ = hg.block_rsvd(X, c.k, c.q, c.seed)
    Ug, sgn, Vg, st = hg.block_rsvd(X, c.k, c.q, c.seed, general=True)
    assert int(st.item()) == 0
    assert float((s - sgn).abs().max() / s.abs().max()) <= 1e-6


def test_uv_bk_layout_and_apply(cfg1):
    c, h, H, w, Y = cfg1
    hg = hgm()
    X, _, _ = hg.build_theta(H, w, c.mu, c.b)
    Ut, sigma, Vt, st = hg.block_rsvd(X, c.k, c.q, c.seed)
    U, sigma2, V, st2 = hg.block_rsvd(X, c.k, c.q, c.seed, uv_bk=True)
    assert int(st.item()) == 0 and int(st2.item()) == 0
    assert U.shape == (c.nb, c.b, c.k) and V.shape == (c.nb, c.b, c.k)
    assert torch.equal(U, Ut.transpose(1, 2)) and torch.equal(V, Vt.transpose(1, 2)) and torch.equal(sigma, sigma2)
    scale = c.mu / (1 + c.mu)
    F1, _ = hg.block_apply_inverse(Ut, sigma, Vt, Y, scale)
    F2, st3 = hg.block_apply_inverse_ex(U, sigma, V, Y, scale, uv_bk=True)
    assert int(st3.item()) == 0
    assert float((F1 - F2).norm() / F1.norm()) <= 1e-6


@pytest.mark.parametrize("T", [7, 1, 13])
def test_ragged_T_solve_matches_oracle(cfg1, T):
    c, h, H, w, Y = cfg1
    hg = hgm()
    Yt = Y[:, :T].contiguous()
    F, sigma, st = hg.solve(H, w, Yt, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    assert int(st.item()) == 0 and F.shape == (c.N, T)
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, np.ascontiguousarray(h.Y[:, :T]), mu=c.mu, b=c.b, k=c.k, q=c.q,
                     seed=c.seed)
    assert rel(F.double().cpu().numpy(), r.F) <= F_TOL
    # the columns are independent: the same as those columns of the full right-hand side
    Ff, _, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    assert float((F - Ff[:, :T]).norm() / Ff[:, :T].norm()) <= 1e-6
    # the host entry too
    Fh, _ = hg.solve_host(torch.from_numpy(h.row_ptr), torch.from_numpy(h.col_idx), torch.from_numpy(h.w),
                          torch.from_numpy(np.ascontiguousarray(h.Y[:, :T])), mu=c.mu, b=c.b, k=c.k, q=c.q,
                          seed=c.seed)
    assert rel(Fh.double().numpy(), r.F) <= F_TOL


def test_weight_normalize():
    hg = hgm()
    rng = np.random.default_rng(3)
    w = rng.uniform(0.5, 1.5, 1000).astype(np.float32)
    wo, st = hg.weight_normalize(torch.from_numpy(w).cuda())
    assert int(st.item()) == 0
    ref = w.astype(np.float64) / w.astype(np.float64).sum()
    assert np.abs(wo.double().cpu().numpy() - ref).max() <= 1e-7 * ref.max()
    w[5] = -1.0
    wo2, st2 = hg.weight_normalize(torch.from_numpy(w).cuda())
    assert int(st2.item()) == 128   # HG_ST_SIMPLEX_DEGENERATE
