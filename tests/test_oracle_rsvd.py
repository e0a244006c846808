"""Oracle pins for Alg. 1 and the Eq. 3/15 apply (CPU only).

Pins: exact rank-k recovery (P4),
diagonal blocks (P5), identity (P6), k = b against LAPACK eigvalsh / LU (P3),
the closed form M = X^T Z (Z^T X X^T Z)^-1 Z^T with Z = (X X^T)^q X Omega
(P7, derived in DESIGN.md), Petrov-Galerkin invariants (P8), brute force on
tiny inputs (P10), monotone range capture and the Eckart-Young bound (P11).
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth.hypergraph import CONFIGS, make_tiny

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def closed_form_M(X, Om, q):
    Z = X @ Om
    for _ in range(q):
        Z = X @ (X.T @ Z)
    return X.T @ Z @ np.linalg.solve(Z.T @ X @ X.T @ Z, Z.T)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_exact_rank_k_block_recovered():
    # P4: X = G G^T (G b x k) is recovered to 1e-10 and Sigma = nonzero eig(X)
    rng = np.random.default_rng(1)
    for b, k, q in [(64, 5, 0), (64, 5, 2), (128, 16, 1)]:
        G = rng.standard_normal((b, k))
        X = G @ G.T
        U, s, V, resid = oracle.rsvd_block(X, rng.standard_normal((b, k)), q)
        assert rel(U @ np.diag(s) @ V.T, X) <= 1e-10
        assert resid <= 1e-10 * np.linalg.norm(X)
        np.testing.assert_allclose(s, np.linalg.eigvalsh(G.T @ G)[::-1], rtol=1e-10)


def test_diagonal_blocks():
    # P5: SPEC.md:132 diag(5,4,3,0,0), k=3 -> (5,4,3); distinct diagonal with k=b -> sorted diagonal
    g = GOLD["rsvd_diag54300"]
    X = np.diag(np.array(g["X"], float))
    rng = np.random.default_rng(2)
    _, s, _, _ = oracle.rsvd_block(X, rng.standard_normal((5, g["k"])), 2)
    np.testing.assert_allclose(s, g["sigma"], rtol=1e-12)
    d = rng.uniform(0.5, 1.0, 24)
    _, s, _, _ = oracle.rsvd_block(np.diag(d), rng.standard_normal((24, 24)), 1)
    np.testing.assert_allclose(s, np.sort(d)[::-1], rtol=1e-12)


@pytest.mark.parametrize("b,k", [(16, 4), (32, 32), (40, 13)])
def test_identity_block(b, k):
    # P6: SPEC.md:123 -- ||I - S S^T I||_F = sqrt(b - k); sigma = 1; M = S S^T
    rng = np.random.default_rng(b + k)
    U, s, V, resid, S = oracle.rsvd_block(np.eye(b), rng.standard_normal((b, k)), 1, want_S=True)
    np.testing.assert_allclose(s, 1.0, rtol=1e-13)
    assert abs(resid - np.sqrt(b - k)) < 1e-12
    M = V @ np.diag(1 / s) @ U.T
    np.testing.assert_allclose(M, S @ S.T, atol=1e-13)


@pytest.mark.parametrize("name", ["invert_diag24", "inverse_2112"])
def test_k_equals_b_small_inverses_golden(name):
    # SPEC.md:150 / SPEC.md:209: with k = b, V Sigma^-1 U^T = X^-1 (Eq. 15)
    g = GOLD[name]
    X = np.array(g["X"], float)
    U, s, V, _ = oracle.rsvd_block(X, np.random.default_rng(0).standard_normal((2, 2)), 1)
    F = oracle.apply_block(U, s, V, np.eye(2), 1.0)
    np.testing.assert_allclose(F, g["Xinv"], atol=1e-14)


def test_k_equals_b_on_hypergraph_blocks(cfg_inputs):
    # P3: Sigma = eigvalsh(X_ii) (X_ii is SPD); X M = I; F = c * LU solve
    h = cfg_inputs(1)
    b = 128
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=b, k=b, q=1, seed=0,
                     blocks=[0, 3], want_UV=True, want_X=True)
    for s_, blk in enumerate(r.blocks):
        X = r.X[s_]
        np.testing.assert_allclose(r.sigma[s_], np.linalg.eigvalsh(X)[::-1], rtol=1e-12)
        M = r.V[s_] @ np.diag(1 / r.sigma[s_]) @ r.U[s_].T
        assert np.abs(X @ M - np.eye(b)).max() <= 1e-9
        Yi = h.Y[blk * b:(blk + 1) * b].astype(float)
        F_lu = 0.5 * np.linalg.solve(X, Yi)
        assert rel(r.F[s_ * b:(s_ + 1) * b], F_lu) <= 1e-11


def test_single_block_is_eq3_exactly():
    # tiny N with b = N: the path is f* = c X^-1 y (Eq. 3) on the whole hypergraph
    h = make_tiny(24, 24, 24, 2)
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=24, k=24, q=2, seed=1, want_X=True)
    X = r.X[0]
    # X from Eq. 1 built densely with numpy (independent of the oracle's sparse loop)
    H = np.zeros((h.N, h.E))
    for v in range(h.N):
        H[v, h.col_idx[h.row_ptr[v]:h.row_ptr[v + 1]]] = 1
    w = h.w.astype(float)
    dv, de = H @ w, H.sum(0)
    Th = np.diag(dv ** -0.5) @ H @ np.diag(w / de) @ H.T @ np.diag(dv ** -0.5)
    np.testing.assert_allclose(X, np.eye(24) - Th / 2, atol=1e-14)
    assert rel(r.F, 0.5 * np.linalg.solve(X, h.Y.astype(float))) < 1e-12


@pytest.mark.parametrize("q", [0, 1, 2])
def test_closed_form_cfg1(cfg_inputs, q):
    # P7: F_i = c X^T Z (Z^T X X^T Z)^-1 Z^T Y_i, Z = (X X^T)^q X Omega_i, LAPACK solve in FP64
    h = cfg_inputs(1)
    c = CONFIGS[1]
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=c.b, k=c.k, q=q, seed=0, want_X=True)
    Om = oracle.omega(0, c.N, c.k).astype(float)
    for s_, blk in enumerate(r.blocks):
        M = closed_form_M(r.X[s_], Om[blk * c.b:(blk + 1) * c.b], q)
        Fc = 0.5 * M @ h.Y[blk * c.b:(blk + 1) * c.b].astype(float)
        assert rel(r.F[s_ * c.b:(s_ + 1) * c.b], Fc) <= 1e-10


def test_brute_force_tiny():
    # P10: N = 8, b = 4, every k in 1..4 and q in 0..2 against the closed form; k = b against LU
    h = make_tiny(8, 4, 4, 0, K=2, n_tag=3)
    Om_all = oracle.omega(11, 8, 4)
    for k in range(1, 5):
        Om = oracle.omega(11, 8, k).astype(float)
        for q in range(3):
            r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=4, k=k, q=q, seed=11, want_X=True)
            for s_, blk in enumerate(r.blocks):
                X = r.X[s_]
                Yi = h.Y[blk * 4:(blk + 1) * 4].astype(float)
                Fc = 0.5 * closed_form_M(X, Om[blk * 4:(blk + 1) * 4], q) @ Yi
                Fo = r.F[s_ * 4:(s_ + 1) * 4]
                assert np.abs(Fo - Fc).max() <= 1e-12 * max(1, np.abs(Fc).max())
                if k == 4:
                    assert np.abs(Fo - 0.5 * np.linalg.solve(X, Yi)).max() <= 1e-12
    assert Om_all.shape == (8, 4)


def test_petrov_galerkin_invariants(cfg_inputs):
    # P8: S^T (X F - c Y) = 0, (I - V V^T) F = 0, M X M = M
    h = cfg_inputs(1)
    c = CONFIGS[1]
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=c.b, k=c.k, q=c.q, seed=0,
                     blocks=[1], want_UV=True, want_X=True)
    X, U, V, s = r.X[0], r.U[0], r.V[0], r.sigma[0]
    Om = oracle.omega(0, c.N, c.k).astype(float)[c.b:2 * c.b]
    _, _, _, _, S = oracle.rsvd_block(X, Om, c.q, want_S=True)
    Yi = h.Y[c.b:2 * c.b].astype(float)
    F = r.F
    assert np.abs(S.T @ (X @ F - 0.5 * Yi)).max() < 1e-12
    assert np.abs(F - V @ (V.T @ F)).max() < 1e-12
    M = V @ np.diag(1 / s) @ U.T
    assert np.abs(M @ X @ M - M).max() < 1e-12
    # sign rule: largest-|.| entry of each U column is >= 0
    idx = np.abs(U).argmax(0)
    assert np.all(U[idx, np.arange(c.k)] > 0)


def test_monotone_range_capture_and_eckart_young(cfg_inputs):
    # P11: SPEC.md:156 -- more passes never (materially) increase ||X - S S^T X||_F,
    # and no rank-k basis beats the tail of the spectrum
    h = cfg_inputs(2)
    b, k = 256, 64
    X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, b, 2, mu=1.0)
    Om = oracle.omega(0, h.N, k).astype(float)[2 * b:3 * b]
    res = [oracle.rsvd_block(X, Om, q)[3] for q in range(4)]
    assert all(res[i + 1] <= res[i] + 1e-10 for i in range(3))
    sv = np.linalg.svd(X, compute_uv=False)
    assert res[-1] >= np.sqrt((sv[k:] ** 2).sum()) - 1e-10


def test_sigma_bracket_and_determinism(cfg_inputs):
    # P2 on the rSVD output: sigma(B) in [mu/(1+mu), 1]; bit-identical reruns
    h = cfg_inputs(2)
    c = CONFIGS[2]
    r1 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=c.b, k=c.k, q=c.q, seed=0, blocks=[0, 7, 15])
    r2 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=c.b, k=c.k, q=c.q, seed=0, blocks=[15, 0])
    assert r1.sigma.max() <= 1 + 1e-12 and r1.sigma.min() >= 0.5 - 1e-12
    assert np.array_equal(r1.sigma[0], r2.sigma[1]) and np.array_equal(r1.F[-c.b:], r2.F[:c.b])
    assert np.all(np.diff(r1.sigma, axis=1) <= 0)


def test_invalid_arguments():
    h = make_tiny(16, 8, 4, 1)
    for kw in [dict(b=5, k=2, q=1), dict(b=8, k=9, q=1), dict(b=8, k=0, q=1), dict(b=8, k=2, q=-1)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, seed=0, **kw)
        assert e.value.status == oracle.ERR_INVALID
    with pytest.raises(oracle.OracleError):
        oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=0.0, b=8, k=2, q=1, seed=0)
