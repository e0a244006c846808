"""Oracle pins for the primitives (CPU only): Philox/Omega, degrees, Eq. 1, QR, SVD.

Each test pins an oracle function to something other than itself: a library
implementation (numpy's Philox, LAPACK via numpy), a closed form, a worked
example (tests/golden/spec_examples.json, each cited) or an invariant the
mathematics fixes.
"""
import json
import os

import numpy as np
import pytest
from scipy import stats

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------- Omega (A6)
@pytest.mark.parametrize("seed", [0, 7, 123456789, 2**63 + 11])
def test_philox_raw_matches_numpy_philox(seed):
    # numpy.random.Philox is an independent Philox4x64-10 implementation;
    # raw block j == Philox(counter=(j+1,0,0,0), key=(seed,0)) (A6)
    ours = oracle.philox_raw(seed, 64)
    ref = np.random.Philox(key=seed).random_raw(256).astype(np.uint64)
    assert np.array_equal(ours, ref)


def test_philox_counter_offset_matches_numpy_advance():
    ours = oracle.philox_raw(5, 4, first_block=1000)
    g = np.random.Philox(key=5)
    g.advance(1000)
    assert np.array_equal(ours, g.random_raw(16).astype(np.uint64))


def test_gaussian_is_standard_normal():
    # mean and variance within 0.05 at 1e4 samples; plus a KS test
    z = oracle.gaussian_f32(0, 200_000).astype(np.float64)
    assert abs(z[:10_000].mean()) < 0.05 and abs(z[:10_000].var() - 1) < 0.05
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # pairs from one Box-Muller draw are uncorrelated
    assert abs(np.corrcoef(z[0::2], z[1::2])[0, 1]) < 0.01


def test_gaussian_deterministic_and_offsettable():
    a = oracle.gaussian_f32(3, 1001)
    assert np.array_equal(a, oracle.gaussian_f32(3, 1001))
    assert np.array_equal(a[37:901], oracle.gaussian_f32(3, 864, start=37))
    assert not np.array_equal(a, oracle.gaussian_f32(4, 1001))


def test_gaussian_box_muller_from_numpy_uniforms():
    # an independent route to the same numbers: numpy's raw Philox words,
    # mapped to uniforms and through Box-Muller in numpy
    raw = np.random.Philox(key=9).random_raw(400).astype(np.uint64).reshape(-1, 4)
    u = ((raw >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53
    r0, r1 = np.sqrt(-2 * np.log(u[:, 0])), np.sqrt(-2 * np.log(u[:, 2]))
    z = np.stack([r0 * np.cos(2 * np.pi * u[:, 1]), r0 * np.sin(2 * np.pi * u[:, 1]),
                  r1 * np.cos(2 * np.pi * u[:, 3]), r1 * np.sin(2 * np.pi * u[:, 3])], 1).reshape(-1)
    ours = oracle.gaussian_f32(9, 400)
    np.testing.assert_array_max_ulp(ours, z.astype(np.float32), maxulp=1)


# ---------------------------------------------------- degrees, Eq. 1, X
def test_degrees_golden():
    g = GOLD["degrees_triple"]
    dv, de = oracle.degrees(np.array(g["row_ptr"], np.int64), np.array(g["col_idx"], np.int32),
                            np.array(g["w"], np.float32))
    assert np.array_equal(dv, g["dv"]) and np.array_equal(de, g["de"])


@pytest.mark.parametrize("name", ["theta_pair", "theta_singleton"])
def test_theta_golden(name):
    g = GOLD[name]
    n = len(g["row_ptr"]) - 1
    th = oracle.theta_block(np.array(g["row_ptr"]), np.array(g["col_idx"]), np.array(g["w"]), n, 0)
    np.testing.assert_allclose(th, g["Theta"], rtol=0, atol=1e-15)


def test_isolated_vertex_and_empty_edge_are_errors():
    # zero vertex degree / empty hyperedge signal numerical errors
    with pytest.raises(oracle.OracleError) as e:
        oracle.degrees(np.array([0, 1, 1], np.int64), np.array([0], np.int32), np.ones(1, np.float32))
    assert e.value.status == oracle.ERR_NUMERICAL and "isolated vertex 1" in str(e.value)
    with pytest.raises(oracle.OracleError) as e:
        oracle.degrees(np.array([0, 1, 2], np.int64), np.array([0, 0], np.int32), np.ones(2, np.float32))
    assert e.value.status == oracle.ERR_NUMERICAL and "empty hyperedge 1" in str(e.value)


def test_full_theta_perron_symmetry_spectrum(cfg_inputs):
    # With b = N the single diagonal block is the whole Theta (Eq. 1).
    # Theta D^{1/2} 1 = D^{-1/2} H W De^{-1} (H^T 1) = D^{-1/2} H W 1 = D^{1/2} 1 (Perron vector),
    # Theta = K K^T with K = Dv^-1/2 H W^1/2 De^-1/2 is PSD with spectral radius 1.
    h = cfg_inputs(1)
    th = oracle.theta_block(h.row_ptr, h.col_idx, h.w, h.N, 0)
    dv, _ = oracle.degrees(h.row_ptr, h.col_idx, h.w)
    r = np.sqrt(dv)
    np.testing.assert_allclose(th @ r, r, rtol=1e-13)
    assert np.abs(th - th.T).max() <= 1e-16 and th.min() >= 0.0
    ev = np.linalg.eigvalsh(th)
    assert ev.min() > -1e-12 and abs(ev.max() - 1.0) < 1e-12


def test_theta_scale_invariance_in_w(cfg_inputs):
    # reading A9: a global scale of w cancels between W and D_v
    h = cfg_inputs(2)
    a = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 256, 3)
    b = oracle.theta_block(h.row_ptr, h.col_idx, (h.w * 4.0).astype(np.float32), 256, 3)
    np.testing.assert_allclose(a, b, rtol=1e-14, atol=1e-16)


def test_x_block_spectral_bracket(cfg_inputs):
    # eig(Theta_ii) in [0, 1] by interlacing => sigma(X_ii) in [mu/(1+mu), 1] (SURVEY pin P2)
    h = cfg_inputs(2)
    for mu in (1.0, 1.0 / 9.0):
        X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 256, 5, mu=mu)
        s = np.linalg.svd(X, compute_uv=False)
        assert s.max() <= 1 + 1e-12 and s.min() >= mu / (1 + mu) - 1e-12


def test_theta_block_matches_slice_of_full_theta():
    from synth.hypergraph import make_tiny
    h = make_tiny(64, 16, 4, 1, G=2, n_tag=5)
    full = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 64, 0)
    for i in range(4):
        blk = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 16, i)
        np.testing.assert_array_equal(blk, full[16 * i:16 * (i + 1), 16 * i:16 * (i + 1)])


# ---------------------------------------------------------------- QR
def test_qr_golden():
    g = GOLD["qr_3040"]
    Q, R = oracle.qr_householder(np.array(g["A"], float))
    np.testing.assert_allclose(Q[:, 0], g["q0"], atol=1e-15)
    assert abs(R[0, 0] - g["R00"]) < 1e-15


@pytest.mark.parametrize("m,n", [(50, 10), (128, 32), (7, 7), (300, 1)])
def test_qr_properties_and_span_vs_lapack(m, n):
    A = np.random.default_rng(m * n).standard_normal((m, n))
    Q, R = oracle.qr_householder(A)
    assert np.abs(Q.T @ Q - np.eye(n)).max() < 1e-13
    assert np.abs(Q @ R - A).max() < 1e-13 * max(1.0, np.abs(A).max())
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    Ql, Rl = np.linalg.qr(A)
    # the thin QR with diag(R) >= 0 is unique: matches LAPACK's up to column signs
    sg = np.sign(np.diag(Rl))
    np.testing.assert_allclose(Q, Ql * sg, atol=1e-12)
    np.testing.assert_allclose(R, Rl * sg[:, None], atol=1e-12)


# ---------------------------------------------------------------- SVD
@pytest.mark.parametrize("name", ["svd_diag321", "svd_perm"])
def test_svd_golden(name):
    g = GOLD[name]
    U, s, V = oracle.svd_square(np.array(g["A"], float))
    np.testing.assert_allclose(s, g["s"], atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 20, 64, 128])
def test_svd_square_vs_eigvalsh_and_lapack(n):
    M = np.random.default_rng(n).standard_normal((n, n))
    U, s, V = oracle.svd_square(M)
    # singular values = sqrt(eig(M^T M))
    ev = np.sort(np.sqrt(np.maximum(np.linalg.eigvalsh(M.T @ M), 0)))[::-1]
    np.testing.assert_allclose(s, ev, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(s, np.linalg.svd(M, compute_uv=False), rtol=1e-12, atol=1e-13)
    assert np.abs(U @ np.diag(s) @ V.T - M).max() < 1e-12
    assert np.abs(U.T @ U - np.eye(n)).max() < 1e-12 and np.abs(V.T @ V - np.eye(n)).max() < 1e-12
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0)


def test_svd_rank_deficient_and_degenerate():
    rng = np.random.default_rng(0)
    G = rng.standard_normal((10, 3))
    U, s, V = oracle.svd_square(G @ G.T)
    assert np.abs(s[3:]).max() < 1e-12
    np.testing.assert_allclose(s[:3], np.linalg.eigvalsh(G.T @ G)[::-1], rtol=1e-12)
    assert np.array_equal(oracle.svd_square(np.zeros((4, 4)))[1], np.zeros(4))
    # graded spectrum
    D = np.diag(10.0 ** -np.arange(8))
    Qa, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    Qb, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    _, s, _ = oracle.svd_square(Qa @ D @ Qb)
    np.testing.assert_allclose(s, np.diag(D), rtol=1e-8)


@pytest.mark.parametrize("k,m", [(1, 5), (8, 30), (32, 128), (64, 64)])
def test_svd_wide(k, m):
    B = np.random.default_rng(k + m).standard_normal((k, m))
    Ut, s, Vb = oracle.svd_wide(B)
    assert np.abs(Ut @ np.diag(s) @ Vb.T - B).max() < 1e-12
    np.testing.assert_allclose(s, np.linalg.svd(B, compute_uv=False), rtol=1e-12)
    assert np.abs(Vb.T @ Vb - np.eye(k)).max() < 1e-12
