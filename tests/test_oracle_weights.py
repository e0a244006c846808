"""Oracle pins for NEXT-4, the hyperedge-weight update with f fixed
(PAPER.md:46-58): objective P(w) = sum_t f_t^T L f_t + kappa ||w||^2, the frozen-degree
gradient (SPEC.md gradient_frozen) and the simplex-constrained steepest-descent step
(SPEC.md steepest_descent_step; readings N1-N2).

  * SPEC.md worked examples for all three operations (tests/golden/spec_examples.json is
    not needed: the values are restated here with their SPEC lines);
  * the gradient equals central finite differences of the frozen-degree objective, built
    here densely from H with numpy (a different computation from the oracle's edge loops);
  * the step keeps 1^T w = 1 and w >= 0, clamped weights stay 0, a constant gradient is
    annihilated, and a huge kappa drives w to the uniform point (the minimum-norm simplex point).
"""
import numpy as np
import pytest

import oracle
from synth.hypergraph import make_tiny


def csr(edges_of_vertex):
    rp = [0]
    ci = []
    for es in edges_of_vertex:
        ci += sorted(es)
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int32)


def test_objective_spec_examples():
    # SPEC.md:387 objective: f = 0 -> kappa ||w||^2
    rp, ci = csr([[0, 1], [0, 2], [0, 3]])          # 3 vertices, edge 0 holds all, edges 1-3
    w = np.array([0.4, 0.3, 0.2, 0.1], np.float32)
    assert oracle.weight_objective(rp, ci, w, np.zeros(3), kappa=2.0) == pytest.approx(2.0 * np.sum(w.astype(float) ** 2))
    # SPEC.md:388 2-vertex / 1-edge toy, w = (1), f = (1, -1), kappa = 0 -> 2
    rp2, ci2 = csr([[0], [0]])
    assert oracle.weight_objective(rp2, ci2, np.ones(1, np.float32), np.array([1.0, -1.0]), kappa=0.0) == pytest.approx(2.0)
    # SPEC.md:389 n = 4, w = (1, 0, 0, 0), kappa = 1, f = 0 -> 1 (every vertex lies on edge 0)
    w4 = np.array([1, 0, 0, 0], np.float32)
    assert oracle.weight_objective(rp, ci, w4, np.zeros(3), kappa=1.0) == pytest.approx(1.0)


def test_gradient_spec_examples():
    # SPEC.md:396 (f = 0 -> 2 kappa w) and SPEC.md:397 (toy, f = (1, 1), w = (1), kappa = 0 -> -2)
    rp, ci = csr([[0, 1], [0, 2], [0, 3]])
    w = np.array([0.4, 0.3, 0.2, 0.1], np.float32)
    np.testing.assert_allclose(oracle.weight_gradient(rp, ci, w, np.zeros(3), kappa=1.5), 3.0 * w.astype(float))
    rp2, ci2 = csr([[0], [0]])
    g = oracle.weight_gradient(rp2, ci2, np.ones(1, np.float32), np.array([1.0, 1.0]), kappa=0.0)
    assert g[0] == pytest.approx(-2.0)


def frozen_objective_dense(rp, ci, w0, w, F, kappa):
    """P~(w) with D_v, D_e frozen at w0: sum_t f^T (I - Dv0^-1/2 H W De^-1 H^T Dv0^-1/2) f + kappa ||w||^2."""
    N, E = len(rp) - 1, len(w)
    H = np.zeros((N, E))
    for v in range(N):
        H[v, ci[rp[v]:rp[v + 1]]] = 1.0
    dv0 = H @ w0
    de = H.sum(0)
    K = np.diag(dv0 ** -0.5) @ H
    A = K @ np.diag(w / de) @ K.T
    return float(np.sum(F * F) - np.sum(F * (A @ F)) + kappa * np.sum(w * w))


def test_gradient_matches_finite_differences():
    h = make_tiny(8, 4, 2, 1, K=2, n_tag=3)
    rng = np.random.default_rng(4)
    w0 = h.w.astype(np.float64)
    F = rng.standard_normal((8, 3))
    kappa = 0.7
    g = oracle.weight_gradient(h.row_ptr, h.col_idx, h.w, F, kappa=kappa)
    step = 1e-6
    for e in range(len(w0)):
        wp, wm = w0.copy(), w0.copy()
        wp[e] += step
        wm[e] -= step
        fd = (frozen_objective_dense(h.row_ptr, h.col_idx, w0, wp, F, kappa) -
              frozen_objective_dense(h.row_ptr, h.col_idx, w0, wm, F, kappa)) / (2 * step)
        assert fd == pytest.approx(g[e], rel=1e-5, abs=1e-8)


def test_step_spec_examples():
    # SPEC.md:406, 407 (n = 2 cases), SPEC.md:405 (constant gradient annihilated)
    w, a = oracle.weight_step([0.5, 0.5], [0, 0], [1.0, -1.0], 0.1)
    np.testing.assert_allclose(w, [0.4, 0.6], atol=1e-15)
    w, a = oracle.weight_step([0.05, 0.95], [0, 0], [1.0, -1.0], 0.1)
    np.testing.assert_allclose(w, [0.0, 1.0], atol=1e-15)
    assert list(a) == [1, 0]
    w, a = oracle.weight_step([0.2, 0.3, 0.5], [0, 0, 0], [2.0, 2.0, 2.0], 0.3)   # constant gradient
    np.testing.assert_allclose(w, [0.2, 0.3, 0.5], atol=1e-15)
    with pytest.raises(oracle.OracleError):
        oracle.weight_step([0.0, 1.0], [1, 1], [1.0, 1.0], 0.1)


def test_step_invariants_and_large_kappa_uniform():
    rng = np.random.default_rng(9)
    E = 50
    w = rng.dirichlet(np.ones(E))
    a = np.zeros(E, np.int32)
    for _ in range(20):
        w, a = oracle.weight_step(w, a, rng.standard_normal(E), 0.05)
        assert abs(w.sum() - 1.0) <= 1e-12 and w.min() >= 0.0
        assert np.all(w[a == 1] == 0.0)
    # SPEC.md:414 kappa -> infinity: gradient 2 kappa w, step 0.25/kappa halves the distance to uniform
    h = make_tiny(8, 4, 2, 1, K=2, n_tag=3)
    E = len(h.w)
    w = h.w.astype(np.float64) / h.w.sum()
    a = np.zeros(E, np.int32)
    kappa = 1e6
    F = np.random.default_rng(1).standard_normal((8, 2))
    for _ in range(60):
        g = oracle.weight_gradient(h.row_ptr, h.col_idx, w.astype(np.float32), F, kappa=kappa)
        w, a = oracle.weight_step(w, a, g, 0.25 / kappa)
    np.testing.assert_allclose(w, 1.0 / E, atol=1e-3)


def test_objective_gradient_identity():
    # P is linear in w at fixed degrees apart from the penalty, so at the gradient's own w:
    # P(w) = ||F||^2 + w^T grad(w) - kappa ||w||^2  (the identity hg_weight_objective uses)
    h = make_tiny(8, 4, 2, 1, K=2, n_tag=3)
    rng = np.random.default_rng(12)
    F = rng.standard_normal((8, 3))
    for kappa in (0.0, 0.7):
        g = oracle.weight_gradient(h.row_ptr, h.col_idx, h.w, F, kappa=kappa)
        w = h.w.astype(np.float64)
        P = oracle.weight_objective(h.row_ptr, h.col_idx, h.w, F, kappa=kappa)
        assert P == pytest.approx(np.sum(F * F) + w @ g - kappa * w @ w, rel=1e-12)
