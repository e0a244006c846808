"""Oracle pins for the paper's second approach, CG on Eq. 5 (Eqs. 16-20).

The oracle (oracle/hg_oracle.c: or_apply_X, or_cg_solve) is pinned against what
the paper and the mathematics fix, not against itself:
  * X p matrix-free through H equals the assembled X of Eq. 1 (the separately
    pinned or_theta_block with b = N) times p, and the Perron closed form
    X Dv^1/2 1 = c Dv^1/2 1 (Theta has eigenvalue 1 on Dv^1/2 1);
  * CG converges to the dense LU solve of Eq. 5 (numpy.linalg.solve);
  * iterate i is the X-norm minimiser over the Krylov space K_i(X, r_0) --
    f_i = K (K^T X K)^-1 K^T c y, a closed form independent of the
    alpha/beta recurrences (a wrong alpha, beta or sign breaks it at i >= 2);
  * scipy.sparse.linalg.cg with x0 = 0 gives the same iterates (library);
  * residuals are mutually orthogonal; finite termination in <= N steps;
  * a right-hand side on the Perron vector converges in one iteration;
  * stopping rule (reading C2), zero columns, invalid arguments.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle
from synth.hypergraph import CONFIGS, make_input, make_tiny


@pytest.fixture(scope="module")
def cfg1():
    return make_input(CONFIGS[1])


def full_X(h, mu):
    N = len(h.row_ptr) - 1
    return oracle.theta_block(h.row_ptr, h.col_idx, h.w, N, 0, mu=mu)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_apply_X_matches_assembled_X(cfg1):
    h, mu = cfg1, 1.0
    X = full_X(h, mu)
    rng = np.random.default_rng(3)
    for _ in range(3):
        p = rng.standard_normal(len(h.row_ptr) - 1)
        assert rel(oracle.apply_X(h.row_ptr, h.col_idx, h.w, p, mu=mu), X @ p) <= 1e-14


@pytest.mark.parametrize("mu", [1.0, 1.0 / 9.0])
def test_apply_X_perron_closed_form(cfg1, mu):
    h = cfg1
    dv, _ = oracle.degrees(h.row_ptr, h.col_idx, h.w)
    s = np.sqrt(dv)
    c = mu / (1.0 + mu)
    assert rel(oracle.apply_X(h.row_ptr, h.col_idx, h.w, s, mu=mu), c * s) <= 1e-14


def test_cg_converges_to_lu_solve(cfg1):
    h, mu = cfg1, 1.0
    c = mu / (1 + mu)
    r = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=mu, max_iter=200, tol=1e-13)
    F_lu = np.linalg.solve(full_X(h, mu), c * h.Y.astype(np.float64))
    assert rel(r.F, F_lu) <= 1e-11
    assert np.all(r.rel_res <= 1e-13)
    # cond(X) <= 2 (sigma(X) in [theta/(1+theta), 1]): few iterations
    assert r.iters.max() <= 20


def test_cg_iterate_is_krylov_minimiser(cfg1):
    h, mu = cfg1, 1.0
    c = mu / (1 + mu)
    X = full_X(h, mu)
    y = h.Y[:, :3]
    for i in range(1, 7):
        r = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y, mu=mu, max_iter=i, tol=0.0)
        assert np.all(r.iters == i)
        for col in range(y.shape[1]):
            b = c * y[:, col].astype(np.float64)
            K = [b]
            for _ in range(i - 1):
                K.append(X @ K[-1])
            Q, _ = np.linalg.qr(np.stack(K, 1))
            f = Q @ np.linalg.solve(Q.T @ X @ Q, Q.T @ b)
            assert rel(r.F[:, col], f) <= 1e-10, (i, col)


def test_cg_matches_scipy_iterates(cfg1):
    h, mu = cfg1, 1.0
    c = mu / (1 + mu)
    X = full_X(h, mu)
    y = h.Y[:, 5:7]
    for i in (1, 2, 4, 8):
        r = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y, mu=mu, max_iter=i, tol=0.0)
        for col in range(y.shape[1]):
            b = c * y[:, col].astype(np.float64)
            f, _ = spla.cg(X, b, x0=np.zeros_like(b), rtol=0.0, atol=0.0, maxiter=i)
            assert rel(r.F[:, col], f) <= 1e-12, (i, col)


def test_cg_residuals_orthogonal(cfg1):
    h, mu = cfg1, 1.0
    c = mu / (1 + mu)
    X = full_X(h, mu)
    y = h.Y[:, :1]
    b = c * y[:, 0].astype(np.float64)
    R = [b]
    for i in range(1, 6):
        f = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y, mu=mu, max_iter=i, tol=0.0).F[:, 0]
        R.append(b - X @ f)
    for i in range(len(R)):
        for j in range(i):
            assert abs(R[i] @ R[j]) <= 1e-10 * np.linalg.norm(R[i]) * np.linalg.norm(R[j]) + 1e-300


def test_cg_finite_termination_tiny():
    h = make_tiny(8, 4, 2, 1, K=2, n_tag=3)
    mu = 1.0
    c = mu / (1 + mu)
    r = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=mu, max_iter=8, tol=0.0)
    F_lu = np.linalg.solve(full_X(h, mu), c * h.Y.astype(np.float64))
    assert rel(r.F, F_lu) <= 1e-10


def test_cg_perron_rhs_one_iteration(cfg1):
    # y = Dv^1/2 1 is an eigenvector: X y = c y, so the solution of X f = c y is f = y,
    # reached by the first step (r_0 = c y is an eigenvector of X).  y is rounded to
    # fp32 (the API's RHS type), so it is an eigenvector to ~1e-8 relative.
    h, mu = cfg1, 1.0
    dv, _ = oracle.degrees(h.row_ptr, h.col_idx, h.w)
    y = np.sqrt(dv).astype(np.float32)[:, None]
    r = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y, mu=mu, max_iter=50, tol=1e-6)
    assert r.iters[0] == 1 and r.rel_res[0] <= 1e-7
    assert rel(r.F[:, 0], y[:, 0].astype(np.float64)) <= 1e-7


def test_cg_stopping_rule_and_degenerate_columns(cfg1):
    h, mu = cfg1, 1.0
    y = np.array(h.Y[:, :4])
    y[:, 2] = 0.0                       # zero column: no iteration, f = 0
    r = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y, mu=mu, max_iter=100, tol=1e-6)
    assert r.iters[2] == 0 and np.all(r.F[:, 2] == 0.0) and r.rel_res[2] == 0.0
    for col in (0, 1, 3):               # minimal i with ||r_i|| <= tol ||r_0||
        i = int(r.iters[col])
        assert r.rel_res[col] <= 1e-6
        prev = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y[:, col:col + 1], mu=mu, max_iter=i - 1, tol=1e-6)
        assert prev.iters[0] == i - 1 and prev.rel_res[0] > 1e-6
    r0 = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, y, mu=mu, max_iter=0, tol=0.0)
    assert np.all(r0.F == 0.0) and np.all(r0.iters == 0)


def test_cg_invalid_arguments(cfg1):
    h = cfg1
    for kw in (dict(mu=0.0, max_iter=5, tol=0.0), dict(mu=1.0, max_iter=-1, tol=0.0),
               dict(mu=1.0, max_iter=5, tol=-1.0)):
        with pytest.raises(oracle.OracleError) as e:
            oracle.cg_solve(h.row_ptr, h.col_idx, h.w, h.Y, **kw)
        assert e.value.status == oracle.ERR_INVALID
