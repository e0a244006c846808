"""Oracle pins for the rest of NEXT-3: oversampling l = k + p with rank-k
truncation ("l = k + pi") and the Eq. 10 power scheme Y = (X X^T)^pi X Omega
(PAPER.md:94-98), both in or_rsvd_block_ex / or_solve_mode.

  * Eq. 10 and Alg. 1 span the same subspace: the closed form M = X^T Z (Z^T X X^T Z)^-1 Z^T,
    Z = (X X^T)^q X Omega, holds for both (P7), and their outputs agree;
  * oversampling, exactly rank-k X: the truncated factorisation recovers X to 1e-10 and the
    surplus singular values are 0;
  * oversampling on Theta blocks (decaying spectrum): the truncated sigma_j never exceed the
    true singular values (interlacing, S^T X is a compression) and move closer to them as p grows;
  * p = 0 and scheme 0 are bitwise the plain path; invalid p rejected.
"""
import numpy as np
import pytest

import oracle
from synth.hypergraph import CONFIGS, make_input


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def closed_form_M(X, Om, q):
    Z = X @ Om
    for _ in range(q):
        Z = X @ (X.T @ Z)
    return X.T @ Z @ np.linalg.solve(Z.T @ X @ X.T @ Z, Z.T)


@pytest.mark.parametrize("q", [0, 1, 2])
def test_eq10_matches_closed_form_and_alg1(q):
    rng = np.random.default_rng(10 + q)
    b, k = 48, 8
    A = rng.standard_normal((b, b))
    X = np.eye(b) + 0.3 * (A + A.T) / np.sqrt(b)          # symmetric, well conditioned
    Om = rng.standard_normal((b, k))
    U1, s1, V1, _ = oracle.rsvd_block(X, Om, q)
    U2, s2, V2, _ = oracle.rsvd_block(X, Om, q, eq10=True)
    M = closed_form_M(X, Om, q)
    M2 = V2 @ np.diag(1 / s2) @ U2.T
    assert rel(M2, M) <= 1e-9
    np.testing.assert_allclose(s2, s1, rtol=1e-10)
    assert rel(U2 @ np.diag(s2) @ V2.T, U1 @ np.diag(s1) @ V1.T) <= 1e-10


def test_oversampling_exact_rank_k():
    rng = np.random.default_rng(11)
    b, k, p = 64, 5, 6
    G = rng.standard_normal((b, k))
    X = G @ G.T
    U, s, V, _ = oracle.rsvd_block(X, rng.standard_normal((b, k + p)), 1)
    assert rel(U[:, :k] @ np.diag(s[:k]) @ V[:, :k].T, X) <= 1e-10
    assert np.all(s[k:] <= 1e-10 * s[0])


def test_oversampling_sigma_interlacing_and_improvement():
    c = CONFIGS[1]
    h = make_input(c)
    Th = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, 0, mu=0.0)
    true = np.linalg.svd(Th, compute_uv=False)
    k = 16
    errs = []
    for p in (0, 4, 16):
        r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=k, q=0, seed=0, blocks=[0],
                         woodbury=True, p=p)
        s = r.sigma[0]
        assert np.all(s <= true[:k] * (1 + 1e-12))
        errs.append(float(np.sum(true[:k] - s)))
    assert errs[0] > errs[1] > errs[2]


def test_p0_scheme0_is_plain_path_and_invalid_p():
    c = CONFIGS[1]
    h = make_input(c)
    a = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, blocks=[1])
    b_ = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, blocks=[1], p=0)
    assert np.array_equal(a.F, b_.F) and np.array_equal(a.sigma, b_.sigma)
    with pytest.raises(oracle.OracleError):
        oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, p=c.b)
