"""Oracle pins for NEXT-1: one level of the 2x2 Schur-complement inverse,
Eqs. 11-14, over super-blocks of two adjacent diagonal blocks, with
X11^-1, X22^-1, Z1^-1, Z2^-1 by randomized SVD in reading R2.

  * the off-diagonal Eq. 1 block equals the slice of the full Theta (the separately pinned
    or_theta_block with b = N) and is the transpose of its mirror;
  * with k = b every inverse is exact, so the result is the dense LU solve of the 2b x 2b
    super-block system c X_s^-1 Y_s (Eq. 12 is an identity) -- to 1e-12;
  * with no hyperedge shared across the two blocks (Theta12 = 0) it reduces to the
    block-diagonal reading-R2 solve (Z = X), bitwise in structure and to 1e-12 in value;
  * at k < b it stays within R2's accuracy of the exact super-block solve and is closer
    to the full solve than the block-diagonal solve (the coupling the method adds).
"""
import numpy as np
import pytest

import oracle
from synth.hypergraph import CONFIGS, make_input, make_tiny


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def cfg1():
    return make_input(CONFIGS[1])


def test_offblock_is_slice_of_full_theta(cfg1):
    h, b = cfg1, 128
    N = len(h.row_ptr) - 1
    T = oracle.theta_block(h.row_ptr, h.col_idx, h.w, N, 0, mu=0.0)
    for (i, j) in [(0, 1), (2, 3), (1, 3)]:
        O = oracle.theta_offblock(h.row_ptr, h.col_idx, h.w, b, i, j)
        assert np.abs(O - T[i * b:(i + 1) * b, j * b:(j + 1) * b]).max() <= 1e-15
        assert np.abs(O - oracle.theta_offblock(h.row_ptr, h.col_idx, h.w, b, j, i).T).max() <= 1e-15


def superblock_exact(h, b, mu):
    N = len(h.row_ptr) - 1
    out = np.zeros((N, h.Y.shape[1]))
    for s in range(N // (2 * b)):
        Xs = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 2 * b, s, mu=mu)
        out[s * 2 * b:(s + 1) * 2 * b] = mu / (1 + mu) * np.linalg.solve(Xs, h.Y[s * 2 * b:(s + 1) * 2 * b].astype(float))
    return out


@pytest.mark.parametrize("N,b,q", [(64, 16, 1), (96, 24, 2)])
def test_k_equals_b_is_exact_superblock_solve(N, b, q):
    h = make_tiny(N, b, b, q, G=2)
    F, _, _ = oracle.solve_schur(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=b, k=b, q=q, seed=0)
    assert rel(F, superblock_exact(h, b, 1.0)) <= 1e-12


def test_no_cross_edges_reduces_to_block_diagonal_r2():
    # two disjoint 8-vertex hypergraphs side by side: Theta12 = 0, so Z1 = X11, Z2 = X22
    rng = np.random.default_rng(3)
    rows = []
    for half in range(2):
        for v in range(8):
            es = {half * 4 + int(rng.integers(0, 4)), half * 4 + (v % 4)}
            rows.append(sorted(es))
    rp = np.array([0] + list(np.cumsum([len(r) for r in rows])), np.int64)
    ci = np.array([e for r in rows for e in r], np.int32)
    w = rng.uniform(0.5, 1.5, 8).astype(np.float32)
    Y = rng.integers(0, 2, (16, 4)).astype(np.float32)
    F, _, _ = oracle.solve_schur(rp, ci, w, Y, mu=1.0, b=8, k=4, q=1, seed=0)
    r2 = oracle.solve(rp, ci, w, Y, mu=1.0, b=8, k=4, q=1, seed=0, woodbury=True)
    assert rel(F, r2.F) <= 1e-12


def test_accuracy_config1(cfg1):
    h, c = cfg1, CONFIGS[1]
    F, _, _ = oracle.solve_schur(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    sb = superblock_exact(h, c.b, c.mu)
    assert rel(F, sb) <= 5e-2
    N = len(h.row_ptr) - 1
    X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, N, 0, mu=c.mu)
    full = c.mu / (1 + c.mu) * np.linalg.solve(X, h.Y.astype(float))
    r2 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, woodbury=True).F
    assert rel(F, full) < rel(r2, full)
