"""Oracle pins for the nested tessellation (NEXT-1; PAPER.md:155-156 with Eq. 12 of PAPER.md:139-150),
oracle.solve_nested: Eq. 12 applied recursively inside super-blocks of m = 2^L b vertices.

  * L = 1 is exactly the one-level Schur solve (oracle.solve_schur, itself pinned in
    test_oracle_schur.py) -- only the order of the final products differs;
  * k = b makes every leaf and every Schur-complement inverse exact (rank = dimension at every
    level, k_l = k 2^(l-1)), so Eq. 12 is an identity and F_s = c X_s^-1 Y_s, the dense LU solve of
    the m x m super-block (Eq. 3), at L = 2 and 3;
  * the same at two values of the regulariser mu;
  * invalid arguments are rejected.
"""
import numpy as np
import pytest

import oracle
from synth.hypergraph import make_tiny


@pytest.fixture(scope="module")
def tiny():
    return make_tiny(64, 16, 16, 1)


def test_one_level_equals_schur(tiny):
    h = tiny
    for k in (4, 8, 16):
        Fs, _, _ = oracle.solve_schur(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=16, k=k, q=1, seed=0)
        Fn, _, _ = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=16, levels=1, k=k, q=1, seed=0)
        assert np.abs(Fs - Fn).max() <= 1e-12 * np.abs(Fs).max()


@pytest.mark.parametrize("levels,b", [(2, 8), (3, 8), (2, 16)])
@pytest.mark.parametrize("mu", [1.0, 1.0 / 9.0])
def test_full_rank_equals_superblock_lu(tiny, levels, b, mu):
    h = tiny
    m = b << levels
    c = mu / (1 + mu)
    Fn, sel, _ = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=mu, b=b, levels=levels, k=b, q=1, seed=3)
    for i, s in enumerate(sel):
        X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, m, s, mu=mu)
        lu = c * np.linalg.solve(X, h.Y[s * m:(s + 1) * m].astype(np.float64))
        got = Fn[i * m:(i + 1) * m]
        assert np.linalg.norm(got - lu) <= 1e-10 * np.linalg.norm(lu)


def test_superblock_selection_is_consistent(tiny):
    h = tiny
    Fa, sel, _ = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=8, levels=2, k=4, q=2, seed=0)
    Fb, _, _ = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=8, levels=2, k=4, q=2, seed=0,
                                   superblocks=[1])
    assert sel == [0, 1] and np.array_equal(Fa[32:64], Fb)


@pytest.mark.parametrize("kw", [dict(levels=0), dict(levels=3, b=16), dict(k=0), dict(k=20)])
def test_invalid_arguments(tiny, kw):
    h = tiny
    args = dict(mu=1.0, b=8, levels=2, k=4, q=1, seed=0)
    args.update(kw)
    with pytest.raises(oracle.OracleError):
        oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, **args)
