"""GPU: the nested tessellation (NEXT-1, hg_solve_nested; PAPER.md:155-156 with Eq. 12) against the FP64
oracle (oracle.solve_nested, pinned in tests/test_oracle_nested.py).  Tolerance: F <= 2e-5 (north_star)."""
import numpy as np
import pytest
import torch

import oracle
from synth.hypergraph import CONFIGS, make_input, make_tiny

pytestmark = pytest.mark.gpu
F_TOL = 2e-5


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _dev(h):
    hg = hgm()
    return (hg.incidence_to_device(h.row_ptr, h.col_idx, h.E), torch.from_numpy(h.w).cuda(),
            torch.from_numpy(h.Y).cuda())


@pytest.mark.parametrize("levels", [1, 2])
def test_nested_config1_matches_oracle(levels):
    hg = hgm()
    c = CONFIGS[1]
    h = make_input(c)
    H, w, Y = _dev(h)
    F, st = hg.solve_nested(H, w, Y, mu=c.mu, b=c.b, levels=levels, k=c.k, q=c.q, seed=c.seed)
    assert int(st.item()) == 0
    r, _, _ = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, levels=levels, k=c.k, q=c.q,
                                  seed=c.seed)
    assert rel(F.double().cpu().numpy(), r) <= F_TOL


def test_nested_level1_equals_schur():
    hg = hgm()
    c = CONFIGS[1]
    h = make_input(c)
    H, w, Y = _dev(h)
    F1, st = hg.solve_nested(H, w, Y, mu=c.mu, b=c.b, levels=1, k=c.k, q=c.q, seed=c.seed)
    F2, st2 = hg.solve_schur(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    assert int(st.item()) == 0 and int(st2.item()) == 0
    assert float((F1 - F2).norm() / F2.norm()) <= 1e-5


@pytest.mark.parametrize("levels,b", [(2, 8), (3, 8)])
def test_nested_full_rank_is_the_superblock_solve(levels, b):
    hg = hgm()
    h = make_tiny(64, 16, 16, 1)
    H, w, Y = _dev(h)
    m = b << levels
    F, st = hg.solve_nested(H, w, Y, mu=1.0, b=b, levels=levels, k=b, q=1, seed=0)
    assert int(st.item()) == 0
    Fg = F.double().cpu().numpy()
    for s in range(64 // m):
        X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, m, s, mu=1.0)
        lu = 0.5 * np.linalg.solve(X, h.Y[s * m:(s + 1) * m].astype(np.float64))
        assert rel(Fg[s * m:(s + 1) * m], lu) <= F_TOL


def test_nested_config2_two_levels_sampled():
    """configs[1] (N=4096, b=256, k=64): super-blocks of 1024 (two levels), oracle on super-blocks 0 and 3."""
    hg = hgm()
    c = CONFIGS[2]
    h = make_input(c)
    H, w, Y = _dev(h)
    F, st = hg.solve_nested(H, w, Y, mu=c.mu, b=c.b, levels=2, k=c.k, q=c.q, seed=c.seed)
    assert int(st.item()) == 0
    r, sel, _ = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, levels=2, k=c.k, q=c.q,
                                    seed=c.seed, superblocks=[0, 3])
    m = c.b << 2
    Fg = F.double().cpu().numpy()
    for i, s in enumerate(sel):
        assert rel(Fg[s * m:(s + 1) * m], r[i * m:(i + 1) * m]) <= F_TOL


def test_tessellate_schedule():
    hg = hgm()
    assert hg.tessellate(1024, 50) == (32, 5)
    assert hg.tessellate(1024, 500) == (256, 2)
    assert hg.tessellate(100, 100) == (100, 0)
    assert hg.tessellate(200, 50) == (50, 2)
