"""GPU parity for NEXT-1: one level of the 2x2 Schur-complement inverse
(Eqs. 11-14) over pairs of adjacent diagonal blocks with reading-R2 inverses,
through the C ABI (hg_solve_schur), against the FP64 oracle (or_solve_schur).  Tolerance:
north_star's F tolerance, 2e-5 relative Frobenius per super-block."""
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


def run(h, mu, b, k, q, superblocks=None):
    hg = hgm()
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    F, st = hg.solve_schur(H, torch.from_numpy(h.w).cuda(), torch.from_numpy(h.Y).cuda(), mu=mu, b=b, k=k, q=q,
                           seed=0)
    assert int(st.item()) == 0
    Fo, sel, _ = oracle.solve_schur(h.row_ptr, h.col_idx, h.w, h.Y, mu=mu, b=b, k=k, q=q, seed=0,
                                    superblocks=superblocks)
    Fg = F.double().cpu().numpy()
    errs = []
    for i, s in enumerate(sel):
        errs.append(rel(Fg[s * 2 * b:(s + 1) * 2 * b], Fo[i * 2 * b:(i + 1) * 2 * b]))
    return Fg, max(errs)


@pytest.mark.parametrize("cfg", [1, 2])
def test_schur_parity(cfg):
    c = CONFIGS[cfg]
    _, err = run(make_input(c), c.mu, c.b, c.k, c.q)
    assert err <= F_TOL, err


def test_schur_parity_config4_sampled():
    c = CONFIGS[4]
    _, err = run(make_input(c), c.mu, c.b, c.k, c.q, superblocks=[0, c.nb // 2 - 1])
    assert err <= F_TOL, err


def test_schur_k_equals_b_is_exact_superblock_solve():
    h = make_tiny(64, 16, 16, 1, G=2)
    Fg, err = run(h, 1.0, 16, 16, 1)
    assert err <= F_TOL
    for s in range(2):
        Xs = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 32, s, mu=1.0)
        ex = 0.5 * np.linalg.solve(Xs, h.Y[s * 32:(s + 1) * 32].astype(float))
        assert rel(Fg[s * 32:(s + 1) * 32], ex) <= F_TOL


def test_schur_rejects_odd_block_count():
    hg = hgm()
    c = CONFIGS[1]
    h = make_input(c)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    with pytest.raises(hg.HGError) as e:
        hg.solve_schur(H, torch.from_numpy(h.w).cuda(), torch.from_numpy(h.Y).cuda(), mu=1.0, b=512, k=32, q=1,
                       seed=0)
    assert e.value.status == hg.HG_ERR_INVALID
