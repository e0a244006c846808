"""Oracle pins for reading R2: Alg. 1 on the PSD low-rank part
Theta_ii and the Woodbury inverse of X_ii = I - Theta_ii/(1+theta).

  * the Woodbury identity itself: (I - U S U^T/(1+mu)) applied to or_apply_woodbury's output
    returns c Y for any orthonormal U and 0 <= s < 1+mu (closed form);
  * exactly rank-k PSD Theta (G G^T): the whole R2 chain (or_rsvd_block + or_apply_woodbury)
    equals the dense LU solve c X^-1 Y (numpy.linalg.solve);
  * k = b on the configs' own Theta blocks: R2 is the exact block inverse (LU);
  * configs[0] at k/b = 1/4: R2 is within 5e-2 of the exact block solve (App. A measured
    2.7e-2) while R1 (the binding reading) is ~0.9 away -- the reason NEXT-3 exists;
  * error falls monotonically in k.
"""
import numpy as np
import pytest

import oracle
from synth.hypergraph import CONFIGS, make_input, make_tiny


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("mu", [1.0, 1.0 / 9.0])
def test_woodbury_identity(mu):
    rng = np.random.default_rng(5)
    m, k, T = 40, 7, 3
    U, _ = np.linalg.qr(rng.standard_normal((m, k)))
    s = np.sort(rng.uniform(0.0, 1.0, k))[::-1]
    Y = rng.standard_normal((m, T))
    F = oracle.apply_woodbury(U, s, Y, mu)
    X = np.eye(m) - U @ np.diag(s) @ U.T / (1 + mu)
    assert rel(X @ F, mu / (1 + mu) * Y) <= 1e-13


def test_exact_rank_k_theta_gives_exact_inverse():
    rng = np.random.default_rng(6)
    b, k, mu, T = 64, 6, 1.0, 5
    G = rng.standard_normal((b, k))
    Th = G @ G.T
    Th *= 0.9 / np.linalg.eigvalsh(Th)[-1]     # PSD, spectrum in [0, 0.9] like Theta (pin P2)
    Y = rng.standard_normal((b, T))
    U, s, V, _ = oracle.rsvd_block(Th, rng.standard_normal((b, k)), 1)
    F = oracle.apply_woodbury(U, s, Y, mu)
    X = np.eye(b) - Th / (1 + mu)
    assert rel(F, mu / (1 + mu) * np.linalg.solve(X, Y)) <= 1e-10


def block_exact(h, c, mu):
    ex = np.zeros((c.N, h.Y.shape[1]))
    for i in range(c.nb):
        X = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, i, mu=mu)
        ex[i * c.b:(i + 1) * c.b] = mu / (1 + mu) * np.linalg.solve(X, h.Y[i * c.b:(i + 1) * c.b].astype(float))
    return ex


def test_k_equals_b_is_exact_block_inverse():
    h = make_tiny(48, 16, 16, 1)
    c = h.cfg
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=1.0, b=16, k=16, q=1, seed=0, woodbury=True)
    assert rel(r.F, block_exact(h, c.with_(N=48, b=16), 1.0)) <= 1e-9


def test_r2_accuracy_against_exact_block_solve_config1():
    c = CONFIGS[1]
    h = make_input(c)
    ex = block_exact(h, c, c.mu)
    errs = {}
    for k in (8, 16, 32, 64):
        r2 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=k, q=c.q, seed=0, woodbury=True)
        errs[k] = rel(r2.F, ex)
        # theta_ii is PSD with spectrum in [0, 1] (pin P2): sigma in [0, 1]
        assert np.all(r2.sigma >= -1e-12) and np.all(r2.sigma <= 1 + 1e-12)
    r1 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    assert errs[32] <= 5e-2 and rel(r1.F, ex) >= 0.5
    assert errs[8] > errs[16] > errs[32] > errs[64]
