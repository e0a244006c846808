"""GPU: the fused Sigma^-1 scale + apply kernel (apply.cu; Eq. 3 with Eq. 15)
against the FP64 oracle's or_apply_block, through hg_block_apply_inverse.

The factors here are NOT this library's rSVD output: random orthonormal U, V (FP64 QR), a geometric
sigma, and variants that leave the unit bound (scaled U / V, large and tiny Y) so the measured-maximum
exponents, the per-CTA exponent of Z, every KP template (k = 32, 64, 128, 256), a ragged last column
tile, a ragged T (padded copies) and several row tiles are all exercised.  k % 32 != 0 and k > 256 take
the two-GEMM path and must meet the same tolerance.  Tolerance: north_star's F <= 2e-5 relative.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

F_TOL = 2e-5


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def factors(nb, b, k, seed):
    rng = np.random.default_rng(seed)
    U = np.stack([np.linalg.qr(rng.standard_normal((b, k)))[0] for _ in range(nb)])   # [nb][b][k]
    V = np.stack([np.linalg.qr(rng.standard_normal((b, k)))[0] for _ in range(nb)])
    sigma = np.stack([np.geomspace(1.0, 0.05, k) * (1.0 + 0.1 * i) for i in range(nb)])
    return U, sigma, V


def run_case(nb, b, k, T, seed, u_scale=1.0, v_scale=1.0, y_scale=1.0, y_kind="normal"):
    hg = hgm()
    U, sigma, V = factors(nb, b, k, seed)
    U = U * u_scale
    V = V * v_scale
    rng = np.random.default_rng(seed + 1)
    if y_kind == "labels":   # the paper's tag-label matrix: 0 / 1 entries
        Y = (rng.random((nb * b, T)) < 0.1).astype(np.float64)
    else:
        Y = rng.standard_normal((nb * b, T)) * y_scale
    Ut = torch.from_numpy(np.ascontiguousarray(U.transpose(0, 2, 1)).astype(np.float32)).cuda()
    Vt = torch.from_numpy(np.ascontiguousarray(V.transpose(0, 2, 1)).astype(np.float32)).cuda()
    sg = torch.from_numpy(sigma.astype(np.float32)).cuda()
    Yd = torch.from_numpy(Y.astype(np.float32)).cuda()
    scale = 0.5
    F, st = hg.block_apply_inverse(Ut, sg, Vt, Yd, scale)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    Fg = F.double().cpu().numpy()
    # the oracle on exactly the fp32 inputs the GPU saw
    Uf, Vf = Ut.double().cpu().numpy(), Vt.double().cpu().numpy()
    sf, Yf = sg.double().cpu().numpy(), Yd.double().cpu().numpy()
    for i in range(nb):
        ref = oracle.apply_block(Uf[i].T, sf[i], Vf[i].T, Yf[i * b:(i + 1) * b], scale)
        assert rel(Fg[i * b:(i + 1) * b], ref) <= F_TOL, (i, rel(Fg[i * b:(i + 1) * b], ref))


@pytest.mark.parametrize("b,k,T", [(128, 32, 20), (256, 64, 100), (512, 128, 500), (1024, 256, 1000),
                                   (384, 96, 132), (256, 256, 260)])
def test_fused_apply_matches_oracle(b, k, T):
    run_case(3, b, k, T, seed=11)


@pytest.mark.parametrize("T", [7, 1, 129])
def test_fused_apply_ragged_T(T):
    run_case(2, 256, 64, T, seed=5)


def test_fused_apply_label_matrix():
    run_case(2, 512, 128, 256, seed=3, y_kind="labels")


@pytest.mark.parametrize("u_scale,v_scale,y_scale", [(5.0, 0.01, 1.0), (1.0, 1.0, 3e4), (0.02, 300.0, 1e-6),
                                                     (1.0, 1.0, 1e-30)])
def test_fused_apply_exponents_follow_the_data(u_scale, v_scale, y_scale):
    """Factors and right-hand sides far from the unit bound: the measured maxima set the fp16 prescale
    (scaled U / V model caller-provided factors; F scales with the product, the relative error must not)."""
    run_case(2, 256, 64, 96, seed=7, u_scale=u_scale, v_scale=v_scale, y_scale=y_scale)


@pytest.mark.parametrize("b,k", [(256, 40), (1024, 512), (100, 20)])
def test_unfused_fallback_shapes(b, k):
    """k % 32 != 0, k > 256, b % 32 != 0: the two-GEMM path, same tolerance."""
    run_case(2, b, k, 64, seed=9)


def test_zero_rhs_and_singular_sigma_flag():
    hg = hgm()
    nb, b, k, T = 2, 256, 64, 64
    U, sigma, V = factors(nb, b, k, 1)
    Ut = torch.from_numpy(np.ascontiguousarray(U.transpose(0, 2, 1)).astype(np.float32)).cuda()
    Vt = torch.from_numpy(np.ascontiguousarray(V.transpose(0, 2, 1)).astype(np.float32)).cuda()
    sg = torch.from_numpy(sigma.astype(np.float32)).cuda()
    F, st = hg.block_apply_inverse(Ut, sg, Vt, torch.zeros((nb * b, T), device="cuda"), 0.5)
    assert int(st.item()) == 0 and float(F.abs().max()) == 0.0
    # reading A14: sigma_j <= 1e-6 sigma_1 is flagged (and its triplet dropped), not divided by
    sg2 = sg.clone()
    sg2[1, -1] = 1e-9
    Y = torch.randn((nb * b, T), device="cuda")
    F2, st2 = hg.block_apply_inverse(Ut, sg2, Vt, Y, 0.5)
    torch.cuda.synchronize()
    assert int(st2.item()) != 0 and bool(torch.isfinite(F2).all())
