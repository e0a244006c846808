"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle.

Tolerances (BASELINE.json north_star): relative Frobenius error of the applied
inverse F <= 2e-5, singular values relative <= 1e-5.  Theta blocks: <= 1e-6 of
max|Theta| (fp32 sums of a few dozen terms).  Reconstructions U Sigma V^T are
compared (span-determined), never the sign-ambiguous vectors themselves.
"""
import numpy as np
import pytest
import torch

import oracle
from synth.hypergraph import CONFIGS, cfg5_points, make_input, make_tiny

pytestmark = pytest.mark.gpu

F_TOL, SIG_TOL, THETA_TOL, ORTH_TOL = 2e-5, 1e-5, 1e-6, 1e-5

_cache = {}


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


def dev_inputs(h):
    hg = hgm()
    key = id(h)   # the entry keeps h alive, so its id cannot be reused by another input
    if key not in _cache or _cache[key][0] is not h:
        _cache[key] = (h, hg.incidence_to_device(h.row_ptr, h.col_idx, h.E), torch.from_numpy(h.w).cuda(),
                       torch.from_numpy(h.Y).cuda())
    return _cache[key][1:]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def inputs():
    cache = {}

    def get(i):
        if i not in cache:
            cache[i] = make_input(CONFIGS[i])
        return cache[i]
    return get


# ------------------------------------------------------------------ Omega
@pytest.mark.parametrize("rows,cols,seed", [(1000, 33, 0), (4096, 64, 0), (7, 5, 123)])
def test_gaussian_matches_oracle(rows, cols, seed):
    g = hgm().fill_gaussian(seed, rows, cols).cpu().numpy()
    o = oracle.gaussian_f32(seed, rows * cols).reshape(rows, cols)
    d = np.abs(g.view(np.int32).astype(np.int64) - o.view(np.int32).astype(np.int64))
    assert d.max() <= 1 and np.mean(d == 0) >= 0.9999


# ------------------------------------------------------------------ GEMM
SHAPES = [(128, 64, 128, 2), (256, 256, 1024, 3), (100, 20, 72, 2), (32, 32, 256, 4), (300, 1000, 256, 2),
          (1024, 256, 1024, 1), (40, 500, 36, 3)]


@pytest.mark.parametrize("simt,prec", [(False, 0), (True, 0), (False, 1)])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_all_layouts_vs_fp64(shape, simt, prec):
    hg = hgm()
    M, N, K, batch = shape
    gen = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    for a_mn in (False, True):
        for b_mn in (False, True):
            for d_trans in (False, True):
                A = torch.randn(batch, *((K, M) if a_mn else (M, K)), device="cuda", generator=gen)
                B = torch.randn(batch, *((K, N) if b_mn else (N, K)), device="cuda", generator=gen)
                D = torch.full((batch, N, M) if d_trans else (batch, M, N), float("nan"), device="cuda")
                rs = torch.rand(batch, M, device="cuda", generator=gen) + 0.5
                cs = torch.rand(batch, N, device="cuda", generator=gen) + 0.5
                hg.gemm(A, B, M=M, N=N, K=K, batch=batch, a_mn=a_mn, lda=A.shape[2], sa=A[0].numel(), b_mn=b_mn,
                        ldb=B.shape[2], sb=B[0].numel(), D=D, d_trans=d_trans, ldd=D.shape[2], sd=D[0].numel(),
                        alpha=0.75, rs=rs, srs=M, cs=cs, scs=N, simt=simt, prec=prec, a_exp=11, b_exp=11)
                Am = A.double().transpose(1, 2) if a_mn else A.double()
                Bm = B.double() if b_mn else B.double().transpose(1, 2)
                ref = 0.75 * rs.double()[:, :, None] * (Am @ Bm) * cs.double()[:, None, :]
                got = D.double().transpose(1, 2) if d_trans else D.double()
                assert torch.isfinite(got).all()
                err = float((got - ref).norm() / ref.norm())
                # 3xTF32 keeps fp32-level accuracy (1xTF32 would give ~1e-3; measured
                # 7.8e-7 at K=1024 with the truncation split, 4.7e-7 with rna); 3xF16 with the
                # operands prescaled by 2^11 (|randn| < 32) carries the same 22 significant bits
                assert err < 2e-6, (a_mn, b_mn, d_trans, err)


# ------------------------------------------------------------------ Theta (Eq. 1)
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_theta_blocks_parity(inputs, cfg):
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, _ = dev_inputs(h)
    th, dvr, st = hg.build_theta(H, w, c.mu, c.b, raw=True)
    X, _, st2 = hg.build_theta(H, w, c.mu, c.b)
    assert int(st.item()) == 0 and int(st2.item()) == 0
    assert bool((th == th.transpose(1, 2)).all()), "blocks must be bitwise symmetric (reading A12)"
    assert bool((X == X.transpose(1, 2)).all())
    sel = range(c.nb) if c.nb <= 16 else [0, 1, c.nb // 2, c.nb - 1]
    dv, _ = oracle.degrees(h.row_ptr, h.col_idx, h.w)
    # delta(v) is an fp32 sum of ~20-60 weights: a few ulps (1e-6 = 16 ulp)
    np.testing.assert_allclose(dvr.double().cpu().numpy(), dv ** -0.5, rtol=1e-6)
    for blk in sel:
        ref = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, blk)
        got = th[blk].double().cpu().numpy()
        assert np.abs(got - ref).max() <= THETA_TOL * np.abs(ref).max()
        refx = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, blk, mu=c.mu)
        assert np.abs(X[blk].double().cpu().numpy() - refx).max() <= THETA_TOL


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_assembly_paths_bit_identical(inputs, cfg, monkeypatch):
    """The radix-sorted row kernel (default), the segment-sorted row kernel and the hashed-tile
    kernel add the same terms in the same order (ascending edge id per (u, v)): identical bits."""
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, _ = dev_inputs(h)
    monkeypatch.delenv("HG_ASSEMBLE", raising=False)
    X1, _, s1 = hg.build_theta(H, w, c.mu, c.b)
    monkeypatch.setenv("HG_ASSEMBLE", "tiles")
    X2, _, s2 = hg.build_theta(H, w, c.mu, c.b)
    monkeypatch.setenv("HG_ASSEMBLE", "segments")   # the per-segment bitonic-sort path
    X3, _, s3 = hg.build_theta(H, w, c.mu, c.b)
    monkeypatch.delenv("HG_ASSEMBLE")
    assert int(s1.item()) == 0 and int(s2.item()) == 0 and int(s3.item()) == 0
    assert torch.equal(X1, X2)
    assert torch.equal(X1, X3)


def test_theta_error_flags():
    hg = hgm()
    # vertex 3 isolated; hyperedge 2 empty
    rp = np.array([0, 2, 3, 4, 4], np.int64)
    ci = np.array([0, 1, 0, 1], np.int32)
    H = hg.incidence_to_device(rp, ci, 3)
    w = torch.ones(3, device="cuda")
    _, _, st = hg.build_theta(H, w, 1.0, 4)
    s = int(st.item())
    assert s & 1 and s & 2
    with pytest.raises(hg.HGError) as e:
        hg.solve(H, w, torch.zeros(4, 4, device="cuda"), mu=1.0, b=4, k=4, q=1, seed=0)
    assert e.value.status == hg.HG_ERR_NUMERICAL


# ------------------------------------------------------------------ whole path
def check_against_oracle(h, c, F, sigma, blocks, Ut=None, Vt=None, X=None, k=None, q=None):
    k = k or c.k
    q = c.q if q is None else q
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=k, q=q, seed=c.seed, blocks=blocks,
                     want_UV=Ut is not None)
    Fg = F.double().cpu().numpy()
    sg = sigma.double().cpu().numpy()
    worst = {"F": 0.0, "sigma": 0.0, "recon": 0.0, "orth": 0.0}
    for s_, blk in enumerate(blocks):
        fo = r.F[s_ * c.b:(s_ + 1) * c.b]
        worst["F"] = max(worst["F"], rel(Fg[blk * c.b:(blk + 1) * c.b], fo))
        worst["sigma"] = max(worst["sigma"], float(np.max(np.abs(sg[blk] - r.sigma[s_]) / r.sigma[s_])))
        assert np.all(np.diff(sg[blk]) <= 0)
        if Ut is not None:
            U = Ut[blk].double().cpu().numpy().T
            V = Vt[blk].double().cpu().numpy().T
            rec = U @ np.diag(sg[blk]) @ V.T
            rec_o = r.U[s_] @ np.diag(r.sigma[s_]) @ r.V[s_].T
            worst["recon"] = max(worst["recon"], rel(rec, rec_o))
            worst["orth"] = max(worst["orth"], np.abs(U.T @ U - np.eye(k)).max(), np.abs(V.T @ V - np.eye(k)).max())
            idx = np.abs(U).argmax(0)
            assert np.all(U[idx, np.arange(k)] > 0), "sign rule (SPEC.md:86)"
    assert worst["F"] <= F_TOL, worst
    assert worst["sigma"] <= SIG_TOL, worst
    assert worst["recon"] <= F_TOL, worst
    assert worst["orth"] <= ORTH_TOL, worst
    return worst


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_solve_parity_configs_1_to_3(inputs, cfg):
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, Y = dev_inputs(h)
    X, _, _ = hg.build_theta(H, w, c.mu, c.b)
    # x_unit: build_theta's blocks satisfy |X_ij| <= 1, ||X_ii|| <= 1 -- the 3xF16 products hg_solve uses
    Ut, sigma, Vt, st = hg.block_rsvd(X, c.k, c.q, c.seed, x_unit=True)
    F, st2 = hg.block_apply_inverse(Ut, sigma, Vt, Y, c.mu / (1 + c.mu))
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and int(st2.item()) == 0
    check_against_oracle(h, c, F, sigma, list(range(c.nb)), Ut, Vt)
    # the 3xTF32 products (no x_unit) meet the same bar
    Ut0, sigma0, Vt0, st0 = hg.block_rsvd(X, c.k, c.q, c.seed)
    F0, _ = hg.block_apply_inverse(Ut0, sigma0, Vt0, Y, c.mu / (1 + c.mu))
    assert int(st0.item()) == 0
    check_against_oracle(h, c, F0, sigma0, list(range(c.nb)), Ut0, Vt0)
    # the composite entry point gives the same bits
    F2, sigma2, st3 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    assert int(st3.item()) == 0
    assert torch.equal(F, F2) and torch.equal(sigma, sigma2)


def test_solve_parity_config4_sampled_blocks(inputs):
    """configs[3] (the bench workload) at full size; oracle on blocks {0, nb/2, nb-1}."""
    hg = hgm()
    h = inputs(4)
    c = CONFIGS[4]
    H, w, Y = dev_inputs(h)
    X, _, _ = hg.build_theta(H, w, c.mu, c.b)
    Ut, sigma, Vt, st = hg.block_rsvd(X, c.k, c.q, c.seed)
    F, st2 = hg.block_apply_inverse(Ut, sigma, Vt, Y, c.mu / (1 + c.mu))
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and int(st2.item()) == 0
    check_against_oracle(h, c, F, sigma, [0, c.nb // 2, c.nb - 1], Ut, Vt)


def test_solve_parity_config4_every_stream_part(inputs):
    """configs[3] through hg_solve (the bench entry: 8 stream parts of 8 blocks on forked streams,
    CUDA-graph replay): one block per part (0, 8, ..., 56) and the last block, against the oracle."""
    hg = hgm()
    h = inputs(4)
    c = CONFIGS[4]
    H, w, Y = dev_inputs(h)
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    assert int(st.item()) == 0
    check_against_oracle(h, c, F, sigma, list(range(0, c.nb, 8)) + [c.nb - 1])


def _cfg5_cost(p):
    b, k, q = p
    return b * b * k * (q + 1) + b * k * k * (2 * q + 1)


@pytest.fixture(scope="module")
def cfg5_oracle(inputs):
    """The FP64 oracle on blocks {0, nb-1} of all 36 configs[4] points, computed once as one
    parallel batch (host threads x 2 OpenMP threads each, largest points first)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    h = inputs(5)
    ncores = len(os.sched_getaffinity(0))

    def run(p):
        b, k, q = p
        oracle.set_num_threads(2)   # per host thread (OpenMP ICV): 2 blocks per point
        nb = CONFIGS[5].N // b
        return p, oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=CONFIGS[5].mu, b=b, k=k, q=q,
                               seed=CONFIGS[5].seed, blocks=[0, nb - 1])

    pts = sorted(cfg5_points(), key=_cfg5_cost, reverse=True)
    with ThreadPoolExecutor(max_workers=max(1, ncores // 2)) as ex:
        res = dict(ex.map(run, pts))
    oracle.set_num_threads(ncores)
    return res


@pytest.mark.parametrize("b,k,q", cfg5_points())
def test_solve_parity_config5_all_points(inputs, cfg5_oracle, b, k, q):
    """Every configs[4] (b, k, q) point (36) through hg_solve: F <= 2e-5 and sigma <= 1e-5 against
    the FP64 oracle on the first and last block (north_star: parity on all five configs)."""
    hg = hgm()
    h = inputs(5)
    c = CONFIGS[5].with_(b=b, k=k, q=q)
    H, w, Y = dev_inputs(h)
    F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=b, k=k, q=q, seed=c.seed)
    assert int(st.item()) == 0
    r = cfg5_oracle[(b, k, q)]
    Fg = F.double().cpu().numpy()
    sg = sigma.double().cpu().numpy()
    for s_, blk in enumerate(r.blocks):
        fo = r.F[s_ * b:(s_ + 1) * b]
        fe = rel(Fg[blk * b:(blk + 1) * b], fo)
        se = float(np.max(np.abs(sg[blk] - r.sigma[s_]) / r.sigma[s_]))
        assert fe <= F_TOL and se <= SIG_TOL, (blk, fe, se)
        assert np.all(np.diff(sg[blk]) <= 0)


def test_tiny_inputs_and_k_equals_b():
    """Small ragged-tile shapes; with k = b the path is the exact block inverse (LU)."""
    hg = hgm()
    for (N, b, k, q) in [(32, 8, 4, 0), (32, 8, 8, 2), (48, 16, 12, 1), (40, 20, 20, 1)]:
        h = make_tiny(N, b, k, q)
        c = h.cfg
        H, w, Y = dev_inputs(h)
        F, sigma, st = hg.solve(H, w, Y, mu=1.0, b=b, k=k, q=q, seed=0)
        check_against_oracle(h, c, F, sigma, list(range(N // b)))
        if k == b:
            for blk in range(N // b):
                Xo = oracle.theta_block(h.row_ptr, h.col_idx, h.w, b, blk, mu=1.0)
                lu = 0.5 * np.linalg.solve(Xo, h.Y[blk * b:(blk + 1) * b].astype(float))
                assert rel(F[blk * b:(blk + 1) * b].double().cpu().numpy(), lu) <= F_TOL


@pytest.mark.parametrize("cfg", [2, 4])
def test_stream_parts_bitwise_identical(inputs, cfg, monkeypatch):
    """hg_solve runs disjoint block ranges on forked streams (HG_STREAMS parts);
    blocks are independent and Omega is keyed by the global block index, so any
    part count gives the same bits (3 parts: uneven ranges)."""
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, Y = dev_inputs(h)
    out = {}
    for parts in ("1", "2", "3"):
        monkeypatch.setenv("HG_STREAMS", parts)
        F, s, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        assert int(st.item()) == 0
        out[parts] = (F.clone(), s.clone())
    for parts in ("2", "3"):
        assert torch.equal(out[parts][0], out["1"][0]) and torch.equal(out[parts][1], out["1"][1]), parts


def test_timeline_profiler_parts_overlap(inputs, monkeypatch):
    """hg_profile_enable(2): stream parts stay concurrent and every stage of every part is
    recorded with its part index; the result equals the unprofiled one bit for bit."""
    hg = hgm()
    h = inputs(2)
    c = CONFIGS[2]
    H, w, Y = dev_inputs(h)
    monkeypatch.setenv("HG_STREAMS", "2")
    F0, s0, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    hg.profile_enable(2)
    try:
        F1, s1, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        recs = hg.profile_timeline()
    finally:
        hg.profile_enable(0)
    assert torch.equal(F0, F1) and torch.equal(s0, s1)
    parts = {r[1] for r in recs}
    assert parts == {0, 1}
    for p in parts:
        stages = {r[0] for r in recs if r[1] == p}
        assert {"assemble", "omega", "gemm_power", "gemm_gram", "gemm_qform", "cholinv", "jacobi", "finalize",
                "gemm_apply"} <= stages, stages
    assert all(r[3] >= r[2] >= -1.0 for r in recs)
    # the two parts run concurrently: their spans (first stage start .. last stage end) overlap
    span = sorted((min(r[2] for r in recs if r[1] == p), max(r[3] for r in recs if r[1] == p)) for p in parts)
    assert span[1][0] < span[0][1], span


def test_graph_replay_matches_direct_enqueue(inputs, monkeypatch):
    """hg_solve replays a cached CUDA graph of its launch sequence; the direct path
    (HG_NO_GRAPH=1), a second workspace (new capture) and a repeat call (replay) agree
    bit for bit."""
    hg = hgm()
    h = inputs(2)
    c = CONFIGS[2]
    H, w, Y = dev_inputs(h)
    monkeypatch.setenv("HG_NO_GRAPH", "1")
    F0, s0, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    monkeypatch.delenv("HG_NO_GRAPH")
    F1, s1, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    F2, s2, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)   # fresh outputs: new key
    ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
    F3, s3, st3 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, sync=False)
    hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F3, sigma=s3, status=st3, sync=False)
    torch.cuda.synchronize()
    assert int(st3.item()) == 0
    for F, sg in ((F1, s1), (F2, s2), (F3, s3)):
        assert torch.equal(F, F0) and torch.equal(sg, s0)


def test_deterministic_and_host_entry(inputs):
    hg = hgm()
    h = inputs(2)
    c = CONFIGS[2]
    H, w, Y = dev_inputs(h)
    F1, s1, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    F2, s2, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    assert torch.equal(F1, F2) and torch.equal(s1, s2)
    Fh, sh = hg.solve_host(torch.from_numpy(h.row_ptr), torch.from_numpy(h.col_idx), torch.from_numpy(h.w),
                           torch.from_numpy(h.Y).pin_memory(), mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    assert torch.equal(Fh, F1.cpu()) and torch.equal(sh, s1.cpu())
    F3, _, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=1)
    assert not torch.equal(F1, F3)
    # reading R2 through the host entry (prioritised part streams) gives the device entry's bits
    Fw, sw, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, woodbury=True)
    Fhw, shw = hg.solve_host(torch.from_numpy(h.row_ptr), torch.from_numpy(h.col_idx), torch.from_numpy(h.w),
                             torch.from_numpy(h.Y).pin_memory(), mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0,
                             woodbury=True)
    assert torch.equal(Fhw, Fw.cpu()) and torch.equal(shw, sw.cpu())


def test_host_entry_bitwise_equal_at_k256(inputs):
    """configs[3] (k = 256, 2-CTA Jacobi clusters): the host entry (prioritised part streams, Y
    uploads and F downloads per part) gives the device entry's bits."""
    hg = hgm()
    h = inputs(4)
    c = CONFIGS[4]
    H, w, Y = dev_inputs(h)
    F1, s1, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    assert int(st.item()) == 0
    Fh, sh = hg.solve_host(torch.from_numpy(h.row_ptr), torch.from_numpy(h.col_idx), torch.from_numpy(h.w),
                           torch.from_numpy(h.Y).pin_memory(), mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    assert torch.equal(Fh, F1.cpu()) and torch.equal(sh, s1.cpu())


def test_simt_verification_path_agrees(inputs):
    hg = hgm()
    h = inputs(1)
    c = CONFIGS[1]
    H, w, Y = dev_inputs(h)
    Ft, st_, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    Fs, ss, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, simt=True)
    assert rel(Ft.double().cpu().numpy(), Fs.double().cpu().numpy()) < 1e-5
    check_against_oracle(h, c, Fs, ss, list(range(c.nb)))


def test_device_call_validation():
    hg = hgm()
    h = make_tiny(32, 8, 4, 1)
    H, w, Y = dev_inputs(h)
    ws = hg.Workspace(1024)
    with pytest.raises(hg.HGError) as e:
        hg.solve(H, w, Y, mu=1.0, b=8, k=4, q=1, seed=0, ws=ws)
    assert e.value.status == hg.HG_ERR_INVALID and "workspace too small" in str(e.value)
    with pytest.raises(hg.HGError) as e:
        hg.solve(H, w, Y, mu=-1.0, b=8, k=4, q=1, seed=0)
    assert e.value.status == hg.HG_ERR_INVALID
    with pytest.raises(hg.HGError) as e:
        hg.solve(H, w, Y, mu=1.0, b=8, k=12, q=1, seed=0)
    assert e.value.status == hg.HG_ERR_INVALID


@pytest.mark.parametrize("cfg", [2, 3])
def test_qr_passes_knob_both_parity_green(inputs, cfg, monkeypatch):
    """Intermediate bases take one CholeskyQR pass by default, the final S CholeskyQR2
    (DESIGN.md "QR"); HG_QR_PASSES=2 runs CholeskyQR2 for every QR.  Both meet parity and
    agree with each other to well inside the tolerance (same span, rounding differences)."""
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, Y = dev_inputs(h)
    F1, s1, st1 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    monkeypatch.setenv("HG_QR_PASSES", "2")
    F2, s2, st2 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    monkeypatch.delenv("HG_QR_PASSES")
    blocks = [0, c.nb - 1]
    check_against_oracle(h, c, F1, s1, blocks)
    check_against_oracle(h, c, F2, s2, blocks)
    assert rel(F1.double().cpu().numpy(), F2.double().cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_qr_skip_half_variant_parity_green(inputs, cfg, monkeypatch):
    """HG_QR_SKIP_HALF=1 (opt-in variant): the half-step basis S~ = qr(X^T S) of Alg. 1
     stays un-orthonormalised -- Eq. 10 inside one iteration, one QR
    per iteration.  range(S) is unchanged, so F and sigma still match the oracle's literal Alg. 1."""
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, Y = dev_inputs(h)
    F1, s1, st1 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    monkeypatch.setenv("HG_QR_SKIP_HALF", "1")
    F2, s2, st2 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    n2 = hg.last_launch_count()
    monkeypatch.delenv("HG_QR_SKIP_HALF")
    F3, s3, st3 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    n3 = hg.last_launch_count()
    assert int(st2.item()) == 0 and n2 < n3          # fewer launches: the variant really ran
    assert torch.equal(F1, F3) and torch.equal(s1, s3)   # and the default is back afterwards
    check_against_oracle(h, c, F2, s2, list(range(c.nb)) if cfg < 3 else [0, c.nb - 1])
    assert rel(F1.double().cpu().numpy(), F2.double().cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_lazy_qr_and_explicit_qr_both_parity_green(inputs, cfg, monkeypatch):
    """Default: an intermediate S_j = Y_j R_j^-1 of Alg. 1 is applied lazily,
    Y_{j+1} = (X Y_j) R_j^-1, with X Y_j concurrent to the Cholesky; HG_QR_LAZY=0 forms every
    S_j explicitly.  The same matrices up to rounding: both meet the oracle tolerances and agree closely."""
    hg = hgm()
    h = inputs(cfg)
    c = CONFIGS[cfg]
    H, w, Y = dev_inputs(h)
    F1, s1, st1 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    monkeypatch.setenv("HG_QR_LAZY", "0")
    F2, s2, st2 = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    monkeypatch.delenv("HG_QR_LAZY")
    assert int(st1.item()) == 0 and int(st2.item()) == 0
    blocks = list(range(c.nb)) if cfg < 3 else [0, c.nb - 1]
    check_against_oracle(h, c, F1, s1, blocks)
    check_against_oracle(h, c, F2, s2, blocks)
    assert rel(F1.double().cpu().numpy(), F2.double().cpu().numpy()) <= 1e-5


def test_solve_without_rhs_returns_sigma_only(inputs):
    """T = 0 (no right-hand sides): the factorisation runs, sigma matches the oracle, F is empty."""
    hg = hgm()
    h = inputs(2)
    c = CONFIGS[2]
    H, w, _ = dev_inputs(h)
    Y0 = torch.empty((c.N, 0), dtype=torch.float32, device="cuda")
    F, sigma, st = hg.solve(H, w, Y0, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    assert int(st.item()) == 0 and F.numel() == 0
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, np.zeros((c.N, 0), np.float32), mu=c.mu, b=c.b, k=c.k, q=c.q,
                     seed=c.seed, blocks=[0, c.nb - 1])
    sg = sigma.double().cpu().numpy()
    for s_, blk in enumerate(r.blocks):
        assert np.max(np.abs(sg[blk] - r.sigma[s_]) / r.sigma[s_]) <= SIG_TOL


def test_concurrent_host_threads_distinct_workspaces(inputs):
    """hg_solve from two host threads at once (distinct workspaces, streams and outputs) gives the
    single-thread bits: the library's part streams and fork/join events are per host thread."""
    import threading
    hg = hgm()
    h = inputs(2)
    c = CONFIGS[2]
    H, w, Y = dev_inputs(h)
    F0, s0, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    torch.cuda.synchronize()
    results, errors = {}, []

    def worker(i):
        try:
            st = torch.cuda.Stream()
            ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
            with torch.cuda.stream(st):
                for _ in range(3):
                    F, s, status = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed, ws=ws, stream=st)
            st.synchronize()
            results[i] = (F, s, int(status.item()))
        except Exception as e:   # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for i in range(2):
        F, s, status = results[i]
        assert status == 0 and torch.equal(F, F0) and torch.equal(s, s0)


def test_solve_blocks_shards_equal_full_solve(inputs):
    """hg_solve_blocks on disjoint block ranges (one rank's share each) reproduces hg_solve's bits."""
    import bench
    hg = hgm()
    h = inputs(2)
    c = CONFIGS[2]
    H, w, Y = dev_inputs(h)
    F0, s0, _ = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed)
    F = torch.zeros_like(F0)
    sig = []
    for r in range(3):
        b0, cnt = bench.shard_range(c.nb, r, 3)
        _, s, st = hg.solve_blocks(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed, blk_begin=b0, blk_count=cnt,
                                   F=F)
        assert int(st.item()) == 0
        sig.append(s)
    assert torch.equal(F, F0) and torch.equal(torch.cat(sig, 0), s0)
    with pytest.raises(hg.HGError):
        hg.solve_blocks(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=c.seed, blk_begin=c.nb - 1, blk_count=2)
