"""GPU parity for NEXT-4, the hyperedge-weight update:
hg_weight_gradient and hg_weight_step through the C ABI against the FP64 oracle
(or_weight_gradient, or_weight_step), plus the SPEC.md step examples and a short
alternating loop whose objective (oracle P(w)) does not increase."""
import numpy as np
import pytest
import torch

import oracle
from synth.hypergraph import CONFIGS, make_input

pytestmark = pytest.mark.gpu
_inp = {}


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


def get(cfg):
    if cfg not in _inp:
        h = make_input(CONFIGS[cfg])
        hg = hgm()
        _inp[cfg] = (h, hg.incidence_to_device(h.row_ptr, h.col_idx, h.E), torch.from_numpy(h.w).cuda(),
                     torch.from_numpy(h.Y).cuda())
    return _inp[cfg]


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_weight_gradient_matches_oracle(cfg):
    hg = hgm()
    h, H, w, Y = get(cfg)
    F, _, _, st = hg.cg_solve(H, w, Y, mu=CONFIGS[cfg].mu, max_iter=30, tol=1e-6)
    g, st2 = hg.weight_gradient(H, w, F, kappa=0.3)
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and int(st2.item()) == 0
    go = oracle.weight_gradient(h.row_ptr, h.col_idx, h.w, F.double().cpu().numpy(), kappa=0.3)
    gg = g.double().cpu().numpy()
    assert np.max(np.abs(gg - go)) <= 1e-5 * np.max(np.abs(go))


def test_weight_step_spec_examples():
    hg = hgm()
    for w0, g0, want, act in [([0.5, 0.5], [1.0, -1.0], [0.4, 0.6], [0, 0]),
                              ([0.05, 0.95], [1.0, -1.0], [0.0, 1.0], [1, 0])]:
        w = torch.tensor(w0, dtype=torch.float32, device="cuda")
        a = torch.zeros(2, dtype=torch.int32, device="cuda")
        st = hg.weight_step(w, a, torch.tensor(g0, dtype=torch.float32, device="cuda"), 0.1)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        np.testing.assert_allclose(w.cpu().numpy(), want, atol=1e-7)
        assert a.cpu().tolist() == act
    w = torch.tensor([0.0, 1.0], device="cuda")
    a = torch.ones(2, dtype=torch.int32, device="cuda")
    st = hg.weight_step(w, a, torch.ones(2, device="cuda"), 0.1)
    torch.cuda.synchronize()
    assert int(st.item()) & 128


def test_weight_step_matches_oracle_and_loop_decreases_objective():
    hg = hgm()
    h, H, w0, Y = get(2)
    c = CONFIGS[2]
    F, _, _, _ = hg.cg_solve(H, w0, Y, mu=c.mu, max_iter=30, tol=1e-6)
    Fh = F.double().cpu().numpy()
    w = (w0 / w0.sum()).contiguous()
    a = torch.zeros(h.E, dtype=torch.int32, device="cuda")
    kappa = 1.0
    objs = [oracle.weight_objective(h.row_ptr, h.col_idx, w.cpu().numpy(), Fh, kappa=kappa)]
    for step in range(8):
        g, _ = hg.weight_gradient(H, w, F, kappa=kappa)
        w_prev, a_prev = w.double().cpu().numpy(), a.cpu().numpy()
        gh = g.double().cpu().numpy()
        mu = 0.5 * w_prev.min() / np.max(np.abs(gh - gh.mean()))   # small step: descent, no vertex isolated
        st = hg.weight_step(w, a, g, mu)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        wo, ao = oracle.weight_step(w_prev, a_prev, g.double().cpu().numpy(), mu)
        wg = w.double().cpu().numpy()
        assert np.array_equal(a.cpu().numpy(), ao)
        assert np.max(np.abs(wg - wo)) <= 1e-6 * np.max(wo) + 1e-9
        assert abs(wg.sum() - 1.0) <= 1e-5 and wg.min() >= 0.0
        objs.append(oracle.weight_objective(h.row_ptr, h.col_idx, w.cpu().numpy(), Fh, kappa=kappa))
    assert all(objs[i + 1] <= objs[i] + 1e-9 * abs(objs[i]) for i in range(len(objs) - 1)), objs


def test_weight_step_with_clamping_matches_oracle():
    hg = hgm()
    h, H, w0, Y = get(2)
    c = CONFIGS[2]
    F, _, _, _ = hg.cg_solve(H, w0, Y, mu=c.mu, max_iter=30, tol=1e-6)
    w = (w0 / w0.sum()).contiguous()
    a = torch.zeros(h.E, dtype=torch.int32, device="cuda")
    g, _ = hg.weight_gradient(H, w, F, kappa=1.0)
    gh = g.double().cpu().numpy()
    w_prev = w.double().cpu().numpy()
    dev_ = gh - gh.mean()
    thr = w_prev[dev_ > 0] / dev_[dev_ > 0]                      # step at which each weight would reach 0
    mu = float(np.quantile(thr, 0.2))                            # clamps ~20% of those weights
    st = hg.weight_step(w, a, g, mu)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    wo, ao = oracle.weight_step(w_prev, np.zeros(h.E, np.int32), gh, mu)
    assert 0 < ao.sum() < h.E
    assert np.array_equal(a.cpu().numpy(), ao)
    assert np.max(np.abs(w.double().cpu().numpy() - wo)) <= 1e-6 * np.max(wo) + 1e-9


def oracle_learn(h, w0, F, kappa, mu, steps):
    w = w0 / w0.sum()
    a = np.zeros(len(w), np.int32)
    g = oracle.weight_gradient(h.row_ptr, h.col_idx, w.astype(np.float32), F, kappa=kappa)
    P = oracle.weight_objective(h.row_ptr, h.col_idx, w.astype(np.float32), F, kappa=kappa)
    trace, done, tries = [P], 0, 0
    while done < steps and tries < 8 * steps:
        tries += 1
        wt, at = oracle.weight_step(w, a, g, mu)
        try:
            gt = oracle.weight_gradient(h.row_ptr, h.col_idx, wt.astype(np.float32), F, kappa=kappa)
            Pt = oracle.weight_objective(h.row_ptr, h.col_idx, wt.astype(np.float32), F, kappa=kappa)
        except oracle.OracleError:
            mu *= 0.5
            continue
        if not Pt <= P:
            mu *= 0.5
            continue
        w, a, g, P = wt, at, gt, Pt
        trace.append(P)
        done += 1
    return w, a, trace


def test_weight_objective_and_learn_loop_match_oracle():
    hg = hgm()
    h, H, w0, Y = get(1)
    c = CONFIGS[1]
    F, _, _, _ = hg.cg_solve(H, w0, Y, mu=c.mu, max_iter=30, tol=1e-6)
    Fh = F.double().cpu().numpy()
    kappa = 0.5
    w = (w0 / w0.sum()).contiguous()
    g, _ = hg.weight_gradient(H, w, F, kappa=kappa)
    P = hg.weight_objective(F, w, g, kappa=kappa)
    Po = oracle.weight_objective(h.row_ptr, h.col_idx, w.cpu().numpy(), Fh, kappa=kappa)
    assert abs(P - Po) <= 1e-5 * abs(Po)
    wg, ag, trace, _ = hg.learn_weights(H, w0, F, kappa=kappa, mu=1e-4, steps=6)
    wo, ao, traceo = oracle_learn(h, h.w.astype(np.float64), Fh, kappa, 1e-4, 6)
    assert len(trace) == len(traceo) == 7
    assert all(trace[i + 1] <= trace[i] for i in range(6))
    np.testing.assert_allclose(trace, traceo, rtol=1e-5)
    assert np.array_equal(ag.cpu().numpy(), ao)
    assert np.max(np.abs(wg.double().cpu().numpy() - wo)) <= 1e-5 * np.max(wo)


@pytest.mark.parametrize("solver", ["cg", "rsvd", "nested"])
def test_adaptive_learning_alternation(solver):
    """Two outer passes of solve F -> learn w: every weight phase lowers its objective
    and the weights stay on the simplex (the solves and steps themselves are checked above)."""
    hg = hgm()
    h, H, w0, Y = get(1)
    c = CONFIGS[1]
    F, w, hist = hg.adaptive_learning(H, w0, Y, mu=c.mu, kappa=0.5, outer=2, weight_steps=3, step=1e-4,
                                      solver=solver, b=c.b, k=c.k, q=c.q, super_block=c.N)
    assert len(hist) == 2 and all(after <= before for before, after in hist)
    wn = w.double().cpu().numpy()
    assert abs(wn.sum() - 1.0) <= 1e-5 and wn.min() >= 0.0
    assert F.shape == Y.shape and bool(torch.isfinite(F).all())
