"""GPU: memory-safety and race checks without compute-sanitizer (closed on this pool: runs under
it left GPUs needing a reset).  DESIGN.md "Sanitizers":

  * bounds   -- tools/sanitize_run.py (hg_solve device + host entries, CG, Schur, R2, HG_GENERAL /
               HG_UV_BK, ragged T at configs[0], configs[1] and the bench workload configs[3])
               against libhgrsvd_check.so, whose kernels check their shared / global indices and
               trap on a violation (HG_DCHECK, -DHG_BOUNDS_CHECK);
  * initcheck-- a workspace pre-filled with NaN bit patterns gives bitwise the result of a zeroed
               one: no kernel reads scratch it did not write first;
  * memcheck -- guard bytes after the workspace and after the outputs stay untouched;
  * racecheck-- repeated runs are bitwise identical (every reduction has a fixed order; the only
               atomics order work, never values -- DESIGN.md §6).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from synth.hypergraph import CONFIGS, make_input

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def hgm():
    from paper_1908_08281_b200 import hg
    return hg


@pytest.fixture(scope="module")
def inputs():
    hg = hgm()
    cache = {}

    def get(i):
        if i not in cache:
            c = CONFIGS[i]
            h = make_input(c)
            cache[i] = (c, h, hg.incidence_to_device(h.row_ptr, h.col_idx, h.E), torch.from_numpy(h.w).cuda(),
                        torch.from_numpy(h.Y).cuda())
        return cache[i]
    return get


def test_bounds_checked_build_runs_clean():
    assert os.path.exists(os.path.join(ROOT, "paper_1908_08281_b200", "libhgrsvd_check.so"))
    env = dict(os.environ, HG_LIB="check")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "1", "2", "4"], env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "HG_DCHECK failed" not in out, out[-3000:]
    assert out.count(": ok,") == 3, out[-3000:]


@pytest.mark.parametrize("cfg", [1, 2])
def test_poisoned_workspace_gives_identical_bits(inputs, cfg):
    hg = hgm()
    c, h, H, w, Y = inputs(cfg)
    n = hg.workspace_size(c.N, h.E, h.nnz, c.b, c.k, c.T)
    res = []
    for fill in (0x00, 0xFF):   # 0xFFFFFFFF is a NaN as fp32 and -1 as int32
        ws = hgm().Workspace(n + (1 << 20))
        ws.buf.fill_(fill)
        ws.nbytes = n
        F = torch.full((c.N + 64, c.T), 7.0, device="cuda")   # 64 guard rows after the output
        sig = torch.full((c.nb + 4, c.k), 7.0, device="cuda")
        Fo, so, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F[:c.N], sigma=sig[:c.nb])
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        off = ws.ptr.value - ws.buf.data_ptr()
        assert bool((ws.buf[off + n:off + n + (1 << 20)] == fill).all()), "write past the workspace"
        assert bool((F[c.N:] == 7.0).all()) and bool((sig[c.nb:] == 7.0).all()), "write past an output"
        res.append((Fo.clone(), so.clone()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])


def test_poisoned_workspace_cg_and_schur(inputs):
    hg = hgm()
    c, h, H, w, Y = inputs(2)
    out = []
    for fill in (0x00, 0xFF):
        n = hg.cg_workspace_size(c.N, h.E, h.nnz, c.T, 5)
        ws = hg.Workspace(n + (1 << 20))
        ws.buf.fill_(fill)
        ws.nbytes = n
        Fc, it, _, st = hg.cg_solve(H, w, Y, mu=c.mu, max_iter=5, tol=0.0, ws=ws)
        assert int(st.item()) == 0
        n2 = hg.schur_workspace_size(c.N, h.E, h.nnz, c.b, c.k, c.T)
        ws2 = hg.Workspace(n2 + (1 << 20))
        ws2.buf.fill_(fill)
        ws2.nbytes = n2
        Fs, st2 = hg.solve_schur(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws2)
        assert int(st2.item()) == 0
        for wsx, nn in ((ws, n), (ws2, n2)):
            off = wsx.ptr.value - wsx.buf.data_ptr()
            assert bool((wsx.buf[off + nn:off + nn + (1 << 20)] == fill).all())
        out.append((Fc.clone(), Fs.clone()))
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])


def test_repeated_runs_bitwise_identical(inputs):
    hg = hgm()
    c, h, H, w, Y = inputs(4)
    ref = None
    for _ in range(3):
        F, s, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        assert int(st.item()) == 0
        if ref is None:
            ref = (F.clone(), s.clone())
        else:
            assert torch.equal(F, ref[0]) and torch.equal(s, ref[1])
