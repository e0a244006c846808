"""The block Jacobi's stopping rule ("Stopping rule"): the sweep loop ends after a
sweep whose largest measure |a_pq| / sqrt(a_pp a_qq) is <= 4 tol instead of after a sweep without
rotations (HG_JACOBI_STOP=1).  The dropped sweeps only rotate fp32 noise: fewer sweeps, and F and
sigma within a small fraction of the north_star tolerances (2e-5 / 1e-5) of the old rule's -- and
both against the FP64 oracle in the parity tests.  The env knob is read once per process, so each
rule runs in its own subprocess."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1908_08281_b200 import hg
from synth.hypergraph import CONFIGS, make_input
c = CONFIGS[{ci}]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda(); Y = torch.from_numpy(h.Y).cuda()
hg.debug_counters(reset=True)
F, sig, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
torch.cuda.synchronize()
d = hg.debug_counters()
np.save({out!r} + ".F.npy", F.cpu().numpy()); np.save({out!r} + ".s.npy", sig.cpu().numpy())
print(json.dumps({{"sweeps": d["jacobi_total_sweeps"], "blocks": d["jacobi_blocks"]}}))
"""


def run(ci, stop, tmp_path):
    out = str(tmp_path / f"run_{stop}")
    env = dict(os.environ, HG_JACOBI_STOP=str(stop))
    p = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT, ci=ci, out=out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    meta = json.loads(p.stdout.strip().splitlines()[-1])
    return meta, np.load(out + ".F.npy"), np.load(out + ".s.npy")


@pytest.mark.parametrize("ci", [2, 3])
def test_noise_floor_stop_matches_old_rule(ci, tmp_path):
    old, F1, s1 = run(ci, 1, tmp_path)
    new, F4, s4 = run(ci, 4, tmp_path)
    assert new["blocks"] == old["blocks"] > 0
    assert new["sweeps"] <= old["sweeps"]
    assert np.linalg.norm(F4 - F1) / np.linalg.norm(F1) <= 2e-6      # 10% of the F tolerance
    assert np.max(np.abs(s4 - s1) / np.abs(s1)) <= 1e-6              # 10% of the sigma tolerance
