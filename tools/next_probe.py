"""One call each of the §8(f) entry points at configs[3] (for an ncu launch list):
hg_solve_schur, hg_weight_gradient (+ step, objective), hg_solve(HG_WOODBURY)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HG_NO_GRAPH", "1")
import torch  # noqa: E402

from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402

c = CONFIGS[4]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda()
Y = torch.from_numpy(h.Y).cuda()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
F, st = hg.solve_schur(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
g, st2 = hg.weight_gradient(H, w, F, kappa=1.0)
ws_ = (w / w.sum()).contiguous()
act = torch.zeros(h.E, dtype=torch.int32, device="cuda")
hg.weight_step(ws_, act, g, 1e-9)
P = hg.weight_objective(F, w, g, kappa=1.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("status", int(st.item()), int(st2.item()), "P", P)
