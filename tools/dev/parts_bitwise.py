import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1908_08281_b200 import hg
from synth.hypergraph import CONFIGS, make_input
c = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda(); Y = torch.from_numpy(h.Y).cuda()
nb = c.N // c.b
def run(p):
    os.environ["HG_STREAMS"] = str(p)
    F, s, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, simt=bool(int(os.environ.get("SIMT", "0"))))
    return F.clone(), s.clone()
ref = run(1)
for p in (1, 2, 3, 4):
    for rep in range(4):
        F, s = run(p)
        bad = [i for i in range(nb) if not torch.equal(s[i], ref[1][i]) or not torch.equal(F[i*c.b:(i+1)*c.b], ref[0][i*c.b:(i+1)*c.b])]
        print("parts", p, "rep", rep, "differing blocks", bad, flush=True)
