import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1908_08281_b200 import hg
from synth.hypergraph import CONFIGS, make_input
c = CONFIGS[4]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda(); Y = torch.from_numpy(h.Y).cuda()
ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T)
F, s, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, sync=False)
torch.cuda.synchronize()
for parts in (1, 4):
    os.environ["HG_STREAMS"] = str(parts)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, ws=ws, F=F, sigma=s, status=st, sync=False)
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    print(f"parts {parts}: host enqueue {1e3*min(ts):.3f} ms (launches {hg.last_launch_count()})")
