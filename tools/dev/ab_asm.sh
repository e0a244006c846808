# A/B of one kernel change: F/sigma hash at configs 2 and 4, then bench stage times
python -c "
import torch, hashlib
from paper_1908_08281_b200 import hg
from synth.hypergraph import CONFIGS, make_input
for cfg in (2, 4):
    c = CONFIGS[cfg]; h = make_input(c)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    F, s, st = hg.solve(H, torch.from_numpy(h.w).cuda(), torch.from_numpy(h.Y).cuda(), mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    print(cfg, int(st.item()), hashlib.md5(F.cpu().numpy().tobytes() + s.cpu().numpy().tobytes()).hexdigest())
"
python bench.py --no-cg --no-r2 --no-schur --no-weights --no-cpu-baseline --steps 20 | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['stages']['assemble']['ms_per_step'], d['parity']['F_rel_fro'])"
