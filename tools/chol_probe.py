"""Phase clock stamps (clock64) of the last full CholeskyQR factorization of one configs[3] solve.

    python tools/chol_probe.py
Prints cycles: load, POTRF(0), then per panel p: TRSM, trailing update (+lookahead POTRF), and
the TRTRI phases, from hg_debug_counters' chol_clk stamps (block 0 of the launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HG_STREAMS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402

c = CONFIGS[4]
h = make_input(c)
H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
w = torch.from_numpy(h.w).cuda()
Y = torch.from_numpy(h.Y).cuda()
for _ in range(2):
    hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
torch.cuda.synchronize()
clk = np.array(hg.debug_counters()["chol_clk"], dtype=np.int64)
t0 = clk[0]
names = {0: "start", 1: "loaded", 40: "factor done", 41: "trtri diag", 60: "trtri done", 61: "stored",
         30: "p0 lookahead potrf in", 31: "p0 lookahead potrf out", 32: "p1 lookahead potrf in",
         33: "p1 lookahead potrf out", 36: "trtri diag (second run)"}
for i, v in enumerate(clk):
    if v == 0:
        continue
    nm = names.get(i)
    if nm is None and 2 <= i < 40:
        p, ph = divmod(i - 2, 3)
        nm = f"panel {p} " + ("start" if ph == 0 else ("trsm done" if ph == 1 else "update done"))
    if nm is None and 42 <= i < 60:
        nm = f"trtri col {i - 42}"
    if nm is None:
        nm = f"stamp {i}"
    print(f"{i:3d} {nm:26s} {v - t0:9d}")
for a, b in ((30, 31), (32, 33), (40, 41), (41, 36), (41, 42), (59, 60), (60, 61)):
    if clk[a] and clk[b]:
        print(f"  {a}->{b}: {clk[b] - clk[a]}")
