"""Phase clock stamps of the Jacobi eigen-preconditioner (eig.cu, block 0) for one solve.

    python tools/eig_probe.py [--config 4]
Prints cycles for: load, tridiagonalisation, bisection, each inverse iteration.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--b", type=int)
    ap.add_argument("--k", type=int)
    ap.add_argument("--q", type=int)
    a = ap.parse_args()
    os.environ["HG_STREAMS"] = "1"
    c = CONFIGS[a.config]
    c = c.with_(**{n: getattr(a, n) for n in ("b", "k", "q") if getattr(a, n) is not None})
    h = make_input(c)
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
    w = torch.from_numpy(h.w).cuda()
    Y = torch.from_numpy(h.Y).cuda()
    for _ in range(2):
        F, sigma, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
    torch.cuda.synchronize()
    clk = np.zeros(32, np.int64)
    assert hg._lib.hg_debug_eig_clocks(clk.ctypes.data_as(ctypes.c_void_p)) == 0
    names = ["load", "tridiag", "gap", "bisection", "invit1", "invit2", "invit3"]
    d = np.diff(clk[:8])
    print("eig phases (cycles, block 0):", {n: int(x) for n, x in zip(names, d)}, "total", int(clk[7] - clk[0]))
    for q in range(4):
        s = clk[8 + 5 * q: 13 + 5 * q]
        print(f"tridiag step {64 * q}: symv {s[1] - s[0]}, scalars/v/y {s[2] - s[1]}, w {s[3] - s[2]}, update {s[4] - s[3]}")


if __name__ == "__main__":
    main()
