"""Small end-to-end runs for compute-sanitizer (one tool per invocation):
hg_solve (device and host entries), hg_cg_solve and hg_solve_schur at configs[0] and configs[1],
plus the boundary variants (HG_GENERAL, HG_UV_BK, ragged T).  Kernels are enqueued directly
(HG_NO_GRAPH=1) so every launch is visible to the tool.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [configs...]
compute-sanitizer is closed on this pool; tests/test_gpu_sanitize.py runs this driver against the
bounds-checked build instead (HG_LIB=check: device traps on index violations).
"""
import os
import sys

os.environ.setdefault("HG_NO_GRAPH", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402
from synth.hypergraph import CONFIGS, make_input  # noqa: E402


def main():
    cfgs = [int(x) for x in sys.argv[1:]] or [1, 2]
    for ci in cfgs:
        c = CONFIGS[ci]
        h = make_input(c)
        H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E)
        w = torch.from_numpy(h.w).cuda()
        Y = torch.from_numpy(h.Y).cuda()
        F, s, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        assert int(st.item()) == 0, ci
        Fh, _ = hg.solve_host(torch.from_numpy(h.row_ptr), torch.from_numpy(h.col_idx), torch.from_numpy(h.w),
                              torch.from_numpy(h.Y), mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        Fc, it, _, st = hg.cg_solve(H, w, Y, mu=c.mu, max_iter=5, tol=0.0)
        assert int(st.item()) == 0, ci
        Fs, st = hg.solve_schur(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        assert int(st.item()) == 0, ci
        Fw, _, st = hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0, woodbury=True)
        X, _, _ = hg.build_theta(H, w, c.mu, c.b)
        Ug, sg, Vg, st = hg.block_rsvd(X, c.k, c.q, 0, general=True, uv_bk=True)
        F7, _, st = hg.solve(H, w, Y[:, :7].contiguous(), mu=c.mu, b=c.b, k=c.k, q=c.q, seed=0)
        torch.cuda.synchronize()
        print(f"cfg{ci}: ok, |F| {float(F.norm()):.4f} |F_host - F| {float((Fh.cuda() - F).norm()):.2e} "
              f"|F_cg| {float(Fc.norm()):.4f} |F_schur| {float(Fs.norm()):.4f}")


if __name__ == "__main__":
    main()
