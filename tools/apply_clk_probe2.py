"""k_apply_fused phase timeline (HG_APPLY_CLK build) through hg_block_apply_inverse on NB random blocks:
how the per-k-block time depends on the number of CTAs in flight (per-SM vs aggregate operand-feed limit).
    NB=4 python tools/apply_clk_probe2.py"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_08281_b200 import hg  # noqa: E402
b, k, T = 1024, 256, int(os.environ.get("T", "1000"))
for nb in [int(x) for x in os.environ.get("NB", "1,2,4,8,18,64").split(",")]:
    g = torch.Generator(device="cuda").manual_seed(1)
    Ut = (torch.rand((nb, k, b), device="cuda", generator=g) - 0.5) * 0.06
    Vt = (torch.rand((nb, k, b), device="cuda", generator=g) - 0.5) * 0.06
    sigma = torch.ones((nb, k), device="cuda")
    Y = torch.rand((nb * b, T), device="cuda", generator=g)
    for _ in range(3):
        F, st = hg.block_apply_inverse(Ut, sigma, Vt, Y, 0.5)
    torch.cuda.synchronize()
    n = 160 * 32
    out = (ctypes.c_ulonglong * n)()
    hg._lib.hg_debug_apply_clk(out, n)
    a = np.array(out[:], dtype=np.int64).reshape(160, 32)
    nc = min(160, nb * ((T + 127) // 128))
    r = a[:nc]
    rel = (r - r[:, :1]) / 1e3
    p1 = (rel[:, 3] - rel[:, 2]).mean()
    p2 = (rel[:, 7 + 14] - rel[:, 6]).mean()
    print(f"nb {nb:3d} ctas {nb * ((T + 127) // 128):4d}: product1 {p1:.1f} us ({p1 / 32:.2f}/k-block) "
          f"Zs {(rel[:, 5] - rel[:, 3]).mean():.1f} product2 {p2:.1f} us ({p2 / 8:.2f}/tile) total {rel[:, 31].mean():.1f}")
