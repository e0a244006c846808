#!/usr/bin/env python
"""Benchmark of the block randomized SVD hot path (arXiv:1908.08281) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A step is one pass of the whole hot path -- hg_solve: degrees, diagonal-block
assembly, Alg. 1 on every block (Omega, 2q+2 block GEMMs, 2q+1 CholeskyQR2,
B = S^T X, one-sided Jacobi SVD, U/V), and the Eq. 15 apply to the N x T
tag-label RHS -- on configs[3] of BASELINE.json (N=65536, b=1024, k=256, q=3,
T=1000) with inputs resident in HBM.  value = diagonal blocks per second over
all ranks; the per-block inputs (256 MiB of X blocks, 250 MiB of Y) exceed the
126 MB L2 every step, so no L2 flush is needed.

One JSON line on rank 0.  N > 1 (torchrun, or
`--gpus N` alone, which spawns the N ranks itself): ONE problem sharded by
contiguous block ranges -- rank r solves its blocks (hg_solve_blocks, no
collective on the data path), then F and sigma are all-gathered over NCCL;
strong scaling, the step time is the max over ranks.  --independent: one
problem per rank (Omega seed = rank), weak scaling.

--impl reference times the FP64 CPU oracle (oracle/, the stand-in reference:
there is no reference implementation, only the paper) on a bounded sample of
the same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

TF32_OVER_BF16 = 1.1 / 2.25   # nominal dense tf32 / bf16 ratio (B200_PROFILING.md)


# ---------------------------------------------------------------- distributed plumbing
def dist_setup(backend: str):
    """(rank, world, local_rank); initialises torch.distributed when WORLD_SIZE > 1."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return rank, world, local


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_range(nb: int, rank: int, world: int):
    """Contiguous diagonal-block range [begin, begin + count) of one rank:
    blocks are independent, so a problem shards over ranks with no collective on the data path."""
    b0 = nb * rank // world
    return b0, nb * (rank + 1) // world - b0


def shard_rows(nb: int, b: int, world: int):
    """Row ranges (row0, nrows) of every rank's block range: known to all ranks without a collective."""
    return [(shard_range(nb, r, world)[0] * b, shard_range(nb, r, world)[1] * b) for r in range(world)]


def allgather_rows(F_local, row0: int, nrows: int, world: int, counts=None, out=None):
    """The optional exchange of a sharded solve: every rank's F rows [row0, row0 + nrows) gathered
    into the full F on every rank (NCCL over NVLink on GPUs; gloo in the CPU tests).  `counts` =
    every rank's (row0, nrows) (shard_rows; exchanged with all_gather_object when absent); `out`:
    the full-size destination (F_local itself is allowed: its own rows are already in place)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return F_local[row0:row0 + nrows]
    if counts is None:
        counts = [None] * world
        dist.all_gather_object(counts, (row0, nrows))
    mx = max(n for _, n in counts)   # collectives need equal sizes: pad to the largest share
    if all(n == mx for _, n in counts) and all(r0 == i * mx for i, (r0, _) in enumerate(counts)):
        # equal contiguous shares: one all_gather_into_tensor straight into the full F
        full = out if out is not None else torch.empty((world * mx, F_local.shape[1]), dtype=F_local.dtype,
                                                       device=F_local.device)
        mine = F_local[row0:row0 + nrows]
        if full.data_ptr() == F_local.data_ptr():
            mine = mine.clone()   # in-place all-gather: the input may not alias the output
        dist.all_gather_into_tensor(full, mine.contiguous())
        return full
    mine = torch.zeros((mx, F_local.shape[1]), dtype=F_local.dtype, device=F_local.device)
    mine[:nrows] = F_local[row0:row0 + nrows]
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    res = torch.cat([parts[r][:n] for r, (_, n) in enumerate(counts)], 0)
    if out is not None:
        out.copy_(res)
        return out
    return res


def free_port() -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def spawn_ranks(n: int, argv) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 with the same arguments; rank 0 prints the JSON line."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def nccl_env():
    """Communicator-init lines of NCCL on stderr (rank verification), unless the caller set NCCL_DEBUG."""
    if "NCCL_DEBUG" not in os.environ:
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def selftest_dist(args) -> int:
    """The multi-rank harness on CPU (gloo): ranks from the environment (or spawned by --gpus), the
    block shard ranges, the all-gather of F and sigma into full arrays, max-over-ranks timing.  Each
    rank writes a closed-form value into its own rows only, so a wrong range or gather is visible."""
    import torch
    from synth.hypergraph import CONFIGS
    rank, world, _ = dist_setup("gloo")
    c = CONFIGS[args.config]
    nb, b, T, k = c.nb, c.b, max(c.T, 1), c.k
    b0, cnt = shard_range(nb, rank, world)
    F = torch.zeros((nb * b, T))
    rows = torch.arange(b0 * b, (b0 + cnt) * b, dtype=torch.float32)[:, None]
    F[b0 * b:(b0 + cnt) * b] = rows * 1000.0 + torch.arange(T, dtype=torch.float32)[None, :]
    sig = torch.arange(b0, b0 + cnt, dtype=torch.float32)[:, None] + torch.zeros(cnt, k)
    F_all = torch.empty_like(F)
    sigma = torch.empty(nb, k)
    allgather_rows(F, b0 * b, cnt * b, world, counts=shard_rows(nb, b, world), out=F_all)
    allgather_rows(sig, 0, cnt, world, counts=[shard_range(nb, r, world) for r in range(world)], out=sigma)
    want = torch.arange(nb * b, dtype=torch.float32)[:, None] * 1000.0 + torch.arange(T, dtype=torch.float32)[None, :]
    ok = bool(torch.equal(F_all, want)) and bool(torch.equal(sigma[:, 0], torch.arange(nb, dtype=torch.float32)))
    ms = max_over_ranks(1.0 + rank)
    oks = max_over_ranks(0.0 if ok else 1.0)
    if rank == 0:
        print(json.dumps({"selftest": "dist", "n_gpus": world, "ok": oks == 0.0, "ms_per_step_max": ms,
                          "shards": [shard_range(nb, r, world) for r in range(world)], "nb": nb}), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0 if oks == 0.0 else 1


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - no NVML
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


F16_STAGES = ("gemm_power", "gemm_gram")


def measure_tf32_peak(dev, n: int = 8192, sustain_s: float = 4.0):
    """The TF32 dense tensor peak on this GPU, measured like MEASURED_PEAKS.json's bf16 figures
    (SURVEY.md §8(d)): torch.matmul fp32 with TF32 allowed (cuBLAS picks its tf32 tensor-core
    kernel), n^3, 2 n^3 flop per product; best of 10 (burst) and back to back for `sustain_s`
    seconds (sustained, under the power cap), with the SM clocks sampled during the loop."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        g = torch.Generator(device=dev).manual_seed(0)
        a = torch.randn(n, n, device=dev, generator=g)
        b = torch.randn(n, n, device=dev, generator=g)
        c = torch.empty(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize(dev)
        flop = 2.0 * n ** 3
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1) / 1e3)
        reps = max(10, int(sustain_s / best))
        with ClockSampler(dev.index, period_s=0.02) as clk:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize(dev)
        sust = e0.elapsed_time(e1) / 1e3 / reps
        return {"tf32_tflops": flop / best / 1e12, "tf32_tflops_sustained": flop / sust / 1e12,
                "n": n, "sustained_s": sust * reps, "clocks_sustained": clk.summary(),
                "how": f"torch.matmul fp32, allow_tf32, {n}^3 (2 n^3 flop): best of 10 (burst) and "
                       f"{reps} back to back (sustained), CUDA events"}
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def workload_config(args):
    from synth.hypergraph import CONFIGS
    c = CONFIGS[args.config]
    kw = {}
    if args.b:
        kw["b"] = args.b
    if args.k:
        kw["k"] = args.k
    if args.q is not None:
        kw["q"] = args.q
    return c.with_(**kw) if kw else c


def config_json(c, note=None):
    d = {"workload": f"configs[{ {'cfg1': 0, 'cfg2': 1, 'cfg3': 2, 'cfg4': 3, 'cfg5': 4}[c.name] }] {c.name}: "
                     f"N={c.N}, b={c.b}, nb={c.nb}, k={c.k}, q={c.q}, T={c.T}, mu={c.mu}",
         "N": c.N, "b": c.b, "nb": c.nb, "k": c.k, "q": c.q, "T": c.T, "mu": c.mu,
         "l2": "inputs larger than L2 (X blocks 4*N*b bytes, Y 4*N*T bytes per step); no flush",
         "data": "synthetic seeded image-tagging hypergraph (synth/hypergraph.py), stands in for the paper's "
                 "private Flickr dataset"}
    if note:
        d["note"] = note
    return d


def oracle_sample(h, c, n_blocks, seed=0):
    import oracle
    nb = c.nb
    blocks = [int(round(i * (nb - 1) / max(1, n_blocks - 1))) for i in range(n_blocks)] if n_blocks > 1 else [0]
    r = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, blocks=blocks)
    return r


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        nccl_env()
    rank, world, local = dist_setup("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1908_08281_b200 import hg
    from synth.hypergraph import make_input

    c = workload_config(args)
    h = make_input(c)
    # N > 1 default: ONE problem sharded by contiguous block ranges: rank r solves
    # its blocks with hg_solve_blocks (no collective on the data path), then F and sigma are
    # all-gathered (NCCL over NVLink) -- strong scaling.  --independent: one problem per rank (Omega
    # seed = rank), weak scaling.
    shard = world > 1 and not args.independent
    seed = 0 if (shard or world == 1) else rank
    H = hg.incidence_to_device(h.row_ptr, h.col_idx, h.E, device=dev)
    w = torch.from_numpy(h.w).to(dev)
    Y = torch.from_numpy(h.Y).to(dev)
    ws = hg.Workspace.for_sizes(c.N, h.E, h.nnz, c.b, c.k, c.T, device=dev)
    F = torch.empty((c.N, c.T), dtype=torch.float32, device=dev)
    sigma = torch.empty((c.nb, c.k), dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    sb0, scnt = shard_range(c.nb, rank, world) if shard else (0, c.nb)
    sig_sh = torch.empty((scnt, c.k), dtype=torch.float32, device=dev)
    F_all = torch.empty_like(F) if shard else F
    rows_all = shard_rows(c.nb, c.b, world) if shard else None
    blks_all = [shard_range(c.nb, r, world) for r in range(world)] if shard else None

    def step():
        if shard:
            hg.solve_blocks(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, blk_begin=sb0, blk_count=scnt,
                            sync=False, ws=ws, F=F, sigma=sig_sh, status=status, stream=stream)
            allgather_rows(F, sb0 * c.b, scnt * c.b, world, counts=rows_all, out=F_all)
            allgather_rows(sig_sh, 0, scnt, world, counts=blks_all, out=sigma)
        else:
            hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, sync=False, ws=ws, F=F, sigma=sigma,
                     status=status, stream=stream)

    for _ in range(args.warmup):
        step()
    launches_per_step = hg.last_launch_count()
    torch.cuda.synchronize(dev)
    if int(status.item()) != 0:
        raise RuntimeError(f"device status {int(status.item())} during warm-up")
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, dev)
    value = (c.nb if shard else world * c.nb) / (ms / 1e3)
    # the device status word of the timed steps (OR-ed over all of them; checked after the region so
    # the check adds no host synchronisation inside it), and the timed outputs of the sampled blocks
    # for the parity check in the cpu_baseline leg
    timed_status = int(status.item())
    par_blocks = [0, c.nb - 1] if c.nb > 1 else [0]
    F_timed = {blk: F_all[blk * c.b:(blk + 1) * c.b].double().cpu().numpy() for blk in par_blocks}
    s_timed = {blk: sigma[blk].double().cpu().numpy() for blk in par_blocks}
    if timed_status != 0:
        raise RuntimeError(f"device status {timed_status} during the timed steps")

    # per-stage attribution: the same steps with per-stage CUDA events on the stream
    hg.debug_counters(reset=True)
    hg.profile_enable(True)
    torch.cuda.synchronize(dev)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(args.steps):
        step()
    pe1.record(stream)
    prof = hg.profile_collect()
    hg.profile_enable(False)
    torch.cuda.synchronize(dev)
    prof_ms_per_step = pe0.elapsed_time(pe1) / args.steps
    dbg = hg.debug_counters()
    sweeps_avg = dbg["jacobi_total_sweeps"] / max(1, dbg["jacobi_blocks"])
    chol_full_frac = dbg["chol_full"] / max(1, dbg["chol_full"] + dbg["chol_near_identity"])
    stages = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                  "share": v[0] / args.steps / prof_ms_per_step} for k, v in prof.items()}

    # (the end-to-end timing comes BEFORE the TF32 peak measurement below: its 4 s sustained GEMM loop drives the
    #  GPU into its power cap, and a host-entry timing taken right after it read 0.3-0.6 ms high)
    # end to end through the host entry point (pinned buffers, copies inside the timed region).
    # Sharded (N > 1): per rank, the pinned H2D of H, w and its Y rows into the device buffers, its
    # block range (hg_solve_blocks), the all-gather of F and sigma, and the D2H of the full F and
    # sigma on rank 0 (the user's result), all inside the timed region.
    rp = torch.from_numpy(h.row_ptr).pin_memory()
    ci = torch.from_numpy(h.col_idx).pin_memory()
    wh = torch.from_numpy(h.w).pin_memory()
    Yh = torch.from_numpy(h.Y).pin_memory()
    Fh = torch.empty((c.N, c.T), dtype=torch.float32).pin_memory()
    sh = torch.empty((c.nb, c.k), dtype=torch.float32).pin_memory()
    yr0, yr1 = sb0 * c.b, (sb0 + scnt) * c.b

    def e2e_step():
        if not shard:
            hg.solve_host(rp, ci, wh, Yh, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, F=Fh, sigma=sh, ws=ws,
                          stream=stream)
            return
        H.row_ptr.copy_(rp, non_blocking=True)
        H.col_idx.copy_(ci, non_blocking=True)
        w.copy_(wh, non_blocking=True)
        Y[yr0:yr1].copy_(Yh[yr0:yr1], non_blocking=True)
        step()
        if rank == 0:
            Fh.copy_(F_all, non_blocking=True)
            sh.copy_(sigma, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()

    for _ in range(max(3, min(args.warmup, 5))):   # pinned buffers first-touched, graph uploaded, copy engines warm
        e2e_step()
    barrier()
    n_e2e = max(5, min(args.steps, 20))
    t0 = time.perf_counter()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    for _ in range(n_e2e):
        e2e_step()
    ee1.record(stream)
    torch.cuda.synchronize(dev)
    wall_e2e = (time.perf_counter() - t0) / n_e2e
    e2e_ms = max_over_ranks(max(ee0.elapsed_time(ee1) / n_e2e, wall_e2e * 1e3), dev)
    if shard:
        h2d = (c.N + 1) * 8 + h.nnz * 4 + h.E * 4 + (yr1 - yr0) * c.T * 4
        d2h = (c.N * c.T * 4 + c.nb * c.k * 4) if rank == 0 else 0
    else:
        h2d = (c.N + 1) * 8 + h.nnz * 4 + h.E * 4 + c.N * c.T * 4
        d2h = c.N * c.T * 4 + c.nb * c.k * 4

    peaks, peak_src = load_peaks()
    # TF32 peak: measured here (cuBLAS tf32 8192^3, burst and sustained); the
    # bf16-derived figure (MEASURED_PEAKS bf16 x nominal 1.1/2.25) only with --no-tf32-peak
    tf32_meas = None if args.no_tf32_peak else measure_tf32_peak(dev)
    if tf32_meas:
        tf32_burst, tf32_sust = tf32_meas["tf32_tflops"], tf32_meas["tf32_tflops_sustained"]
        tf32_src = "measured in this run: " + tf32_meas["how"]
    else:
        tf32_sust = peaks["bf16_tflops_sustained"] * TF32_OVER_BF16
        tf32_burst = peaks["bf16_tflops"] * TF32_OVER_BF16
        tf32_src = f"derived: MEASURED_PEAKS bf16 ({peak_src}) x nominal tf32/bf16 1.1/2.25"
    # the denominator for kernels timed inside the step: burst when the timed region's clocks
    # show no power cap (the GPU held its boost clock), else the sustained figure
    power_capped = "sw_power_cap" in (clk.summary().get("reasons") or [])
    tf32_peak = tf32_sust if power_capped else tf32_burst
    tf32_peak_kind = "sustained (sw_power_cap seen in the timed region)" if power_capped else \
        "burst (no power cap in the timed region)"
    # the power products and Grams run 3xF16 on pre-split operands unless HG_GEMM_F16=0
    f16_gemms = os.environ.get("HG_GEMM_F16", "1") != "0" and c.b % 32 == 0
    apply_fused = "gemm_apply" in prof and round(prof["gemm_apply"][1] / args.steps) == 1
    # algorithmic work per launch
    nb, b, k, q, T = c.nb, c.b, c.k, c.q, c.T
    work = {
        "gemm_power": ("tensor", 2.0 * b * b * k * nb, 2 * q + 2),
        "gemm_gram": ("tensor", 2.0 * b * k * k * nb, 4 * q + 3),
        "gemm_qform": ("tensor", 2.0 * b * k * k * nb, 4 * q + 2),
        # the fused kernel (apply.cu: both products of Eq. 15 in one launch, 3xF16) or the two 3xTF32 GEMMs
        "gemm_apply": ("tensor", (4.0 if apply_fused else 2.0) * b * k * T * nb, 1 if apply_fused else 2),
        "assemble": ("hbm", 4.0 * b * b * nb, 1),
    }

    # CUDA-core fp32 peak for ALU-bound stages: 148 SMs x 128 FMA/clk x 2 flop x max SM clock
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    # one-sided Jacobi: per sweep k(k-1)/2 pairs x k rows x (3 dot FMA + 4 rotation ops) ~ 6 k^3 flop
    work["jacobi"] = ("alu", 6.0 * k ** 3 * sweeps_avg * nb, 1)
    # Cholesky k^3/3 + triangular inverse k^3/3 FMA per full factorization (first-order ones ~k^2)
    work["cholinv"] = ("alu", 2.0 * (2.0 / 3.0) * k ** 3 * chol_full_frac * nb, 4 * q + 3)
    # Jacobi preconditioner (eig.cu): Householder tridiagonalisation (4/3) k^3 + back-transform 2 k^3 flop
    # per block (the Sturm bisection and inverse iteration are O(k^2) per eigenvalue ... O(k^3) with a small
    # constant and are not counted)
    work["eig_precond"] = ("alu", (4.0 / 3.0 + 2.0) * k ** 3 * nb, 1)

    def roof(stage):
        if stage not in work or stage not in prof:
            return None
        bound, per_launch, _ = work[stage]
        if bound == "alu":
            total_ms, n = prof[stage]
            avg_s = total_ms / n / 1e3
            tf = per_launch / avg_s / 1e12
            return {"kernel": stage, "bound": "alu", "achieved": tf, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": tf / fp32_peak, "avg_launch_ms": avg_s * 1e3, "launches_per_step": n / args.steps,
                    "peak_note": "fp32 CUDA-core peak: 148 SM x 128 FMA/clk x 2 x sm_max_mhz (B200_PROFILING.md units)",
                    "work_note": {"jacobi": "6 k^3 flop per block per sweep, %.2f sweeps avg" % sweeps_avg,
                                  "cholinv": "(4/3) k^3 flop per full factorization, %.0f%% full" % (100 * chol_full_frac),
                                  "eig_precond": "(4/3) k^3 tridiagonalisation + 2 k^3 back-transform flop per block"}[stage],
                    "traffic": None}
        total_ms, n = prof[stage]
        avg_s = total_ms / n / 1e3
        if bound == "tensor":
            useful = per_launch / avg_s / 1e12
            achieved = 3.0 * useful          # 3xTF32 / 3xF16: three tensor products per fp32 product
            if (stage in F16_STAGES and f16_gemms) or (stage == "gemm_apply" and apply_fused):
                # kind::f16 (3xF16 pre-split operands): the fp16 dense peak = the measured bf16 one
                f16_burst, f16_sust = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
                f16_peak = f16_sust if power_capped else f16_burst
                return {"kernel": stage, "bound": "tensor", "precision": "3xF16 (kind::f16)", "achieved": achieved,
                        "peak": f16_peak, "unit": "TFLOP/s", "frac": achieved / f16_peak, "useful_fp32_tflops": useful,
                        "frac_vs_burst": achieved / f16_burst, "frac_vs_sustained": achieved / f16_sust,
                        "tf32_equivalent_frac": achieved / tf32_peak,
                        "peak_note": f"fp16 dense = bf16 dense {tf32_peak_kind.split(' ')[0]} from MEASURED_PEAKS.json "
                                     f"({peak_src}: cuBLAS bf16 8192^3); tf32_equivalent_frac = the same tensor work "
                                     f"against the tf32 peak ({tf32_src})",
                        "avg_launch_ms": avg_s * 1e3, "launches_per_step": n / args.steps, "traffic": None}
            return {"kernel": stage, "bound": "tensor", "precision": "3xTF32 (kind::tf32)", "achieved": achieved,
                    "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": achieved / tf32_peak, "useful_fp32_tflops": useful,
                    "frac_vs_burst": achieved / tf32_burst, "frac_vs_sustained": achieved / tf32_sust,
                    "peak_note": f"tf32 dense {tf32_peak_kind}; {tf32_src}",
                    "avg_launch_ms": avg_s * 1e3, "launches_per_step": n / args.steps, "traffic": None}
        gbs = per_launch / avg_s / 1e9
        return {"kernel": stage, "bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / peaks["hbm_gbs"], "avg_launch_ms": avg_s * 1e3, "traffic": None}

    dominant = max(stages, key=lambda s: stages[s]["ms_per_step"]) if stages else None
    traffic_file = os.path.join(HERE, "profiles", "traffic.json")
    traffic = json.load(open(traffic_file)) if os.path.exists(traffic_file) else {}
    gemm_roof = roof("gemm_power")
    if gemm_roof and "gemm_power" in traffic:
        gemm_roof["traffic"] = traffic["gemm_power"]
    # the fused Eq. 15 kernel: tensor work of both products, and its algorithmic HBM bytes (Y read + F written)
    apply_roof = roof("gemm_apply")
    if apply_roof:
        apply_roof["fused"] = bool(apply_fused)
        apply_roof["hbm_algorithmic_gbs"] = 2.0 * 4.0 * c.N * T / (apply_roof["avg_launch_ms"] / 1e3) / 1e9 * \
            (1.0 if apply_fused else 0.5)
        apply_roof["hbm_frac"] = apply_roof["hbm_algorithmic_gbs"] / peaks["hbm_gbs"]
    if apply_roof and traffic.get("gemm_apply") and apply_fused:
        apply_roof["traffic"] = traffic["gemm_apply"]
    dom_roof = roof(dominant) if dominant in work else None
    if dom_roof is None and dominant is not None:
        dom_roof = {"kernel": dominant, "bound": "alu", "achieved": None, "peak": None, "unit": None, "frac": None,
                    "note": "latency/ALU-bound SIMT stage; see DESIGN.md"}
    if dom_roof and dominant in traffic:
        dom_roof["traffic"] = traffic[dominant]
    gemm_useful_tflops = None
    if "gemm_power" in prof:
        gemm_useful_tflops = (2 * q + 2) * 2.0 * b * b * k * nb / (prof["gemm_power"][0] / args.steps / 1e3) / 1e12

    # Every use of the FP64 oracle below is deferred into the cpu_baseline leg (cpu_baseline_leg, run
    # once after all GPU timing on rank 0): the CPU baseline timing itself and the parity / accuracy
    # references of the timed outputs.  Nothing on the GPU path depends on it.
    leg = []
    result = {"parity": None, "cpu_baseline": None}

    def leg_main():
        r = oracle_sample(h, c, 2, seed=seed) if c.nb > 1 else oracle_sample(h, c, 1, seed=seed)
        assert list(r.blocks) == par_blocks, (r.blocks, par_blocks)

        def errs(Fblk, sblk):
            fe = max(float(np.linalg.norm(Fblk(blk) - r.F[s_ * c.b:(s_ + 1) * c.b]) /
                           np.linalg.norm(r.F[s_ * c.b:(s_ + 1) * c.b])) for s_, blk in enumerate(r.blocks))
            se = max(float(np.max(np.abs(sblk(blk) - r.sigma[s_]) / r.sigma[s_])) for s_, blk in enumerate(r.blocks))
            return fe, se

        # the outputs of the timed steps themselves (device entry, the `value` above)
        ferr, serr = errs(lambda blk: F_timed[blk], lambda blk: s_timed[blk])
        result["parity"] = {"blocks": r.blocks, "F_rel_fro": ferr, "sigma_rel_max": serr,
                            "tol": {"F": 2e-5, "sigma": 1e-5}, "ok": ferr <= 2e-5 and serr <= 1e-5,
                            "of": "outputs of the last timed step (hg_solve%s)" % ("_blocks + all-gather" if shard
                                                                                  else ""),
                            "status_timed_steps": timed_status}
        # the host entry's outputs (the e2e key)
        Fg = Fh.double().numpy()
        sg = sh.double().numpy()
        fe2, se2 = errs(lambda blk: Fg[blk * c.b:(blk + 1) * c.b], lambda blk: sg[blk])
        result["parity"]["host_entry"] = {"F_rel_fro": fe2, "sigma_rel_max": se2, "ok": fe2 <= 2e-5 and se2 <= 1e-5}
        if world == 1 and not args.no_cpu_baseline:
            nthreads = cores()
            n_s = max(1, min(c.nb, nthreads))
            rr = oracle_sample(h, c, n_s, seed=seed)
            cpu_base = {"value": n_s / rr.seconds, "unit": "blocks/s", "cores": rr.threads, "kind": "oracle",
                        "sample": f"{n_s} of {c.nb} diagonal blocks of the same workload (Alg. 1 + apply, FP64, "
                                  f"OpenMP over blocks), {rr.seconds:.1f} s",
                        "cpu_model": cpu_model()}
            # single-thread figure on one block (report 1 thread and all cores)
            import oracle
            oracle.set_num_threads(1)
            try:
                r1 = oracle_sample(h, c, 1, seed=seed)
                cpu_base["value_1thread"] = 1.0 / r1.seconds
            finally:
                oracle.set_num_threads(nthreads)
            result["cpu_baseline"] = cpu_base

    leg.append(leg_main)

    # the paper's second approach (CG on Eq. 5) on the
    # same workload, timed the same way (CUDA events, resident inputs), parity on sampled columns
    cg = None
    if not args.no_cg:
        cg_tol, cg_max = 1e-6, 100
        cws = hg.Workspace(hg.cg_workspace_size(c.N, h.E, h.nnz, c.T, cg_max), device=dev)
        Fc = torch.empty((c.N, c.T), dtype=torch.float32, device=dev)
        itc = torch.empty(c.T, dtype=torch.int32, device=dev)
        rrc = torch.empty(c.T, dtype=torch.float32, device=dev)

        def cg_step():
            hg.cg_solve(H, w, Y, mu=c.mu, max_iter=cg_max, tol=cg_tol, sync=False, ws=cws, F=Fc, iters=itc,
                        rel_res=rrc, status=status, stream=stream)

        for _ in range(3):
            cg_step()
        cg_launches = hg.last_launch_count()
        torch.cuda.synchronize(dev)
        n_cg = max(3, min(args.steps, 10))
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(n_cg):
            cg_step()
        c1.record(stream)
        torch.cuda.synchronize(dev)
        cg_ms = max_over_ranks(c0.elapsed_time(c1) / n_cg, dev)
        its = itc.cpu().numpy()
        n_it = int(its.max())
        ts = 128 if c.T > 64 else (64 if c.T > 32 else 32)
        t_pad = (c.T + ts - 1) // ts * ts
        gather = 2.0 * h.nnz * t_pad * 4 * n_it          # two sparse gathers of a T-row per incidence
        cg = {"workload": "same H, w, Y; X F = theta/(1+theta) Y, one CG per column, tol %g" % cg_tol,
              "solve_ms": cg_ms, "iterations_max": n_it, "iterations_mean": float(its.mean()),
              "rel_res_max": float(rrc.max().item()), "launches_per_solve": cg_launches,
              "gather_bytes_per_solve": gather, "gather_GBps": gather / (cg_ms / 1e3) / 1e9,
              "note": "gathers are L2-resident (slice-major layout); see DESIGN.md §10"}
        def leg_cg():
            import oracle
            cols = np.array([0, 1, c.T // 2, c.T - 1])
            ro = oracle.cg_solve(h.row_ptr, h.col_idx, h.w, np.ascontiguousarray(h.Y[:, cols]), mu=c.mu,
                                 max_iter=cg_max, tol=cg_tol)
            Fcg = Fc[:, torch.from_numpy(cols).to(dev)].double().cpu().numpy()
            cg["parity"] = {"columns": cols.tolist(), "F_rel_fro": float(np.linalg.norm(Fcg - ro.F) /
                                                                        np.linalg.norm(ro.F)), "tol": 2e-5}
            cg["parity"]["ok"] = cg["parity"]["F_rel_fro"] <= 2e-5
            # accuracy of the block rSVD output against the full solve (SURVEY.md §8(d) accuracy axis)
            Fr = Fh.double().numpy()
            Ff = Fc.double().cpu().numpy()
            cg["rsvd_F_vs_full_solve_rel_fro"] = float(np.linalg.norm(Fr - Ff) / np.linalg.norm(Ff))
            cg["oracle_columns_s"] = ro.seconds

        leg.append(leg_cg)

    # SURVEY.md §8(f) NEXT-3, reading R2: Alg. 1 on Theta_ii + the Woodbury inverse of X_ii, same
    # workload and timing; parity on sampled blocks; accuracy against the exact block solve and CG
    r2 = None
    if not args.no_r2:
        F2 = torch.empty((c.N, c.T), dtype=torch.float32, device=dev)
        s2 = torch.empty((c.nb, c.k), dtype=torch.float32, device=dev)

        def r2_step():
            hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, sync=False, woodbury=True, ws=ws, F=F2,
                     sigma=s2, status=status, stream=stream)

        for _ in range(3):
            r2_step()
        torch.cuda.synchronize(dev)
        n_r2 = max(3, min(args.steps, 10))
        r0_, r1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0_.record(stream)
        for _ in range(n_r2):
            r2_step()
        r1_.record(stream)
        torch.cuda.synchronize(dev)
        r2_ms = max_over_ranks(r0_.elapsed_time(r1_) / n_r2, dev)
        r2 = {"workload": "same H, w, Y, b, k, q; Alg. 1 on Theta_ii, F_i = c (Y_i + U diag(s/((1+mu)-s)) U^T Y_i)",
              "solve_ms": r2_ms, "blocks_per_s": world * c.nb / (r2_ms / 1e3),
              "status": int(status.item())}
        def leg_r2():
            import oracle
            ro2 = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed,
                               blocks=[0, c.nb - 1], woodbury=True)
            Fg2 = F2.double().cpu().numpy()
            sg2 = s2.double().cpu().numpy()
            fe, se, ex_r1, ex_r2 = 0.0, 0.0, 0.0, 0.0
            Fr1 = Fh.double().numpy()
            for s_, blk in enumerate(ro2.blocks):
                rows = slice(blk * c.b, (blk + 1) * c.b)
                fo = ro2.F[s_ * c.b:(s_ + 1) * c.b]
                fe = max(fe, float(np.linalg.norm(Fg2[rows] - fo) / np.linalg.norm(fo)))
                se = max(se, float(np.max(np.abs(sg2[blk] - ro2.sigma[s_]) / ro2.sigma[s_])))
                Xo = oracle.theta_block(h.row_ptr, h.col_idx, h.w, c.b, blk, mu=c.mu)
                ex = c.mu / (1 + c.mu) * np.linalg.solve(Xo, h.Y[rows].astype(np.float64))
                ex_r2 = max(ex_r2, float(np.linalg.norm(Fg2[rows] - ex) / np.linalg.norm(ex)))
                ex_r1 = max(ex_r1, float(np.linalg.norm(Fr1[rows] - ex) / np.linalg.norm(ex)))
            r2["parity"] = {"blocks": ro2.blocks, "F_rel_fro": fe, "sigma_rel_max": se, "tol": {"F": 2e-5, "sigma": 1e-5},
                            "ok": fe <= 2e-5 and se <= 1e-5}
            r2["accuracy_vs_exact_block_solve"] = {"r2": ex_r2, "r1": ex_r1, "blocks": ro2.blocks}
            if cg is not None:
                Ff = Fc.double().cpu().numpy()
                r2["accuracy_vs_full_solve"] = {"r2": float(np.linalg.norm(Fg2 - Ff) / np.linalg.norm(Ff)),
                                                "r1": float(np.linalg.norm(Fr1 - Ff) / np.linalg.norm(Ff))}

        leg.append(leg_r2)

    # Variant (opt-in, NOT the headline): HG_QR_SKIP_HALF=1 leaves the half-step basis S~ = qr(X^T S) of Alg. 1
    # un-orthonormalised (Eq. 10 inside one iteration, Alg. 1's QR once per iteration) -- the
    # same subspace, so the same F and sigma to rounding; reported next to the literal Alg. 1 of `value`
    qrv = None
    if not args.no_r2:
        Fv = torch.empty((c.N, c.T), dtype=torch.float32, device=dev)
        sv = torch.empty((c.nb, c.k), dtype=torch.float32, device=dev)
        os.environ["HG_QR_SKIP_HALF"] = "1"

        def qrv_step():
            hg.solve(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, sync=False, ws=ws, F=Fv, sigma=sv,
                     status=status, stream=stream)

        for _ in range(3):
            qrv_step()
        torch.cuda.synchronize(dev)
        n_v = max(3, min(args.steps, 10))
        v0_, v1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0_.record(stream)
        for _ in range(n_v):
            qrv_step()
        v1_.record(stream)
        torch.cuda.synchronize(dev)
        os.environ.pop("HG_QR_SKIP_HALF")
        qrv_ms = max_over_ranks(v0_.elapsed_time(v1_) / n_v, dev)
        qrv = {"workload": "the bench workload with HG_QR_SKIP_HALF=1: one QR per power iteration (after X S~) "
                           "instead of Alg. 1's two; opt-in, not the headline",
               "solve_ms": qrv_ms, "blocks_per_s": world * c.nb / (qrv_ms / 1e3), "status": int(status.item()),
               "F_vs_alg1_gpu_rel_fro": float(((Fv - F).norm() / F.norm()).item()) if not shard else None}

        def leg_qrv():
            import oracle
            rov = oracle.solve(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed,
                               blocks=[0, c.nb - 1])
            Fgv, sgv = Fv.double().cpu().numpy(), sv.double().cpu().numpy()
            fe, se = 0.0, 0.0
            for s_, blk in enumerate(rov.blocks):
                rows = slice(blk * c.b, (blk + 1) * c.b)
                fo = rov.F[s_ * c.b:(s_ + 1) * c.b]
                fe = max(fe, float(np.linalg.norm(Fgv[rows] - fo) / np.linalg.norm(fo)))
                se = max(se, float(np.max(np.abs(sgv[blk] - rov.sigma[s_]) / rov.sigma[s_])))
            qrv["parity"] = {"blocks": rov.blocks, "F_rel_fro": fe, "sigma_rel_max": se,
                             "tol": {"F": 2e-5, "sigma": 1e-5}, "ok": fe <= 2e-5 and se <= 1e-5,
                             "of": "against the oracle's literal Alg. 1"}

        if not shard:
            leg.append(leg_qrv)

    # one Eq. 12 Schur level over pairs of adjacent blocks (reading R2 inverses)
    sch = None
    if not args.no_schur and c.nb % 2 == 0:
        sws = hg.Workspace(hg.schur_workspace_size(c.N, h.E, h.nnz, c.b, c.k, c.T), device=dev)
        Fs = torch.empty((c.N, c.T), dtype=torch.float32, device=dev)
        for _ in range(2):
            hg.solve_schur(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, sync=False, ws=sws, F=Fs, status=status,
                           stream=stream)
        sch_launches = hg.last_launch_count()
        torch.cuda.synchronize(dev)
        n_s = max(3, min(args.steps, 5))
        h0_, h1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0_.record(stream)
        for _ in range(n_s):
            hg.solve_schur(H, w, Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed, sync=False, ws=sws, F=Fs, status=status,
                           stream=stream)
        h1_.record(stream)
        torch.cuda.synchronize(dev)
        sch_ms = max_over_ranks(h0_.elapsed_time(h1_) / n_s, dev)
        sch = {"workload": "same H, w, Y, b, k, q; one Eq. 12 level over super-blocks (2s, 2s+1) of 2b, "
                           "X11^-1, X22^-1, Z1^-1, Z2^-1 by Alg. 1 + Woodbury (reading R2)",
               "solve_ms": sch_ms, "launches_per_solve": sch_launches, "status": int(status.item())}
        del sws
        def leg_schur():
            import oracle
            Fo, sel, osec = oracle.solve_schur(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, k=c.k, q=c.q, seed=seed,
                                               superblocks=[0])
            Fsg = Fs.double().cpu().numpy()
            rows = slice(0, 2 * c.b)
            pe = float(np.linalg.norm(Fsg[rows] - Fo) / np.linalg.norm(Fo))
            sch["parity"] = {"superblocks": sel, "F_rel_fro": pe, "tol": 2e-5, "ok": pe <= 2e-5}
            Xs = oracle.theta_block(h.row_ptr, h.col_idx, h.w, 2 * c.b, 0, mu=c.mu)
            ex = c.mu / (1 + c.mu) * np.linalg.solve(Xs, h.Y[rows].astype(np.float64))
            sch["accuracy_vs_exact_superblock_solve"] = float(np.linalg.norm(Fsg[rows] - ex) / np.linalg.norm(ex))
            if cg is not None:
                Ff = Fc.double().cpu().numpy()
                sch["accuracy_vs_full_solve"] = float(np.linalg.norm(Fsg - Ff) / np.linalg.norm(Ff))
            sch["oracle_superblock_s"] = osec

        leg.append(leg_schur)

    # the nested tessellation -- Eq. 12 recursively inside 2^L b super-blocks
    nst = None
    L_n = args.nested_levels
    if (L_n > 0 and c.N % (c.b << L_n) == 0 and (c.k << (L_n - 1)) <= 512 and c.T % 4 == 0):
        nws = hg.Workspace(hg.nested_workspace_size(c.N, h.E, h.nnz, c.b, L_n, c.k, c.T), device=dev)
        Fn = torch.empty((c.N, c.T), dtype=torch.float32, device=dev)
        for _ in range(2):
            hg.solve_nested(H, w, Y, mu=c.mu, b=c.b, levels=L_n, k=c.k, q=c.q, seed=seed, sync=False, ws=nws, F=Fn,
                            status=status, stream=stream)
        nst_launches = hg.last_launch_count()
        torch.cuda.synchronize(dev)
        n_n = max(3, min(args.steps, 5))
        n0_, n1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0_.record(stream)
        for _ in range(n_n):
            hg.solve_nested(H, w, Y, mu=c.mu, b=c.b, levels=L_n, k=c.k, q=c.q, seed=seed, sync=False, ws=nws, F=Fn,
                            status=status, stream=stream)
        n1_.record(stream)
        torch.cuda.synchronize(dev)
        nst = {"workload": f"same H, w, Y, b, k, q; Eq. 12 applied recursively over {c.N // (c.b << L_n)} super-blocks "
                           f"of 2^{L_n} b = {c.b << L_n}, level-l Schur rank k 2^(l-1) (readings S4, S5)",
               "levels": L_n, "solve_ms": max_over_ranks(n0_.elapsed_time(n1_) / n_n, dev),
               "launches_per_solve": nst_launches, "status": int(status.item())}
        del nws
        def leg_nested():
            import oracle
            m = c.b << L_n
            Fng = Fn.double().cpu().numpy()
            if args.nested_parity:   # the FP64 oracle of one 2^L b super-block: minutes at configs[3]
                Fo, sel, osec = oracle.solve_nested(h.row_ptr, h.col_idx, h.w, h.Y, mu=c.mu, b=c.b, levels=L_n,
                                                    k=c.k, q=c.q, seed=seed, superblocks=[0])
                pe = float(np.linalg.norm(Fng[:m] - Fo) / np.linalg.norm(Fo))
                nst["parity"] = {"superblocks": sel, "F_rel_fro": pe, "tol": 2e-5, "ok": pe <= 2e-5}
                nst["oracle_superblock_s"] = osec
            else:
                nst["parity"] = "tests/test_gpu_nested.py (configs[0]/[1] vs the oracle); --nested-parity for this config"
            Xs = oracle.theta_block(h.row_ptr, h.col_idx, h.w, m, 0, mu=c.mu)
            ex = c.mu / (1 + c.mu) * np.linalg.solve(Xs, h.Y[:m].astype(np.float64))
            nst["accuracy_vs_exact_superblock_solve"] = float(np.linalg.norm(Fng[:m] - ex) / np.linalg.norm(ex))
            if cg is not None:
                Ff = Fc.double().cpu().numpy()
                nst["accuracy_vs_full_solve"] = float(np.linalg.norm(Fng - Ff) / np.linalg.norm(Ff))

        leg.append(leg_nested)

    # the hyperedge-weight update with f = the CG solution
    wts = None
    if cg is not None and not args.no_weights:
        kappa = 1.0
        wg = torch.empty(h.E, dtype=torch.float32, device=dev)
        for _ in range(3):
            hg.weight_gradient(H, w, Fc, kappa=kappa, ws=cws, grad=wg, status=status, stream=stream)
        torch.cuda.synchronize(dev)
        n_w = max(3, min(args.steps, 10))
        w0_, w1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0_.record(stream)
        for _ in range(n_w):
            hg.weight_gradient(H, w, Fc, kappa=kappa, ws=cws, grad=wg, status=status, stream=stream)
        w1_.record(stream)
        torch.cuda.synchronize(dev)
        g_ms = w0_.elapsed_time(w1_) / n_w
        ws_ = (w / w.sum()).contiguous()
        act = torch.zeros(h.E, dtype=torch.int32, device=dev)
        s0_, s1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0_.record(stream)
        for _ in range(n_w):
            hg.weight_step(ws_, act, wg, 1e-9, status=status, stream=stream)
        s1_.record(stream)
        torch.cuda.synchronize(dev)
        st_ms = s0_.elapsed_time(s1_) / n_w
        gather = h.nnz * c.T * 4.0
        wts = {"workload": "grad_e of P(w) = sum_t f_t^T L f_t + kappa||w||^2 at F = the CG solution, kappa 1; "
                           "one simplex step",
               "gradient_ms": g_ms, "step_ms": st_ms, "gather_bytes": gather,
               "gather_GBps": gather / (g_ms / 1e3) / 1e9, "status": int(status.item())}
        def leg_weights():
            import oracle
            go = oracle.weight_gradient(h.row_ptr, h.col_idx, h.w, Fc.double().cpu().numpy(), kappa=kappa)
            gg = wg.double().cpu().numpy()
            err = float(np.max(np.abs(gg - go)) / np.max(np.abs(go)))
            wts["parity"] = {"grad_max_rel": err, "tol": 1e-5, "ok": err <= 1e-5}

        leg.append(leg_weights)

    def cpu_baseline_leg():
        """The oracle (FP64 CPU), run once on rank 0 after all GPU timing: baseline + parity references."""
        for task in leg:
            task()

    if rank == 0:
        cpu_baseline_leg()
    parity, cpu_base = result["parity"], result["cpu_baseline"]

    out = {
        "metric": "diag_blocks_per_s", "value": value, "unit": "blocks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_json(c),
        "solve_ms": ms, "blocks_per_s_per_gpu": c.nb / (ms / 1e3),
        "gemm_useful_tflops": gemm_useful_tflops,
        "gemm_tf32_pipe_frac": gemm_roof["frac"] if gemm_roof else None,
        "roofline": dom_roof, "gemm_roofline": gemm_roof, "apply_roofline": apply_roof,
        "stages": stages, "profiled_ms_per_step": prof_ms_per_step,
        "jacobi_sweeps_avg": sweeps_avg, "jacobi_sweeps_max": dbg["jacobi_max_sweeps"],
        "e2e": {"value": (c.nb if shard else world * c.nb) / (e2e_ms / 1e3), "unit": "blocks/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "entry": "hg_solve_blocks + all-gather (pinned copies)" if shard else "hg_solve_host"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "parity": parity,
        "cpu_baseline": cpu_base,
        "next_rows": {"cg": cg, "r2_woodbury": r2, "schur": sch, "nested": nst, "weights": wts,
                      "qr_once_per_iteration": qrv},
        "peaks": {"source": peak_src, "tf32_tflops_sustained": tf32_sust, "tf32_tflops_burst": tf32_burst,
                  "tf32_source": tf32_src, "tf32_denominator": tf32_peak_kind,
                  "tf32_measured": tf32_meas, "hbm_gbs": peaks["hbm_gbs"]},
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm (the oracle)
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from synth.hypergraph import make_input
    c = workload_config(args)
    h = make_input(c)
    nthreads = cores()
    n_s = max(1, min(c.nb, nthreads))
    for _ in range(args.warmup):
        oracle_sample(h, c, n_s)
    times = []
    for _ in range(args.steps):
        r = oracle_sample(h, c, n_s)
        times.append(r.seconds)
    t = sum(times) / len(times)
    v = n_s / t
    out = {"impl": "reference", "metric": "diag_blocks_per_s", "value": v, "unit": "blocks/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_json(c, note="reference arm = FP64 CPU oracle (no reference implementation exists)"),
           "cpu_baseline": {"value": v, "unit": "blocks/s", "cores": r.threads, "kind": "oracle",
                            "sample": f"{n_s} of {c.nb} diagonal blocks per step (Alg. 1 + apply, FP64, OpenMP)",
                            "cpu_model": cpu_model()},
           "e2e": {"value": v, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--b", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cg", action="store_true", help="skip the CG (NEXT-2) measurement")
    ap.add_argument("--no-r2", action="store_true", help="skip the reading-R2 (NEXT-3) measurement")
    ap.add_argument("--no-weights", action="store_true", help="skip the weight-update (NEXT-4) measurement")
    ap.add_argument("--no-schur", action="store_true", help="skip the Schur-complement (NEXT-1) measurement")
    ap.add_argument("--nested-levels", type=int, default=2,
                    help="levels of the nested-tessellation (NEXT-1) measurement; 0 skips it")
    ap.add_argument("--nested-parity", action="store_true",
                    help="check the nested row against the FP64 oracle on super-block 0 (about 6 min at configs[3])")
    ap.add_argument("--independent", action="store_true",
                    help="N > 1: an independent problem per rank (weak scaling) instead of the default ONE "
                         "problem sharded by block ranges over the ranks + an all-gather of F (strong scaling)")
    ap.add_argument("--shard", action="store_true", help="(default for N > 1; kept for compatibility)")
    ap.add_argument("--no-tf32-peak", action="store_true",
                    help="skip the live TF32 peak measurement (derive it from MEASURED_PEAKS bf16)")
    ap.add_argument("--selftest-dist", action="store_true",
                    help="CPU/gloo self-test of the multi-rank harness (spawn, shard ranges, all-gather, "
                         "max over ranks); no GPU kernels")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not launched by torchrun: spawn the N ranks ourselves (one process per GPU), same arguments
        return spawn_ranks(args.gpus, sys.argv[1:] if argv is None else list(argv))
    if args.selftest_dist:
        return selftest_dist(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
