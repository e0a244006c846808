"""Multi-process host logic of bench.py on CPU (gloo, world size 2): rank setup,
barrier, max-over-ranks timing, and the reference arm's rank-0-only rule."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import bench
    import torch.distributed as dist
    r, w, lr = bench.dist_setup("gloo")
    bench.barrier()
    # per-rank step times: the reported time is the slowest rank's
    m = bench.max_over_ranks(10.0 + 5.0 * r)
    q.put((r, w, lr, m))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [x[0] for x in res] == [0, 1]
    assert all(x[1] == 2 for x in res)
    assert all(abs(x[3] - 15.0) < 1e-12 for x in res)


def test_single_process_needs_no_process_group(monkeypatch):
    import bench
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert bench.dist_setup("gloo") == (0, 1, 0)
    assert bench.max_over_ranks(3.25) == 3.25


def test_reference_arm_is_rank0_only(monkeypatch, capsys):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    bench.main(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3"])
    assert capsys.readouterr().out == ""


def test_reference_arm_json_line(monkeypatch, capsys):
    import json
    import bench
    monkeypatch.delenv("RANK", raising=False)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    bench.main(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3"])
    line = json.loads(capsys.readouterr().out.strip())
    assert line["impl"] == "reference" and line["unit"] == "blocks/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


def _shard_worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import bench
    import torch.distributed as dist
    bench.dist_setup("gloo")
    nb, b, T = 7, 4, 3
    b0, cnt = bench.shard_range(nb, rank, world)
    # each rank fills only its blocks' rows of F (as hg_solve_blocks does); the all-gather assembles F
    F = torch.zeros(nb * b, T)
    F[b0 * b:(b0 + cnt) * b] = torch.arange(b0 * b * T, (b0 + cnt) * b * T, dtype=torch.float32).reshape(-1, T)
    full = bench.allgather_rows(F, b0 * b, cnt * b, world)
    q.put((rank, b0, cnt, full.numpy().tolist()))
    dist.destroy_process_group()


def test_sharded_blocks_and_allgather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    # disjoint contiguous ranges covering every block
    assert [(x[1], x[2]) for x in res] == [(0, 3), (3, 4)]
    import numpy as np
    want = np.arange(7 * 4 * 3, dtype=np.float32).reshape(-1, 3)
    for x in res:
        assert np.array_equal(np.array(x[3], np.float32), want)


def test_bench_gpus2_spawns_ranks_and_shards_gloo(monkeypatch, capfd):
    """`bench.py --gpus 2` without torchrun spawns its two ranks itself (torch.distributed.run on
    127.0.0.1); the harness self-test shards configs[0]'s blocks, all-gathers F and sigma over gloo
    and reports the max over ranks."""
    import json
    import bench
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        monkeypatch.delenv(k, raising=False)
    rc = bench.main(["--gpus", "2", "--selftest-dist", "--config", "2"])
    out = capfd.readouterr().out
    assert rc == 0, out
    line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
    assert line["selftest"] == "dist" and line["ok"] and line["n_gpus"] == 2
    assert line["shards"] == [[0, 8], [8, 8]] and line["ms_per_step_max"] == 2.0


def test_allgather_uneven_and_inplace_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uneven_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(3)]
    assert all(r[1] for r in res), res


def _uneven_worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import bench
    import torch.distributed as dist
    bench.dist_setup("gloo")
    ok = True
    for nb in (7, 6):   # uneven shares (padded path) and equal shares (all_gather_into_tensor)
        b, T = 2, 3
        b0, cnt = bench.shard_range(nb, rank, world)
        F = torch.full((nb * b, T), -1.0)
        F[b0 * b:(b0 + cnt) * b] = rank
        out = torch.empty_like(F)
        bench.allgather_rows(F, b0 * b, cnt * b, world, counts=bench.shard_rows(nb, b, world), out=out)
        want = torch.cat([torch.full((bench.shard_range(nb, r, world)[1] * b, T), float(r)) for r in range(world)])
        ok &= bool(torch.equal(out, want))
    q.put((rank, ok))
    dist.destroy_process_group()
