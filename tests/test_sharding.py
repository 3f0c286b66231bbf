"""Multi-GPU host logic on CPU: LPT sharding of independent images and the
bench's barrier + max-over-ranks timing, exercised with world_size 2 over gloo.
(The data path itself has no collective: each rank owns whole images.)"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parent.parent

from paper_2603_16987_b200.sharding import image_costs, imbalance, lpt_assign, shard  # noqa: E402
from paper_2603_16987_b200.workloads import c4_shapes  # noqa: E402


def test_lpt_partitions_and_balances():
    rng = np.random.default_rng(0)
    costs = rng.integers(1, 100, size=257).astype(float)
    for k in (1, 2, 3, 8):
        parts = lpt_assign(costs, k)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(257))
        loads = [costs[p].sum() for p in parts]
        # LPT bound: max load <= 4/3 OPT; OPT >= mean and >= max item
        opt_lb = max(costs.sum() / k, costs.max())
        assert max(loads) <= 4.0 / 3.0 * opt_lb + 1e-9
    with pytest.raises(ValueError):
        lpt_assign(costs, 0)


def test_c4_shards_are_balanced():
    wh = c4_shapes(512)
    for world in (2, 4, 8):
        assert imbalance(wh, 448, 12, world) < 1.02
        parts = [shard(wh, 448, 12, r, world) for r in range(world)]
        assert sorted(np.concatenate(parts).tolist()) == list(range(512))
    costs = image_costs(wh, 448, 12)
    assert costs.max() / costs.min() > 3  # 13-tile vs 3-tile images: why LPT matters


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(REPO))
    import bench  # the bench's own distributed helper

    d = bench.Dist()
    d.init("gloo")
    wh = c4_shapes(300, start=100)
    mine = shard(wh, 448, 12, rank, world)
    # what each rank would process, gathered here only to check the partition
    sizes = [None] * world
    dist.all_gather_object(sizes, mine.tolist())
    d.barrier()
    t = d.max(float(10 + rank), torch.device("cpu"))
    q.put((rank, sizes, t))
    d.close()


def test_two_rank_gloo_sharding_and_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sizes, t in out:
        assert t == 11.0  # max over ranks
        flat = sorted(i for part in sizes for i in part)
        assert flat == list(range(300))
        assert not set(sizes[0]) & set(sizes[1])


def test_shared_gpu_dryrun_maps_ranks_and_tags_lines(monkeypatch):
    """TP_BENCH_SHARED_GPU_DRYRUN: ranks fold onto the devices present, the barrier backend
    is gloo and every JSON line says it is not a scaling number."""
    sys.path.insert(0, str(REPO))
    import bench

    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("LOCAL_RANK", "3")
    monkeypatch.setenv("TP_BENCH_SHARED_GPU_DRYRUN", "1")
    d = bench.Dist()
    assert d.device_index(1) == 0 and d.device_index(2) == 1
    assert "dryrun" in d.tag({"value": 1.0})
    monkeypatch.delenv("TP_BENCH_SHARED_GPU_DRYRUN")
    d = bench.Dist()
    assert d.device_index(8) == 3
    assert "dryrun" not in d.tag({"value": 1.0})


def test_bench_cpu_baselines_on_a_tiny_workload():
    """bench.py's cpu_baseline helpers (batch-1 latency and the per-core pool, with and
    without the C5 prompt leg) return well-formed objects; sizes kept tiny for the CPU suite."""
    sys.path.insert(0, str(REPO))
    import bench
    from paper_2603_16987_b200.workloads import IMAGENET_MEAN, IMAGENET_STD, Workload, c5_texts

    wl = Workload("T", "tiny", np.array([[96, 64], [64, 96]], np.int32), 32, 6,
                  IMAGENET_MEAN, IMAGENET_STD, True, 7)
    lat = bench.cpu_latency(wl, runs=2)
    assert lat["cores"] == 1 and lat["kind"] in ("port", "reference") and lat["value"] > 0
    assert lat["p99_ms"] >= lat["p50_ms"] > 0
    thr = bench.cpu_throughput_wl(wl, 2, 0.01, c5_texts(2, 7))
    assert thr["cores"] == 2 and thr["value"] > 0 and "prompts" in thr["sample"]


def test_bench_gpus_flag_spawns_ranks_under_torchrun():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run
    with 2 ranks (the reference arm needs no GPU): rank 0 prints the one JSON line with
    n_gpus 2, rank 1 exits 0 without work."""
    import json
    import subprocess

    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "1", "--batch", "2"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["config"]["images_per_gpu"] == 2 and lines[0]["value"] > 0


def test_bench_rejects_world_size_mismatch(monkeypatch):
    sys.path.insert(0, str(REPO))
    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    args = bench.parse_args(["--gpus", "4"])
    with pytest.raises(SystemExit, match="WORLD_SIZE"):
        bench.maybe_spawn(args, ["--gpus", "4"])
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.maybe_spawn(bench.parse_args([]), []) is None
