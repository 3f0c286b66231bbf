#!/usr/bin/env python3
"""Benchmark of the B200 VLM preprocessing hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch: K1 (plan) + K2 (fused
resample/crop/thumbnail/normalize -> bf16 NCHW) over BASELINE configs[1]
(C2: 64 synthetic 1920x1080 RGB images, InternVL3-2B tiling, E=448, max 12 +
thumbnail, ImageNet mean/std).  Inputs (398 MB) are larger than L2 (126 MB).
Under torchrun each rank runs its own 64-image batch on its own GPU (weak
scaling, no data-path collective); the barrier + max-over-ranks timing are
the only cross-rank operations.

`--impl reference` times the reference algorithm on the host cores (the
oracle port of vlmfp's fused/contiguous path, oracle/tileprep_oracle.py) on a
bounded sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "preprocessed images/sec and p50 per-image preprocess latency (ms); % of HBM roofline"
UNIT = "images/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=64, help="images per GPU per step (C2: 64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--latency-iters", type=int, default=300)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = False

    def init(self, backend: str):
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = True

    def barrier(self, device=None):
        if self.pg:
            import torch.distributed as dist

            if device is not None:
                dist.barrier(device_ids=[device.index])
            else:
                dist.barrier()

    def max(self, value: float, device) -> float:
        if not self.pg:
            return value
        import torch
        import torch.distributed as dist

        t = torch.tensor([value], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            import torch.distributed as dist

            dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def start(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def stop(self) -> dict:
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm on host cores (oracle port)

def _cpu_one(args):
    seed, k, w, h = args
    from oracle import tileprep_oracle as O
    from paper_2603_16987_b200.workloads import IMAGENET_MEAN, IMAGENET_STD

    arr = O.synth_image(seed, k, w, h, 3, 0)
    t0 = time.perf_counter()
    O.preprocess_image(arr, 448, 12, IMAGENET_MEAN, IMAGENET_STD, True)
    return time.perf_counter() - t0


def cpu_throughput(n_images: int, cores: int, seed: int = 20260817):
    """images/s of the oracle path over a pool of `cores` processes; inputs are
    generated inside the workers before their timed region."""
    import multiprocessing as mp

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    jobs = [(seed, k, 1920, 1080) for k in range(n_images)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_one, jobs[:cores])  # warm the workers
        t0 = time.perf_counter()
        per = pool.map(_cpu_one, jobs)
        wall = time.perf_counter() - t0
    return n_images / wall, float(np.median(per)) * 1e3, wall


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run_reference(args, dist: Dist):
    """--impl reference: the oracle port on host cores, rank 0 only."""
    if dist.rank != 0:
        return
    cores = host_cores()
    sample = max(cores, 8)
    _, p50_ms, _ = cpu_throughput(cores, cores)  # calibration/warm pool
    for _ in range(args.warmup):
        pass  # warm-up happens inside cpu_throughput (one image per worker)
    times = []
    for _ in range(args.steps):
        ips, p50_ms, wall = cpu_throughput(sample, cores)
        times.append(wall)
    wall = float(np.sum(times))
    value = sample * args.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8->bf16 (fp64 resample)",
        "data": "synthetic",
        "config": {"workload": "C2 sample: 1920x1080 RGB uint8, E=448, max 12 + thumb, "
                               "ImageNet mean/std, bf16 out", "images_per_step": sample},
        "p50_ms": round(p50_ms, 3),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                         "kind": "port",
                         "sample": f"{sample} images x {args.steps} steps, oracle/tileprep_oracle "
                                   "(numpy restatement of vlmfp fused path), "
                                   "multiprocessing pool"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side

def main():
    args = parse_args()
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
        return

    import torch

    from paper_2603_16987_b200 import _lib
    from paper_2603_16987_b200.engine import TilePreprocessor, empty_packed, synth_packed
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.workloads import c2, workload_bytes

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(dist.local_rank)
    device = torch.device("cuda", dist.local_rank)
    dist.init("nccl")

    wl = c2(args.batch)
    cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                           std=wl.std, reduced_precision_normalize=wl.bf16)
    stream = torch.cuda.Stream(device)
    seed = wl.seed + 1_000_003 * dist.rank
    images = synth_packed(wl.wh, 3, device, seed=seed, kind=0)
    prep = TilePreprocessor(cfg, device)
    n = images.n
    out = prep(images)  # allocates outputs at the upper bound
    torch.cuda.synchronize(device)
    n_tiles = out.num_tiles()

    wb = workload_bytes(wl)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(i=None):
        prep.plan(images, out.plans, stream)
        if i is not None:
            ev[i][0].record(stream)
        prep.tile(images, out.plans, out.pixel_values, None, stream)
        if i is not None:
            ev[i][1].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
    torch.cuda.synchronize(device)
    clocks = ClockSampler(dist.local_rank)
    clocks.start()
    dist.barrier(device)
    torch.cuda.synchronize(device)
    start.record(stream)
    for i in range(args.steps):
        step(i)
    stop.record(stream)
    torch.cuda.synchronize(device)
    dist.barrier(device)
    clk = clocks.stop()
    ms_local = start.elapsed_time(stop)
    ms = dist.max(ms_local, device)
    k2_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    ms_step = ms / args.steps
    value = dist.world * n * args.steps / (ms / 1e3)

    # ---- end to end through the public API with host buffers ----------------
    host = empty_packed(wl.wh, 3, "cpu", pin=True)
    host.data.copy_(images.data.cpu())
    host.offsets.copy_(images.offsets.cpu())
    host.wh.copy_(images.wh.cpu())
    plan_host = torch.empty_like(out.plans.plan, device="cpu").pin_memory()
    off_host = torch.empty_like(out.plans.tile_off, device="cpu").pin_memory()
    e2e_steps = max(5, min(args.steps, 30))

    def e2e_step():
        images.copy_from_(host, non_blocking=True)
        prep(images, out=out, stream=stream)
        plan_host.copy_(out.plans.plan, non_blocking=True)
        off_host.copy_(out.plans.tile_off, non_blocking=True)

    with torch.cuda.stream(stream):
        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize(device)
        dist.barrier(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(device)
    e2e_ms = dist.max(e0.elapsed_time(e1), device) / e2e_steps
    h2d = host.nbytes() + host.offsets.numel() * 8 + host.wh.numel() * 4
    d2h = plan_host.numel() * 4 + off_host.numel() * 4

    # ---- batch-1 per-image latency (1 x 1080p, device resident, CUDA graph) --
    latency = None
    if dist.rank == 0:
        latency = batch1_latency(cfg, device, args.latency_iters)

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        # calibrate: ~`cpu-seconds` of total CPU work
        _, p50_ms, _ = cpu_throughput(cores, cores)
        n_cpu = int(max(cores, min(256, args.cpu_seconds * 1e3 / max(p50_ms, 1.0))))
        ips, p50_ms, wall = cpu_throughput(n_cpu, cores)
        cpu = {"value": round(ips, 3), "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n_cpu} C2 images (1920x1080) through oracle/tileprep_oracle "
                         f"(numpy restatement of vlmfp fused path) in a {cores}-process pool, "
                         f"{wall:.1f} s wall; per-image p50 {p50_ms:.1f} ms"}

    if dist.rank == 0:
        bytes_per_launch = wb["total"]
        achieved = bytes_per_launch / (k2_ms / 1e3) / 1e9
        peak = measured_peak()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 in, fp64 resample, bf16 out", "data": "synthetic",
            "config": {"workload": "C2: " + wl.description, "images_per_gpu": n,
                       "tiles_per_gpu": n_tiles, "l2": "inputs (398 MB/GPU) larger than L2",
                       "parallelism": f"dp{dist.world} (independent images, no collective)"},
            "p50_ms": latency["p50_ms"] if latency else None,
            "latency": latency,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak[0],
                         "unit": "GB/s", "frac": round(achieved / peak[0], 4),
                         "traffic": None, "peak_source": peak[1],
                         "kernel": "tp_tile (K2)", "kernel_ms": round(k2_ms, 4),
                         "bytes_per_launch": bytes_per_launch},
            "cpu_baseline": cpu,
            "e2e": {"value": round(dist.world * n / (e2e_ms / 1e3), 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_ms, 4),
                    "path": "pinned host images -> H2D -> TilePreprocessor (K1+K2) -> "
                            "D2H plans/offsets"},
            "gpu_launches": 2 * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.close()


def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"


def batch1_latency(cfg, device, iters: int):
    """p50/p99 of one 1920x1080 image through K1+K2 (device-resident input,
    CUDA-graph launched), plus the same with the 6.2 MB H2D from pinned host."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor, empty_packed, synth_packed

    wh = np.array([[1920, 1080]], dtype=np.int32)
    img = synth_packed(wh, 3, device, seed=7, kind=0)
    prep = TilePreprocessor(cfg, device)
    out = prep(img)
    s = torch.cuda.Stream(device)
    torch.cuda.synchronize(device)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prep(img, out=out, stream=torch.cuda.current_stream(device))
    host = empty_packed(wh, 3, "cpu", pin=True)
    host.data.copy_(img.data.cpu())

    def timed(fn):
        ts = []
        for _ in range(iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                fn()
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ts = np.array(ts[max(3, iters // 10):])
        return float(np.percentile(ts, 50)), float(np.percentile(ts, 99))

    def dev_only():
        g.replay()

    def with_h2d():
        img.data.copy_(host.data, non_blocking=True)
        g.replay()

    p50, p99 = timed(dev_only)
    h50, h99 = timed(with_h2d)
    return {"p50_ms": round(p50, 4), "p99_ms": round(p99, 4), "h2d_p50_ms": round(h50, 4),
            "h2d_p99_ms": round(h99, 4), "iters": iters,
            "workload": "1 x 1920x1080, E=448 InternVL3-2B tiling, bf16 NCHW; CUDA graph "
                        "(K1+K2); h2d_* add the 6.2 MB pinned upload"}


if __name__ == "__main__":
    main()
