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
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=64, help="images per GPU per step (C2: 64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--latency-iters", type=int, default=300)
    ap.add_argument("--workload", choices=["c2", "c4", "c5", "c1", "c3"], default="c2",
                    help="c2 (default, the BASELINE metric config); c4 = 8192-image "
                         "mixed-aspect sweep (sharded, strong scaling); c5 = 1024 images + "
                         "placeholder expansion; c1/c3 = single-image latency configs")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = False
        self.backend = None
        # dry run of the N-rank path on fewer GPUs (ranks share devices, gloo barrier):
        # checks that the sharded bench runs end to end; its numbers are not scaling data
        self.shared_gpu = os.environ.get("TP_BENCH_SHARED_GPU_DRYRUN") == "1"

    def tag(self, line: dict) -> dict:
        if self.shared_gpu and self.world > 1:
            line["dryrun"] = "ranks shared GPUs (TP_BENCH_SHARED_GPU_DRYRUN): not a scaling number"
        return line

    def device_index(self, n_devices: int) -> int:
        return self.local_rank % n_devices if self.shared_gpu else self.local_rank

    def init(self, backend: str):
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            self.backend = "gloo" if self.shared_gpu else backend
            dist.init_process_group(backend=self.backend)
            self.pg = True

    def barrier(self, device=None):
        if self.pg:
            import torch.distributed as dist

            if device is not None and self.backend == "nccl":
                dist.barrier(device_ids=[device.index])
            else:
                dist.barrier()

    def max(self, value: float, device) -> float:
        if not self.pg:
            return value
        import torch
        import torch.distributed as dist

        t = torch.tensor([value], dtype=torch.float64,
                         device=device if self.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            import torch.distributed as dist

            dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    """SM clock and throttle reasons sampled from a thread while the timed region runs.
    In-process NVML (pynvml): no nvidia-smi fork inside the timed region, which used to
    stall the launching thread for milliseconds.  Falls back to nvidia-smi."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int, interval_s: float = 0.002):
        self.gpu = gpu_index
        self.interval = interval_s
        self.samples = []  # (sm_mhz, max_mhz, [reason names])
        self._stop = threading.Event()
        self._thr = None
        self._nvml = None
        self._handle = None
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            handle = None
            try:
                prop = torch.cuda.get_device_properties(gpu_index)
                bus = f"{prop.pci_domain_id:08x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
                handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                handle = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self._nvml, self._handle = pynvml, handle
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml, self._handle
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        names = [n for n, attr in self.REASONS if mask & getattr(nv, attr)]
        self.samples.append((float(sm), float(mx), names))

    def _sample_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={fields}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            v = [x.strip() for x in out.stdout.strip().split(",")]
            names = [n for (n, _), x in zip(self.REASONS, v[2:]) if x.lower() == "active"]
            self.samples.append((float(v[0]), float(v[1]), names))

    def start(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def sample_now(self):
        """One sample from the calling thread: called right after the timed steps are
        enqueued, while the GPU is still executing them, so even a short timed region
        has a sample taken under load."""
        try:
            self._sample_nvml() if self._nvml else self._sample_smi()
        except Exception:
            pass

    def _run(self):
        while True:
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            if self._stop.wait(self.interval if self._nvml else 0.1):
                break

    def stop(self) -> dict:
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clocks unavailable"],
                    "samples": 0}
        return {"sm_mhz": float(np.median([x[0] for x in self.samples])),
                "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": sorted({r for x in self.samples for r in x[2]}),
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm on host cores (oracle port)

def _cpu_one(args):
    """One image through the oracle path; the synthetic input is generated before
    the clock starts, so only the preprocessing itself is timed."""
    seed, k, w, h = args
    from oracle import tileprep_oracle as O
    from paper_2603_16987_b200.workloads import IMAGENET_MEAN, IMAGENET_STD

    arr = O.synth_image(seed, k, w, h, 3, 0)
    t0 = time.perf_counter()
    O.preprocess_image(arr, 448, 12, IMAGENET_MEAN, IMAGENET_STD, True)
    return time.perf_counter() - t0


def cpu_throughput(n_images: int, cores: int, seed: int = 20260817):
    """images/s of the oracle path with `cores` worker processes busy at once:
    cores / mean per-image time (each time measured while all workers run, so
    memory-bandwidth contention is included).  Returns (images/s, p50 ms, CPU-s)."""
    import multiprocessing as mp

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    jobs = [(seed, k, 1920, 1080) for k in range(n_images)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_one, jobs[:cores])  # warm the workers
        per = np.array(pool.map(_cpu_one, jobs, chunksize=1))
    return cores / float(per.mean()), float(np.median(per)) * 1e3, float(per.sum())


_CPU_VOCAB = None


def _cpu_vocab():
    """(byte_ids, table, max_len, marker, ctx, asst) of the synthetic C5 vocab, per worker."""
    global _CPU_VOCAB
    if _CPU_VOCAB is None:
        from oracle import tileprep_oracle as O
        from paper_2603_16987_b200.workloads import synthetic_vocab_text

        toks, byte_ids, table, max_len = O.parse_vocab(synthetic_vocab_text())
        _CPU_VOCAB = (byte_ids, table, max_len, toks.index("<|image|>"),
                      toks.index("<IMG_CONTEXT>"), toks.index("<|assistant|>"))
    return _CPU_VOCAB


def _cpu_wl_one(args):
    """One image of a workload through the oracle path (input generated off the clock);
    with a prompt (C5) also its tokenization, image-token expansion (256 tokens per tile)
    and supervision mask."""
    seed, k, w, h, e, max_tiles, mean, std, bf16, text = args
    from oracle import tileprep_oracle as O

    arr = O.synth_image(seed, k, w, h, 3, 0)
    voc = _cpu_vocab() if text is not None else None
    t0 = time.perf_counter()
    plan, _ = O.preprocess_image(arr, e, max_tiles, mean, std, bf16)
    if voc is not None:
        byte_ids, table, max_len, marker, ctx, asst = voc
        ids = O.tokenize(text, byte_ids, table, max_len)
        out, _, t = O.expand(ids, [O.n_images(plan)], 256, marker, ctx, asst)
        O.supervision_mask(out, t, asst)
    return time.perf_counter() - t0


def _wl_jobs(wl, n: int, texts=None):
    return [(wl.seed, k, int(wl.wh[k % len(wl.wh)][0]), int(wl.wh[k % len(wl.wh)][1]),
             wl.tile_edge, wl.max_tiles, tuple(wl.mean), tuple(wl.std), bool(wl.bf16),
             None if texts is None else texts[k])
            for k in range(n)]


def cpu_latency(wl, runs: int = 15) -> dict:
    """Batch-1 latency of the oracle path on one host core (one process,
    OMP/OPENBLAS_NUM_THREADS=1, p50/p99 over >= 15 runs), as a cpu_baseline object."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    job = _wl_jobs(wl, 1)[0]
    _cpu_wl_one(job)  # warm-up
    t = np.array([_cpu_wl_one(job) for _ in range(runs)]) * 1e3
    p50 = float(np.percentile(t, 50))
    return {"value": round(1e3 / p50, 3), "unit": UNIT, "cores": 1, "kind": "port",
            "p50_ms": round(p50, 2), "p99_ms": round(float(np.percentile(t, 99)), 2),
            "sample": f"{runs} runs of 1 x {job[2]}x{job[3]} through oracle/tileprep_oracle "
                      "(numpy restatement of the vlmfp fused path), one process, one thread; "
                      "value = 1 / p50"}


def cpu_throughput_wl(wl, cores: int, cpu_seconds: float, texts=None) -> dict:
    """images/s of the oracle path on a prefix of the workload's images (and prompts),
    one process per core (all busy at once), sized to about `cpu_seconds` of CPU work."""
    import multiprocessing as mp

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        cal = np.array(pool.map(_cpu_wl_one, _wl_jobs(wl, cores, texts), chunksize=1))
        n = int(max(cores, min(len(wl.wh), cpu_seconds / max(float(cal.mean()), 1e-3))))
        per = np.array(pool.map(_cpu_wl_one, _wl_jobs(wl, n, texts), chunksize=1))
    return {"value": round(cores / float(per.mean()), 3), "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": f"first {n} of the {len(wl.wh)} {wl.name} images"
                      + (" and prompts (tokenize + expand + mask)" if texts else "")
                      + f" through oracle/tileprep_oracle, one process per core, "
                      f"{per.sum():.1f} CPU-s; "
                      f"per-image p50 {np.median(per) * 1e3:.1f} ms"}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run_reference(args, dist: Dist):
    """--impl reference: the reference algorithm (oracle port of vlmfp's fused,
    contiguous path) on all host cores, rank 0 only; each step is a bounded sample
    of C2 images."""
    if dist.rank != 0:
        return
    cores = host_cores()
    sample = max(cores, 16)
    cpu_throughput(cores, cores)  # warm-up
    rates, p50s, cpu_s = [], [], 0.0
    for _ in range(args.steps):
        ips, p50_ms, cs = cpu_throughput(sample, cores)
        rates.append(ips)
        p50s.append(p50_ms)
        cpu_s += cs
    value = float(np.median(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sample / value * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8 in, fp32 + fp64-exact resample, bf16 out",
        "data": "synthetic",
        "config": {"workload": "C2: 1920x1080 RGB uint8, E=448, max 12 + thumb, "
                               "ImageNet mean/std, bf16 out", "images_per_step": sample},
        "p50_ms": round(float(np.median(p50s)), 3),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                         "kind": "port",
                         "sample": f"{sample} images x {args.steps} steps ({cpu_s:.0f} CPU-s) "
                                   "through oracle/tileprep_oracle (numpy restatement of the "
                                   "vlmfp fused/contiguous recipe path), one process per core"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(dist.tag(line)), flush=True)


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
    dev_index = dist.device_index(torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    dist.init("nccl")
    if args.workload in ("c4", "c5"):
        run_sweep(args, dist, device)
        dist.close()
        return
    if args.workload in ("c1", "c3"):
        run_single(args, dist, device)
        dist.close()
        return

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
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(i=None):
        # K1 then K2; K2 is a programmatic dependent launch of K1 (and the next K1 of K2),
        # so no event is recorded between them inside the timed steps
        # steady state: the previous step's K2 is the last kernel on the stream
        prep.plan(images, out.plans, stream, after_kernel=True)
        prep.tile(images, out.plans, out.pixel_values, None, stream, after_plan=True)

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
    torch.cuda.synchronize(device)
    clocks = ClockSampler(dev_index)
    clocks.start()
    dist.barrier(device)
    torch.cuda.synchronize(device)
    start.record(stream)
    for i in range(args.steps):
        step(i)
    stop.record(stream)
    clocks.sample_now()
    torch.cuda.synchronize(device)
    dist.barrier(device)
    clk = clocks.stop()
    ms_local = start.elapsed_time(stop)
    ms = dist.max(ms_local, device)
    # K2's own launch duration (the roofline's denominator): the same launches back to back
    # on the same stream and inputs, CUDA events around all of them
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    k0.record(stream)
    for _ in range(args.steps):
        prep.tile(images, out.plans, out.pixel_values, None, stream)
    k1.record(stream)
    torch.cuda.synchronize(device)
    k2_ms = k0.elapsed_time(k1) / args.steps
    ms_step = ms / args.steps
    value = dist.world * n * args.steps / (ms / 1e3)

    # ---- end to end through the public API with host buffers ----------------
    # The batch sits in a page-locked arena, staged once (pixels + sizes + offsets, one
    # region: transfer.stage_images). Every timed step uploads it with ONE H2D copy on a
    # copy stream, runs K1+K2 on the compute stream and reads the plans and tile offsets
    # back (D2H); device buffers alternate so step i+1's upload overlaps step i's kernels.
    from paper_2603_16987_b200.transfer import HostArena, stage_images, staged_bytes, upload_images

    offs, whs = images.offsets_host, images.wh_host
    host_imgs = [images.data[int(o): int(o) + int(w) * int(h) * 3].cpu().numpy().reshape(int(h), int(w), 3)
                 for o, (w, h) in zip(offs, whs)]
    # only the source rows K2's stencil reads go over the link (stage_images(touched=...),
    # tp_tile_rows: 83% of a 1080p image at E=448); full_bytes is the whole-image upload
    full_bytes = staged_bytes(host_imgs)
    touched = (cfg.tile_edge, cfg.max_tiles)
    nbytes = staged_bytes(host_imgs, touched=touched)
    staged = stage_images(host_imgs, HostArena(nbytes, 256, pin=True), touched=touched)
    del host_imgs
    slabs = [torch.empty(nbytes, dtype=torch.uint8, device=device) for _ in range(2)]
    outs2 = [out, prep(images)]
    plan_host = [torch.empty_like(out.plans.plan, device="cpu").pin_memory() for _ in range(2)]
    off_host = [torch.empty_like(out.plans.tile_off, device="cpu").pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream(device)
    done = [None, None]
    e2e_steps = max(5, min(args.steps, 30))

    def e2e_step(i):
        k = i % 2
        if done[k] is not None:
            copy_stream.wait_event(done[k])  # slab k no longer read by step i-2's K2
        packed_k, copied = upload_images(staged, slabs[k], copy_stream)
        stream.wait_event(copied)
        with torch.cuda.stream(stream):
            prep(packed_k, out=outs2[k], stream=stream)
            plan_host[k].copy_(outs2[k].plans.plan, non_blocking=True)
            off_host[k].copy_(outs2[k].plans.tile_off, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        done[k] = ev

    for i in range(3):
        e2e_step(i)
    torch.cuda.synchronize(device)
    dist.barrier(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(copy_stream)
    for i in range(e2e_steps):
        e2e_step(i)
    e1.record(stream)
    torch.cuda.synchronize(device)
    e2e_ms = dist.max(e0.elapsed_time(e1), device) / e2e_steps
    h2d = len(staged.batch.payload)  # bytes actually copied (incl. 256-byte alignment)
    d2h = plan_host[0].numel() * 4 + off_host[0].numel() * 4

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
        n_cpu = int(max(cores, min(512, args.cpu_seconds * 1e3 / max(p50_ms, 1.0))))
        ips, p50_ms, cpu_s = cpu_throughput(n_cpu, cores)
        cpu = {"value": round(ips, 3), "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n_cpu} C2 images (1920x1080) through oracle/tileprep_oracle "
                         f"(numpy restatement of the vlmfp fused path), one process per core, "
                         f"{cpu_s:.1f} CPU-s; per-image p50 {p50_ms:.1f} ms"}

    traffic = measured_traffic("tp_tile", wb["total"])
    if dist.rank == 0:
        bytes_per_launch = wb["total"]
        achieved = bytes_per_launch / (k2_ms / 1e3) / 1e9
        peak = measured_peak()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 in, fp32 + fp64-exact resample, bf16 out", "data": "synthetic",
            "config": {"workload": "C2: " + wl.description, "images_per_gpu": n,
                       "tiles_per_gpu": n_tiles, "l2": "inputs (398 MB/GPU) larger than L2",
                       "parallelism": f"dp{dist.world} (independent images, no collective)"},
            "p50_ms": latency["p50_ms"] if latency else None,
            "latency": latency,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak[0],
                         "unit": "GB/s", "frac": round(achieved / peak[0], 4),
                         "traffic": traffic, "peak_source": peak[1],
                         "kernel": "tp_tile (K2)", "kernel_ms": round(k2_ms, 4),
                         "kernel_timing": "CUDA events around K back-to-back K2 launches, "
                                          "same stream and inputs, after the timed steps",
                         "bytes_per_launch": bytes_per_launch,
                         "bytes_full_image": int(wb["read_full"] + wb["write"]),
                         "peak_nominal_gbs": 8000.0,
                         "frac_of_nominal": round(achieved / 8000.0, 4)},
            "cpu_baseline": cpu,
            "e2e": {"value": round(dist.world * n / (e2e_ms / 1e3), 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_ms, 4),
                    "path": "page-locked staged batch (touched source rows and columns + maps) -> "
                            "one H2D copy (copy stream) -> TilePreprocessor K1+K2 "
                            "(compute stream, K2 reads rows through the maps) -> D2H "
                            "plans/offsets; two device buffers, so step i+1's upload "
                            "overlaps step i",
                    "h2d_bytes_full_images": int(full_bytes)},
            "gpu_launches": 2 * args.steps,
            "clocks": clk,
        }
        print(json.dumps(dist.tag(line)), flush=True)
    dist.close()


def measured_traffic(kernel: str, algorithmic: int):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    summary (profiles/k2_traffic.json, written from `ncu --set full`), or None."""
    p = REPO / "profiles" / "k2_traffic.json"
    try:
        d = json.loads(p.read_text())
        return int(d["dram_bytes_read"]) + int(d["dram_bytes_write"])
    except Exception:
        return None


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
    f50, _ = timed(_empty_graph(device, s))
    t50, t99, tbytes = _touched_h2d_latency(cfg, img, device, s, iters)
    return {"p50_ms": round(p50, 4), "p99_ms": round(p99, 4), "h2d_p50_ms": round(h50, 4),
            "h2d_p99_ms": round(h99, 4), "iters": iters,
            "h2d_touched_p50_ms": round(t50, 4), "h2d_touched_p99_ms": round(t99, 4),
            "h2d_touched_bytes": tbytes,
            "graph_floor_p50_ms": round(f50, 4),
            "workload": "1 x 1920x1080, E=448 InternVL3-2B tiling, bf16 NCHW; CUDA graph "
                        "(K1+K2); h2d_* add the 6.2 MB pinned upload"}


def _touched_h2d_latency(cfg, img, device, stream, iters: int):
    """p50/p99 of upload + K1 + K2 when only the touched source rows are staged
    (transfer.stage_images(touched=...)): one pinned H2D of the compact payload, then
    a CUDA graph of the preprocessor reading rows through the row maps."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor
    from paper_2603_16987_b200.transfer import HostArena, stage_images, staged_bytes, upload_images

    offs, whs = img.offsets_host, img.wh_host
    arrs = [img.data[int(o): int(o) + int(w) * int(h) * img.channels].cpu().numpy()
            .reshape(int(h), int(w), img.channels) for o, (w, h) in zip(offs, whs)]
    touched = (cfg.tile_edge, cfg.max_tiles)
    nbytes = staged_bytes(arrs, touched=touched)
    staged = stage_images(arrs, HostArena(nbytes, 256, pin=True), touched=touched)
    dest = torch.empty(nbytes, dtype=torch.uint8, device=device)
    packed, done = upload_images(staged, dest)
    done.synchronize()
    prep = TilePreprocessor(cfg, device)
    out = prep(packed)
    torch.cuda.synchronize(device)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        prep(packed, out=out, stream=torch.cuda.current_stream(device))
    src = staged.batch.slab[staged.batch.base: staged.batch.base + nbytes]
    ts = []
    for k in range(iters + 50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        with torch.cuda.stream(stream):
            dest.copy_(src, non_blocking=True)
            g.replay()
        b.record(stream)
        b.synchronize()
        if k >= 50:
            ts.append(a.elapsed_time(b))
    ts = np.array(ts)
    return float(np.percentile(ts, 50)), float(np.percentile(ts, 99)), int(nbytes)


def _empty_graph(device, stream):
    """Replay of a one-tiny-kernel CUDA graph: the launch + event floor under which no
    batch-1 latency measured this way can go (reported beside p50)."""
    import torch

    x = torch.zeros(1, device=device)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        x.add_(1)
    return g.replay


def _timed(fn, steps: int, warmup: int, stream, device, dist, events_per_step=None):
    import torch

    with torch.cuda.stream(stream):
        for _ in range(max(3, warmup)):
            fn()
    torch.cuda.synchronize(device)
    clocks = ClockSampler(device.index)
    clocks.start()
    dist.barrier(device)
    torch.cuda.synchronize(device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    with torch.cuda.stream(stream):
        for i in range(steps):
            fn(i)
    b.record(stream)
    clocks.sample_now()
    torch.cuda.synchronize(device)
    dist.barrier(device)
    clk = clocks.stop()
    return dist.max(a.elapsed_time(b), device), clk


def run_sweep(args, dist, device):
    """C4 (8192 mixed-aspect images, sharded over ranks by LPT; strong scaling) or C5
    (1024 of those images + batched placeholder expansion).  Inputs are generated on
    device before timing; a step processes the rank's whole shard in chunks of 1024."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.sharding import shard
    from paper_2603_16987_b200.tokenizer import PlaceholderExpander
    from paper_2603_16987_b200.workloads import Workload, c4, workload_bytes

    total = 8192 if args.workload == "c4" else 1024
    wl_all = c4(total)
    idx = shard(wl_all.wh, wl_all.tile_edge, wl_all.max_tiles, dist.rank, dist.world)
    wh = wl_all.wh[idx]
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=wl_all.mean, std=wl_all.std,
                           reduced_precision_normalize=True)
    chunk = 1024
    stream = torch.cuda.Stream(device)
    chunks = []
    for c0 in range(0, len(idx), chunk):
        chunks.append(synth_packed(wh[c0:c0 + chunk], 3, device, seed=wl_all.seed + c0, kind=0))
    prep = TilePreprocessor(cfg, device)
    outs = prep(chunks[0], capacity=chunk * 13)
    torch.cuda.synchronize(device)
    with_expand = args.workload == "c5"
    if with_expand:
        # rendered prompts tokenized on the device (K6), then expanded with the tile
        # counts straight from K1 (K3): ids never leave the GPU
        from paper_2603_16987_b200.tokenizer import DeviceTokenizer, parse_vocab
        from paper_2603_16987_b200.workloads import c5_texts, synthetic_vocab_text

        vocab = parse_vocab(synthetic_vocab_text(), "synthetic")
        n = len(idx)
        tok = DeviceTokenizer(vocab, device)
        texts = tok.upload(c5_texts(n, wl_all.seed))
        toks = tok(texts)
        count_off = torch.arange(0, n + 1, dtype=torch.int32, device=device)
        exp = PlaceholderExpander(vocab, 256, device)
        cap = texts.total + n * 13 * 256
        ex = exp(toks.ids, toks.off, outs.plans.n_images, count_off, cap)
        torch.cuda.synchronize(device)
        assert int(toks.err[:n].abs().sum()) == 0 and int(ex.out_off[-1]) > 0

    def step(i=None):
        for ch in chunks:
            if with_expand:
                tok(texts, out=toks, stream=stream)
            prep(ch, out=outs, stream=stream)
            if with_expand:
                exp(toks.ids, toks.off, outs.plans.n_images, count_off, cap, out=ex,
                    stream=stream)

    ms, clk = _timed(step, args.steps, args.warmup, stream, device, dist)
    ms_step = ms / args.steps
    wl = Workload("C4" if not with_expand else "C5", wl_all.description, wh, 448, 12,
                  wl_all.mean, wl_all.std, True, wl_all.seed)
    wb = workload_bytes(wl)
    value = total * args.steps / (ms / 1e3)  # all images of the job over the max-rank time
    if dist.rank == 0:
        peak = measured_peak()
        achieved = wb["total"] / (ms_step / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8 in, fp32/fp64-exact resample, bf16 out", "data": "synthetic",
            "config": {"workload": ("C4: " if not with_expand else "C5: ") + wl_all.description
                       + (" + device tokenization of rendered prompts (K6) and image-token"
                          " expansion (256 tokens/tile)" if with_expand else ""),
                       "images_total": total, "images_rank0": len(idx),
                       "l2": "inputs larger than L2", "parallelism": f"dp{dist.world} LPT shards"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak[0],
                         "unit": "GB/s", "frac": round(achieved / peak[0], 4), "traffic": None,
                         "bytes_per_step_rank0": wb["total"],
                         "note": "whole step (K1+K2" + ("+K6+K3" if with_expand else "") + ")"},
            "gpu_launches": args.steps * len(chunks) * (8 if with_expand else 2),
            "clocks": clk,
        }
        if dist.world == 1 and not args.no_cpu_baseline:
            cpu_texts = None
            if with_expand:
                from paper_2603_16987_b200.workloads import c5_texts
                cpu_texts = c5_texts(total, wl_all.seed)
            line["cpu_baseline"] = cpu_throughput_wl(wl_all, host_cores(), args.cpu_seconds,
                                                     cpu_texts)
        print(json.dumps(dist.tag(line)), flush=True)


def run_single(args, dist, device):
    """C1 (1920x1080, E=512, fp32) / C3 (3840x2160, E=448, bf16): batch-1 latency."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor, empty_packed, synth_packed
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.workloads import c1, c3, workload_bytes

    wl = c1() if args.workload == "c1" else c3()
    cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                           std=wl.std, reduced_precision_normalize=wl.bf16)
    img = synth_packed(wl.wh, 3, device, seed=wl.seed, kind=0)
    prep = TilePreprocessor(cfg, device)
    out = prep(img)
    s = torch.cuda.Stream(device)
    torch.cuda.synchronize(device)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prep(img, out=out, stream=torch.cuda.current_stream(device))
    host = empty_packed(wl.wh, 3, "cpu", pin=True)
    host.data.copy_(img.data.cpu())
    ts, th = [], []
    iters = max(args.latency_iters, 1000)
    for k in range(iters + 50):
        for with_h2d, sink in ((False, ts), (True, th)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                if with_h2d:
                    img.data.copy_(host.data, non_blocking=True)
                g.replay()
            b.record(s)
            b.synchronize()
            if k >= 50:
                sink.append(a.elapsed_time(b))
    ts, th = np.array(ts), np.array(th)
    floor_fn, tf = _empty_graph(device, s), []
    for k in range(550):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            floor_fn()
        b.record(s)
        b.synchronize()
        if k >= 50:
            tf.append(a.elapsed_time(b))
    t50, t99, tbytes = _touched_h2d_latency(cfg, img, device, s, min(iters, 500))
    wb = workload_bytes(wl)
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": round(1e3 / float(np.median(ts)), 2), "unit": UNIT,
            "n_gpus": 1, "steps": iters, "warmup": 50,
            "ms_per_step": round(float(np.median(ts)), 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8 in, bf16/fp32 out",
            "data": "synthetic", "config": {"workload": wl.name + ": " + wl.description},
            "p50_ms": round(float(np.percentile(ts, 50)), 4),
            "p99_ms": round(float(np.percentile(ts, 99)), 4),
            "h2d_p50_ms": round(float(np.percentile(th, 50)), 4),
            "h2d_p99_ms": round(float(np.percentile(th, 99)), 4),
            "graph_floor_p50_ms": round(float(np.median(tf)), 4),
            "h2d_touched_p50_ms": round(t50, 4), "h2d_touched_p99_ms": round(t99, 4),
            "h2d_touched_bytes": tbytes, "h2d_full_bytes": int(host.data.numel()),
            "algorithmic_bytes": wb["total"],
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_latency(wl)
        print(json.dumps(dist.tag(line)), flush=True)


if __name__ == "__main__":
    main()
