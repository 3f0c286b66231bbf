#!/usr/bin/env python3
"""Benchmark of the B200 VLM preprocessing hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch: K1 (plan) + K2 (fused
resample/crop/thumbnail/normalize -> bf16 NCHW) over BASELINE configs[1]
(C2: 64 synthetic 1920x1080 RGB images, InternVL3-2B tiling, E=448, max 12 +
thumbnail, ImageNet mean/std).  Inputs (398 MB) are larger than L2 (126 MB).
Each rank runs its own 64-image batch on its own GPU (weak scaling, no
data-path collective); the barrier + max-over-ranks timing are the only
cross-rank operations.  `--gpus N` without a torchrun environment re-launches
this script under torch.distributed.run with N ranks.

The JSON line also carries, as sub-blocks measured in the same run:
  e2e      the C2 batch end to end from the caller's numpy HWC arrays through the
           public pipeline (native host packing + one pinned H2D + K1 + K2 + D2H of
           the plans), host wall clock, packing inside the timed loop
  latency  batch-1 1080p (C2 tiling) p50/p99
  c3       BASELINE configs[2]: batch-1 4K p50/p99 (>= 1000 CUDA-graph launches)
  c1       BASELINE configs[0]: batch-1 1080p, E=512, fp32
  c4       BASELINE configs[3]: the 8192-image mixed sweep, LPT-sharded over the N
           ranks (strong scaling), per-GPU roofline
  c5       BASELINE configs[4]: 1024 images + device tokenization + expansion
each with its own clock record and CPU baseline.

`--impl reference` times the reference's own CPU implementation (vlmfp, installed
unmodified into baseline/_ref; its fastest recipe path: fused_transform,
contiguous_tensor_path, avoid_per_item_split, skip_pixel_mask) on all host cores,
rank 0 only, on the C2 batch.  Without baseline/_ref it falls back to the numpy
port in oracle/ (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
DTYPE = "u8 in, fp32 + fp64-exact resample, bf16 out"
REF_DIR = REPO / "baseline" / "_ref"


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=64, help="images per GPU per step (C2: 64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of each cpu_baseline sample")
    ap.add_argument("--latency-iters", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-sub", action="store_true",
                    help="skip the c1/c3/c4/c5 sub-blocks of the default line")
    ap.add_argument("--workload", choices=["c2", "c4", "c5", "c1", "c3"], default="c2",
                    help="c2 (default, the BASELINE metric config, with the other configs "
                         "as sub-blocks); c1/c3/c4/c5 alone as the line's workload")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# distributed plumbing

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_command(args_gpus: int, argv) -> list:
    """torch.distributed.run command line that re-runs this script with N ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={args_gpus}", "--master-addr=127.0.0.1",
            f"--master-port={_free_port()}", str(Path(__file__).resolve()), *argv]


def maybe_spawn(args, argv) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: run N ranks under torch.distributed.run and
    return its exit code; inside torchrun: check WORLD_SIZE == N.  None = run here."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            return subprocess.call(spawn_command(args.gpus, argv))
        return None
    if int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return None


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
        return self

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
# CPU side: the reference's own implementation (vlmfp from baseline/_ref), else the port

_VLMFP = None


def reference_module():
    """vlmfp as installed unmodified into baseline/_ref (pip --target), or None.
    TP_BENCH_CPU_IMPL=port forces the oracle port."""
    global _VLMFP
    if _VLMFP is None:
        _VLMFP = False
        if os.environ.get("TP_BENCH_CPU_IMPL") != "port" and (REF_DIR / "vlmfp").is_dir():
            if str(REF_DIR) not in sys.path:
                sys.path.insert(0, str(REF_DIR))
            try:
                import vlmfp

                _VLMFP = vlmfp
            except Exception:  # pragma: no cover - missing PIL / ml_dtypes
                _VLMFP = False
    return _VLMFP or None


def cpu_kind() -> str:
    return "reference" if reference_module() is not None else "port"


def cpu_impl_name() -> str:
    return ("vlmfp (the reference, baseline/_ref) select_tile_plan -> tile_image -> "
            "normalize_tiles with fused_transform, contiguous_tensor_path, "
            "avoid_per_item_split, skip_pixel_mask"
            if reference_module() is not None else
            "oracle/tileprep_oracle (numpy port of vlmfp's fused path, band-shared "
            "vertical blend, in-place ops)")


def cpu_preprocess(arr, e, max_tiles, mean, std, bf16):
    """One image through the CPU path; returns the plan's n_images."""
    V = reference_module()
    if V is not None:
        cfg = V.PreprocessConfig(tile_edge=e, max_tiles=max_tiles, mean=tuple(mean),
                                 std=tuple(std), reduced_precision_normalize=bf16,
                                 fused_transform=True, contiguous_tensor_path=True,
                                 avoid_per_item_split=True, skip_pixel_mask=True)
        img = V.ImageBuffer.from_array(arr)
        plan = V.select_tile_plan(img.width, img.height, cfg)
        V.normalize_tiles(V.tile_image(img, plan, cfg), cfg)
        return plan.n_images
    from oracle import tileprep_oracle as O

    plan, _ = O.preprocess_image(arr, e, max_tiles, mean, std, bf16)
    return O.n_images(plan)


_CPU_VOCAB = None


def _cpu_vocab():
    """(tokenize, expand+mask) closures over the synthetic C5 vocab, per worker."""
    global _CPU_VOCAB
    if _CPU_VOCAB is None:
        from paper_2603_16987_b200.workloads import synthetic_vocab_text

        V = reference_module()
        if V is not None:
            import tempfile

            with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False,
                                             encoding="utf-8") as f:
                f.write(synthetic_vocab_text())
            vocab = V.load_vocab(f.name)
            os.unlink(f.name)

            def tok(text):
                return V.tokenize(text, vocab)

            def expand(ids, n_img):
                seq = V.expand_image_placeholders(ids, [n_img], 256, vocab)
                return V.build_supervision_mask(seq, vocab)
        else:
            from oracle import tileprep_oracle as O

            toks, byte_ids, table, max_len = O.parse_vocab(synthetic_vocab_text())
            marker, ctx, asst = (toks.index("<|image|>"), toks.index("<IMG_CONTEXT>"),
                                 toks.index("<|assistant|>"))

            def tok(text):
                return O.tokenize(text, byte_ids, table, max_len)

            def expand(ids, n_img):
                out, _, t = O.expand(ids, [n_img], 256, marker, ctx, asst)
                return O.supervision_mask(out, t, asst)
        _CPU_VOCAB = (tok, expand)
    return _CPU_VOCAB


def _cpu_wl_one(args):
    """One image of a workload through the CPU path (input generated off the clock);
    with a prompt (C5) also its tokenization, image-token expansion (256 tokens per
    tile) and supervision mask.  Returns seconds."""
    seed, k, w, h, e, max_tiles, mean, std, bf16, text = args
    from oracle import tileprep_oracle as O

    arr = _CPU_IMAGES.get((seed, k, w, h)) if _CPU_IMAGES else None
    if arr is None:
        arr = O.synth_image(seed, k, w, h, 3, 0)
    voc = _cpu_vocab() if text is not None else None
    t0 = time.perf_counter()
    n_img = cpu_preprocess(arr, e, max_tiles, mean, std, bf16)
    if voc is not None:
        voc[1](voc[0](text), n_img)
    return time.perf_counter() - t0


_CPU_IMAGES: dict = {}


def _synth_job(job):
    from oracle import tileprep_oracle as O

    seed, k, w, h = job[:4]
    return O.synth_image(seed, k, w, h, 3, 0)


def _wl_jobs(wl, n: int, texts=None, start: int = 0):
    return [(wl.seed, k, int(wl.wh[k % len(wl.wh)][0]), int(wl.wh[k % len(wl.wh)][1]),
             wl.tile_edge, wl.max_tiles, tuple(wl.mean), tuple(wl.std), bool(wl.bf16),
             None if texts is None else texts[k])
            for k in range(start, start + n)]


def _pool(cores: int):
    import multiprocessing as mp

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    return mp.get_context("fork").Pool(cores)


def cpu_latency(wl, runs: int = 15) -> dict:
    """Batch-1 latency of the CPU path on one host core (one process,
    OMP/OPENBLAS_NUM_THREADS=1, p50/p99 over >= 15 runs), as a cpu_baseline object."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    job = _wl_jobs(wl, 1)[0]
    _cpu_wl_one(job)  # warm-up
    t = np.array([_cpu_wl_one(job) for _ in range(runs)]) * 1e3
    p50 = float(np.percentile(t, 50))
    return {"value": round(1e3 / p50, 3), "unit": UNIT, "cores": 1, "kind": cpu_kind(),
            "p50_ms": round(p50, 2), "p99_ms": round(float(np.percentile(t, 99)), 2),
            "sample": f"{runs} runs of 1 x {job[2]}x{job[3]} through {cpu_impl_name()}; "
                      "one process, one thread; value = 1 / p50"}


def cpu_throughput_wl(wl, cores: int, cpu_seconds: float, texts=None) -> dict:
    """images/s of the CPU path on a prefix of the workload's images (and prompts), one
    process per core (all busy at once, so memory-bandwidth contention is included),
    sized to about `cpu_seconds` of CPU work: cores / mean per-image time."""
    with _pool(cores) as pool:
        cal = np.array(pool.map(_cpu_wl_one, _wl_jobs(wl, cores, texts), chunksize=1))
        n = int(max(cores, min(len(wl.wh), cpu_seconds / max(float(cal.mean()), 1e-3))))
        per = np.array(pool.map(_cpu_wl_one, _wl_jobs(wl, n, texts), chunksize=1))
    return {"value": round(cores / float(per.mean()), 3), "unit": UNIT, "cores": cores,
            "kind": cpu_kind(),
            "sample": f"first {n} of the {len(wl.wh)} {wl.name} images"
                      + (" and prompts (tokenize + expand + mask)" if texts else "")
                      + f" through {cpu_impl_name()}; one process per core, "
                      f"{per.sum():.1f} CPU-s; per-image p50 {np.median(per) * 1e3:.1f} ms"}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def c2_config(wl, n: int, world: int) -> dict:
    return {"workload": "C2: " + wl.description, "images_per_gpu": n,
            "l2": "inputs (398 MB/GPU) larger than L2",
            "parallelism": f"dp{world} (independent images, no collective)"}


def run_reference(args, dist: Dist):
    """--impl reference: the reference's own CPU path (vlmfp from baseline/_ref) on all
    host cores, rank 0 only; each step = the C2 batch (64 images), one process per core."""
    if dist.rank != 0:
        return
    from oracle import tileprep_oracle as O
    from paper_2603_16987_b200.workloads import c2

    wl = c2(args.batch)
    cores = host_cores()
    jobs = _wl_jobs(wl, len(wl.wh))
    # the synthetic batch, generated in parallel and kept in this process before the
    # timing pool forks, so every worker inherits it (nothing generated on the clock)
    with _pool(cores) as pool:
        arrs = pool.map(_synth_job, jobs, chunksize=1)
    for j, a in zip(jobs, arrs):
        _CPU_IMAGES[j[:4]] = a
    del arrs
    times, per_img = [], []
    with _pool(cores) as pool:
        for _ in range(max(1, args.warmup)):
            pool.map(_cpu_wl_one, jobs[:cores], chunksize=1)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            per_img += pool.map(_cpu_wl_one, jobs, chunksize=1)
            times.append(time.perf_counter() - t0)
    total = float(np.sum(times))
    value = len(jobs) * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
        "config": c2_config(wl, len(jobs), dist.world),
        "p50_ms": round(float(np.median(per_img)) * 1e3, 3),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                         "kind": cpu_kind(),
                         "sample": f"the {len(jobs)}-image C2 batch x {args.steps} steps "
                                   f"({np.sum(per_img):.0f} CPU-s) through {cpu_impl_name()}; "
                                   "one process per core, images generated before the clock; "
                                   "p50_ms = per-image time with all cores busy"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(dist.tag(line)), flush=True)


# ---------------------------------------------------------------------------
# GPU side

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


def _timed(fn, steps: int, warmup: int, stream, device, dist):
    """Device time of `steps` calls of fn on `stream` (CUDA events, barrier +
    synchronize on both sides, max over ranks) and the clock record."""
    import torch

    with torch.cuda.stream(stream):
        for _ in range(max(3, warmup)):
            fn()
    torch.cuda.synchronize(device)
    clocks = ClockSampler(device.index).start()
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


def run_c2(args, dist, device, dev_index):
    """The headline: C2 device-resident steps, K2's roofline, and the e2e sub-block."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.workloads import c2, workload_bytes

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

    def step(i=None):
        # K1 then K2; K2 is a programmatic dependent launch of K1 (and the next K1 of K2),
        # so no event is recorded between them inside the timed steps.  Steady state:
        # the previous step's K2 is the last kernel on the stream.
        prep.plan(images, out.plans, stream, after_kernel=True)
        prep.tile(images, out.plans, out.pixel_values, None, stream, after_plan=True)

    ms, clk = _timed(step, args.steps, args.warmup, stream, device, dist)
    # K2's own launch duration (the roofline's denominator): the same launches back to
    # back on the same stream and inputs, CUDA events around all of them
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    k0.record(stream)
    for _ in range(args.steps):
        prep.tile(images, out.plans, out.pixel_values, None, stream)
    k1.record(stream)
    torch.cuda.synchronize(device)
    k2_ms = dist.max(k0.elapsed_time(k1) / args.steps, device)
    # the same K2 launch on smooth synthetic content (tp_synth kind 1): the exact fallback
    # fires far less often than on uniform noise (the headline's pessimistic input)
    smooth = synth_packed(wl.wh, 3, device, seed=seed, kind=1)
    prep.plan(smooth, out.plans, stream)
    torch.cuda.synchronize(device)
    for _ in range(3):
        prep.tile(smooth, out.plans, out.pixel_values, None, stream)
    k0.record(stream)
    for _ in range(args.steps):
        prep.tile(smooth, out.plans, out.pixel_values, None, stream)
    k1.record(stream)
    torch.cuda.synchronize(device)
    k2_smooth_ms = dist.max(k0.elapsed_time(k1) / args.steps, device)
    del smooth
    res = {"ms": ms, "ms_step": ms / args.steps, "value": dist.world * n * args.steps / (ms / 1e3),
           "clk": clk, "k2_ms": k2_ms, "k2_smooth_ms": k2_smooth_ms, "n": n, "n_tiles": n_tiles, "wb": wb, "wl": wl,
           "cfg": cfg}
    host_imgs = [images.data[int(o): int(o) + int(w) * int(h) * 3].cpu().numpy()
                 .reshape(int(h), int(w), 3) for o, (w, h) in zip(images.offsets_host,
                                                                   images.wh_host)]
    del images, out
    res["e2e"] = run_e2e(args, dist, device, cfg, host_imgs)
    res["e2e_jpeg"] = run_e2e_coded(args, dist, device, cfg, "jpeg")
    res["e2e_png"] = run_e2e_coded(args, dist, device, cfg, "png")
    return res


def run_e2e(args, dist, device, cfg, host_imgs) -> dict:
    """The C2 batch end to end through the public pipeline, from the caller's numpy HWC
    arrays (pageable host memory): every step packs the batch into a page-locked slab
    on the library's host threads (tp_stage_pack: only the source rows K2 reads), uploads
    it with one H2D copy, runs K1 + K2 and reads the plans and tile offsets back.  Two
    slabs rotate, so packing step i+1 overlaps the upload and kernels of step i.  Timed on
    the host clock (the host work is part of it), synchronize + barrier on both sides,
    max over ranks."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor
    from paper_2603_16987_b200.transfer import PipelinedPreprocessor, staged_bytes

    touched = (cfg.tile_edge, cfg.max_tiles)
    nbytes = staged_bytes(host_imgs, touched=touched)
    full_bytes = staged_bytes(host_imgs)
    prep = TilePreprocessor(cfg, device)
    pipe = PipelinedPreprocessor(prep, nbytes, depth=2, touched=True)
    outs = [None, None]
    plan_host = [None, None]
    off_host = [None, None]
    pack_s = []

    def e2e_step(i):
        k = i % 2
        t0 = time.perf_counter()
        outs[k] = pipe.submit(host_imgs, out=outs[k])
        pack_s.append(time.perf_counter() - t0)
        with torch.cuda.stream(pipe.compute_stream):
            if plan_host[k] is None:
                plan_host[k] = torch.empty_like(outs[k].plans.plan, device="cpu").pin_memory()
                off_host[k] = torch.empty_like(outs[k].plans.tile_off, device="cpu").pin_memory()
            plan_host[k].copy_(outs[k].plans.plan, non_blocking=True)
            off_host[k].copy_(outs[k].plans.tile_off, non_blocking=True)

    for i in range(3):
        e2e_step(i)
    torch.cuda.synchronize(device)
    pack_s.clear()
    steps = max(5, args.e2e_steps)
    dist.barrier(device)
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for i in range(steps):
        e2e_step(i)
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    dist.barrier(device)
    wall = dist.max(wall, device)
    # the H2D link alone on the same payload (what the packing overlaps with)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    src = pipe.host[0].tensor[: pipe.last_bytes]
    h0.record(pipe.copy_stream)
    for _ in range(5):
        pipe.dev[0][: pipe.last_bytes].copy_(src, non_blocking=True)
    h1.record(pipe.copy_stream)
    torch.cuda.synchronize(device)
    h2d_ms = h0.elapsed_time(h1) / 5
    n = len(host_imgs)
    ms_step = wall / steps * 1e3
    return {"value": round(dist.world * n / (ms_step / 1e3), 2), "unit": UNIT,
            "h2d_bytes_per_step": int(pipe.last_bytes),
            "d2h_bytes_per_step": int(plan_host[0].numel() * 4 + off_host[0].numel() * 4),
            "ms_per_step": round(ms_step, 4), "steps": steps,
            "pack_ms": round(float(np.median(pack_s)) * 1e3, 3),
            "pack_gbs": round(pipe.last_bytes / float(np.median(pack_s)) / 1e9, 2),
            "h2d_ms": round(h2d_ms, 3),
            "h2d_gbs": round(pipe.last_bytes / (h2d_ms / 1e3) / 1e9, 2),
            "host_threads": int(_host_threads()),
            "timing": "host wall clock around all steps (synchronize + barrier both sides, "
                      "max over ranks); pack_ms = median host time of one submit() "
                      "(native row packing into the pinned slab + enqueue)",
            "path": "caller's numpy HWC arrays (pageable) -> PipelinedPreprocessor.submit: "
                    "tp_stage_pack on the host thread pool (touched source rows only) into "
                    "a pinned slab -> one H2D copy (copy stream) -> K1 + K2 (compute "
                    "stream, K2 reads rows through the maps) -> D2H plans/offsets; two "
                    "slabs, so packing step i+1 overlaps the upload of step i",
            "h2d_bytes_full_images": int(full_bytes)}


def _cpu_jpeg_one(args):
    """One JPEG payload through the reference's own preprocess (vlmfp: decode with Pillow
    + plan + fused tiles + normalize, fastest toggles), or the port (Pillow + oracle)."""
    idx, e, mt, mean, std, bf16 = args
    payload = _CPU_PAYLOADS[idx]
    V = reference_module()
    t0 = time.perf_counter()
    if V is not None:
        cfg = V.PreprocessConfig(tile_edge=e, max_tiles=mt, mean=tuple(mean), std=tuple(std),
                                 reduced_precision_normalize=bf16, fused_transform=True,
                                 contiguous_tensor_path=True, avoid_per_item_split=True,
                                 skip_pixel_mask=True, decode_once=True, simd_decode=True)
        V.preprocess(payload, cfg)
    else:
        import io

        from PIL import Image

        arr = np.asarray(Image.open(io.BytesIO(payload)).convert("RGB"))
        cpu_preprocess(arr, e, mt, mean, std, bf16)
    return time.perf_counter() - t0


_CPU_PAYLOADS: list = []


def run_e2e_coded(args, dist, device, cfg, fmt: str = "jpeg") -> dict:
    """The C2 batch as coded payloads, end to end from the caller's bytes -- fmt "jpeg":
    64 corpus-like 1080p scenes, q85 baseline 4:2:0, device JPEG decode (K7: host marker
    parse + one H2D of the compressed scans + parallel Huffman / IDCT / colour on the GPU);
    fmt "png": the same scenes as Pillow PNGs, device PNG decode (K8: host chunk walk +
    one H2D of the IDAT data + block finder / parallel inflate / unfilter on the GPU) --
    then K1 + K2 -> D2H of the plans; two buffer sets, so the host work of step i+1
    overlaps step i.  Host wall clock; the reference's own preprocess (decode included)
    on all host cores beside it."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor
    from paper_2603_16987_b200.jpeg import JpegDecoder
    from paper_2603_16987_b200.png import PngDecoder
    from paper_2603_16987_b200.workloads import jpeg_payloads, png_payloads

    if fmt == "png":
        payloads = png_payloads(args.batch, seed=20260817 + 97 * dist.rank)
        dec = PngDecoder(device, depth=2)
    else:
        payloads = jpeg_payloads(args.batch, seed=20260817 + 97 * dist.rank)
        dec = JpegDecoder(device, depth=2)
    prep = TilePreprocessor(cfg, device)
    # one compute stream (the uploads run on the decoder's copy stream): a stream per
    # buffer set, letting consecutive batches' decodes overlap, measured slower (e2e_jpeg
    # 20.4K vs 22.8K, e2e_png 4.6K vs 5.4K images/s)
    streams = [torch.cuda.Stream(device)] * 2
    stream = streams[0]
    outs, pend = [None, None], [None, None]
    plan_host = [None, None]
    refits = [0]

    def step(i):
        k = i % 2
        stream = streams[k]
        if pend[k] is not None:  # the batch that used these buffers two steps ago
            b, o = pend[k]
            if b.finish():  # host-decoded images patched in: tile that batch again
                refits[0] += 1
                with torch.cuda.stream(stream):
                    prep(b.images, out=o, stream=stream)
        b = dec.decode(payloads, stream=stream, sync=False)
        with torch.cuda.stream(stream):
            outs[k] = prep(b.images, out=outs[k], stream=stream)
            if plan_host[k] is None:
                plan_host[k] = torch.empty_like(outs[k].plans.plan, device="cpu").pin_memory()
            plan_host[k].copy_(outs[k].plans.plan, non_blocking=True)
        pend[k] = (b, outs[k])

    for i in range(4):
        step(i)
    torch.cuda.synchronize(device)
    steps = max(5, args.e2e_steps)
    dist.barrier(device)
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    for k in range(2):
        if pend[k] is not None:
            pend[k][0].finish()
    torch.cuda.synchronize(device)
    wall = dist.max(time.perf_counter() - t0, device)
    # the decode kernels alone on the last batch (CUDA events around relaunches)
    stream = streams[(steps - 1) % 2]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(5):
        dec.launch(stream)
    b.record(stream)
    torch.cuda.synchronize(device)
    n = len(payloads)
    res = {"value": round(dist.world * n * steps / wall, 2), "unit": UNIT,
           "ms_per_step": round(wall / steps * 1e3, 4), "steps": steps,
           "h2d_bytes_per_step": int(dec.last_h2d_bytes),
           "d2h_bytes_per_step": int(plan_host[0].numel() * 4 + 4 * n),
           "payload_kb_avg": round(sum(map(len, payloads)) / n / 1e3, 1),
           "decode_kernels_ms": round(a.elapsed_time(b) / 5, 4),
           "host_fallbacks": dec.last_fallback, "refits": refits[0],
           "path": ("caller's JPEG bytes -> JpegDecoder.decode(sync=False): tp_jpeg_parse + "
                    "tp_jpeg_describe + tp_stage_pack into a pinned slab -> one H2D of the "
                    "compressed scans -> K7 (unstuff, self-synchronizing parallel Huffman, "
                    "ISLOW IDCT, fancy upsampling + YCbCr->RGB) -> K1 + K2 -> D2H plans")
           if fmt == "jpeg" else
           ("caller's PNG bytes (Pillow, default settings) -> PngDecoder.decode(sync=False): "
            "tp_png_parse + tp_png_describe + tp_stage_pack of the IDAT data into a pinned "
            "slab -> one H2D -> K8 (block finder, warp-parallel speculative inflate, chain "
            "check, token expansion, window markers, Adler-32, unfilter wavefront) -> "
            "K1 + K2 -> D2H plans"),
           "timing": "host wall clock around all steps (synchronize + barrier both sides, "
                     "max over ranks)"}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        _CPU_PAYLOADS[:] = payloads
        cores = host_cores()
        from paper_2603_16987_b200.dtypes import FLOAT16_WIDE

        jobs = [(i, cfg.tile_edge, cfg.max_tiles, tuple(cfg.mean), tuple(cfg.std),
                 cfg.effective_precision == FLOAT16_WIDE) for i in range(n)]
        with _pool(cores) as pool:
            pool.map(_cpu_jpeg_one, jobs[:cores], chunksize=1)
            t1 = time.perf_counter()
            per = pool.map(_cpu_jpeg_one, jobs, chunksize=1)
            dt = time.perf_counter() - t1
        res["cpu_baseline"] = {
            "value": round(n / dt, 3), "unit": UNIT, "cores": cores, "kind": cpu_kind(),
            "sample": f"the same {n} {fmt.upper()} payloads through "
                      + ("vlmfp.preprocess (the reference: Pillow decode + plan + fused tiles "
                         "+ normalize, fastest toggles)" if reference_module() is not None
                         else "Pillow decode + the oracle port")
                      + f", one process per core; per-image p50 {np.median(per) * 1e3:.1f} ms"}
    return res


def run_dropin(args, device, runs: int = 60) -> dict:
    """The drop-in per-request path: preprocess(payload, cfg) for one 1080p image as a
    JPEG (device decode, K7) and as a PNG (device decode, K8),
    C2 tiling, sequential requests; p50/p99 and the median of every stage_timings_ns
    key, beside the reference's own vlmfp.preprocess (fastest toggles, one host core)
    on the same payloads."""
    import io

    import torch
    from PIL import Image

    from paper_2603_16987_b200 import imgproc
    from paper_2603_16987_b200.workloads import IMAGENET_MEAN, IMAGENET_STD, scene_image

    px = scene_image(1920, 1080, 4242)
    payloads = {}
    for fmt, kw in (("jpeg", {"quality": 85}), ("png", {})):
        buf = io.BytesIO()
        Image.fromarray(px).save(buf, format=fmt.upper(), **kw)
        payloads[fmt] = buf.getvalue()
    cfg = imgproc.PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN,
                                   std=IMAGENET_STD, reduced_precision_normalize=True,
                                   fused_transform=True, contiguous_tensor_path=True,
                                   avoid_per_item_split=True, skip_pixel_mask=True,
                                   decode_once=True, simd_decode=True)
    out = {}
    for fmt, p in payloads.items():
        for _ in range(5):
            imgproc.preprocess(p, cfg)
        torch.cuda.synchronize(device)
        ts, stages = [], {}
        for _ in range(runs):
            t0 = time.perf_counter_ns()
            r = imgproc.preprocess(p, cfg)
            ts.append((time.perf_counter_ns() - t0) / 1e6)
            for k, v in r.stage_timings_ns.items():
                stages.setdefault(k, []).append(v / 1e6)
        res = {"payload_kb": round(len(p) / 1e3, 1), "p50_ms": round(float(np.median(ts)), 3),
               "p99_ms": round(float(np.percentile(ts, 99)), 3),
               "stages_ms_p50": {k: round(float(np.median(v)), 3) for k, v in stages.items()},
               "tiles": len(r.tiles), "dtype": r.tiles[0].elem}
        V = reference_module()
        if V is not None and not args.no_cpu_baseline:
            vcfg = V.PreprocessConfig(**{f: getattr(cfg, f) for f in (
                "tile_edge", "max_tiles", "mean", "std", "normalize_precision", "fused_transform",
                "contiguous_tensor_path", "decode_once", "reduced_precision_normalize",
                "simd_decode", "skip_pixel_mask", "avoid_per_item_split")})
            V.preprocess(p, vcfg)
            rt, rst = [], {}
            for _ in range(15):
                t0 = time.perf_counter_ns()
                rr = V.preprocess(p, vcfg)
                rt.append((time.perf_counter_ns() - t0) / 1e6)
                for k, v in rr.stage_timings_ns.items():
                    rst.setdefault(k, []).append(v / 1e6)
            res["reference"] = {"p50_ms": round(float(np.median(rt)), 3),
                                "p99_ms": round(float(np.percentile(rt, 99)), 3),
                                "stages_ms_p50": {k: round(float(np.median(v)), 3)
                                                  for k, v in rst.items()},
                                "cores": 1, "kind": "reference",
                                "sample": "15 sequential vlmfp.preprocess calls, fastest toggles"}
        out[fmt] = res
    out["timing"] = ("host wall clock per call (the drop-in returns host ImageBuffers, so "
                     "each call ends after the tiles' readback); sequential, one stream")
    return out


def _host_threads() -> int:
    from paper_2603_16987_b200 import _lib

    return _lib.load().tp_host_threads()


def batch1_latency(cfg, wh, device, iters: int, with_touched: bool = True) -> dict:
    """p50/p99 of one image through the preprocessor (device-resident input, CUDA-graph
    launched: the fused tp_plan_tile), the same with the pinned H2D of the whole image
    and of its touched rows, and the graph floor; with a clock record."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor, empty_packed, synth_packed

    wh = np.asarray(wh, dtype=np.int32).reshape(-1, 2)
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
    floor = _empty_graph(device, s)

    def dev_only():
        g.replay()

    def with_h2d():
        img.data.copy_(host.data, non_blocking=True)
        g.replay()

    clocks = ClockSampler(device.index).start()
    ts = {"dev": [], "h2d": [], "floor": []}
    for k in range(iters + 50):
        for name, fn in (("dev", dev_only), ("h2d", with_h2d), ("floor", floor)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                fn()
            b.record(s)
            b.synchronize()
            if k >= 50:
                ts[name].append(a.elapsed_time(b))
    clk = clocks.stop()
    d, h = np.array(ts["dev"]), np.array(ts["h2d"])
    res = {"p50_ms": round(float(np.percentile(d, 50)), 4),
           "p99_ms": round(float(np.percentile(d, 99)), 4),
           "h2d_p50_ms": round(float(np.percentile(h, 50)), 4),
           "h2d_p99_ms": round(float(np.percentile(h, 99)), 4),
           "h2d_bytes": int(host.data.numel()), "iters": iters,
           "graph_floor_p50_ms": round(float(np.median(ts["floor"])), 4)}
    if with_touched:
        t50, t99, tbytes = _touched_h2d_latency(cfg, img, device, s, min(iters, 500))
        res.update({"h2d_touched_p50_ms": round(t50, 4), "h2d_touched_p99_ms": round(t99, 4),
                    "h2d_touched_bytes": tbytes})
    res["clocks"] = clk
    res["timing"] = ("CUDA events around each CUDA-graph replay (K1+K2 fused, "
                     "tp_plan_tile); h2d_* add the pinned upload of the image (or of its "
                     "touched rows) before the replay; 50 warm-up iterations dropped")
    return res


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


def run_single(args, dist, device, which: str) -> dict:
    """C1 (1920x1080, E=512, fp32) / C3 (3840x2160, E=448, bf16): batch-1 latency on
    rank 0's GPU, with the CPU path's batch-1 latency on one host core beside it."""
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.workloads import c1, c3, workload_bytes

    wl = c1() if which == "c1" else c3()
    cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                           std=wl.std, reduced_precision_normalize=wl.bf16)
    lat = batch1_latency(cfg, wl.wh, device, max(args.latency_iters, 1000))
    res = {"workload": wl.name + ": " + wl.description,
           "value": round(1e3 / lat["p50_ms"], 2), "unit": UNIT, **lat,
           "algorithmic_bytes": workload_bytes(wl)["total"]}
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_latency(wl)
    return res


def run_sweep(args, dist, device, which: str = "c4", steps: int | None = None,
              warmup: int | None = None) -> dict:
    """C4 (8192 mixed-aspect images, LPT-sharded over the ranks; strong scaling) or C5
    (1024 of those images + device tokenization and placeholder expansion).  Inputs are
    generated on device before timing; a step processes the rank's whole shard in
    chunks of 2048 images."""
    import torch

    from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.sharding import imbalance, shard
    from paper_2603_16987_b200.tokenizer import PlaceholderExpander
    from paper_2603_16987_b200.workloads import Workload, c4, workload_bytes

    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    total = 8192 if which == "c4" else 1024
    wl_all = c4(total)
    idx = shard(wl_all.wh, wl_all.tile_edge, wl_all.max_tiles, dist.rank, dist.world)
    wh = wl_all.wh[idx]
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=wl_all.mean, std=wl_all.std,
                           reduced_precision_normalize=True)
    # chunks of 2048 images (inputs of the whole shard stay resident, one 2048-image
    # output buffer is reused): per-chunk K1 and tail cost twice as rare as with 1024
    chunk = 2048
    stream = torch.cuda.Stream(device)
    chunks = [synth_packed(wh[c0:c0 + chunk], 3, device, seed=wl_all.seed + c0, kind=0)
              for c0 in range(0, len(idx), chunk)]
    prep = TilePreprocessor(cfg, device)
    outs = prep(chunks[0], capacity=chunk * 13)
    torch.cuda.synchronize(device)
    with_expand = which == "c5"
    if with_expand:
        # rendered prompts tokenized on the device (K6), then expanded with the tile
        # counts straight from K1 (K3): ids never leave the GPU
        from paper_2603_16987_b200.tokenizer import DeviceTokenizer, parse_vocab
        from paper_2603_16987_b200.workloads import c5_texts, synthetic_vocab_text

        vocab = parse_vocab(synthetic_vocab_text(), "synthetic")
        n = len(idx)
        tok = DeviceTokenizer(vocab, device)
        texts = tok.upload([c5_texts(total, wl_all.seed)[i] for i in idx])
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
            else:
                # steady state as C2: K1 is a programmatic dependent of the previous
                # chunk's K2 (it waits for it before writing the plans), K2 of K1
                prep.plan(ch, outs.plans, stream, after_kernel=True)
                prep.tile(ch, outs.plans, outs.pixel_values, None, stream, after_plan=True)
            if with_expand:
                exp(toks.ids, toks.off, outs.plans.n_images, count_off, cap, out=ex,
                    stream=stream)

    ms, clk = _timed(step, steps, warmup, stream, device, dist)
    ms_step = ms / steps
    wl = Workload(wl_all.name, wl_all.description, wh, 448, 12, wl_all.mean, wl_all.std, True,
                  wl_all.seed)
    wb = workload_bytes(wl)  # this rank's shard
    peak = measured_peak()
    achieved = wb["total"] / (ms_step / 1e3) / 1e9
    res = {"workload": ("C4: " if not with_expand else "C5: ") + wl_all.description
           + (" + device tokenization of rendered prompts (K6) and image-token"
              " expansion (256 tokens/tile, K3)" if with_expand else ""),
           "value": round(total * steps / (ms / 1e3), 2), "unit": UNIT,
           "n_gpus": dist.world, "scaling": "strong", "steps": steps, "warmup": warmup,
           "ms_per_step": round(ms_step, 4), "images_total": total,
           "images_per_rank": len(idx), "parallelism": f"dp{dist.world} LPT shards",
           "lpt_imbalance": round(imbalance(wl_all.wh, 448, 12, dist.world), 4),
           "l2": "inputs larger than L2",
           "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak[0],
                        "unit": "GB/s", "frac": round(achieved / peak[0], 4),
                        "bytes_per_step_rank0": wb["total"],
                        "note": "per GPU: rank 0's shard bytes / the max-over-ranks step "
                                "time, whole step (K1+K2" + ("+K6+K3" if with_expand else "")
                                + ")"},
           "gpu_launches": steps * len(chunks) * (8 if with_expand else 2),
           "clocks": clk}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu_texts = None
        if with_expand:
            from paper_2603_16987_b200.workloads import c5_texts
            cpu_texts = c5_texts(total, wl_all.seed)
        res["cpu_baseline"] = cpu_throughput_wl(wl_all, host_cores(), args.cpu_seconds,
                                                cpu_texts)
    del chunks, outs
    torch.cuda.empty_cache()
    return res


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    args = parse_args(argv)
    rc = maybe_spawn(args, argv)
    if rc is not None:
        sys.exit(rc)
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
        return

    import torch

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    dev_index = dist.device_index(torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    dist.init("nccl")

    if args.workload != "c2":  # one config alone as the line's workload
        if args.workload in ("c4", "c5"):
            r = run_sweep(args, dist, device, args.workload)
        else:
            r = run_single(args, dist, device, args.workload) if dist.rank == 0 else None
        if dist.rank == 0:
            line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": dist.world,
                    "steps": r.get("steps", args.latency_iters), "warmup": args.warmup,
                    "higher_is_better": True, "scaling": r.get("scaling", "weak"),
                    "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
                    "config": {"workload": r["workload"]}, **{k: v for k, v in r.items()
                                                             if k not in ("value", "workload")}}
            print(json.dumps(dist.tag(line)), flush=True)
        dist.close()
        return

    r = run_c2(args, dist, device, dev_index)
    wl, wb = r["wl"], r["wb"]
    latency = batch1_latency(r["cfg"], [[1920, 1080]], device, args.latency_iters) \
        if dist.rank == 0 else None
    sub = {}
    if not args.no_sub:
        # every rank runs the sharded sweeps; only rank 0 runs the batch-1 configs
        sub["c4"] = run_sweep(args, dist, device, "c4", steps=5, warmup=3)
        sub["c5"] = run_sweep(args, dist, device, "c5", steps=20, warmup=3)
        if dist.rank == 0:
            sub["c3"] = run_single(args, dist, device, "c3")
            sub["c1"] = run_single(args, dist, device, "c1")
            sub["dropin"] = run_dropin(args, device)

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_throughput_wl(wl, host_cores(), args.cpu_seconds)

    traffic = measured_traffic("tp_tile", wb["total"])
    if dist.rank == 0:
        bytes_per_launch = wb["total"]
        achieved = bytes_per_launch / (r["k2_ms"] / 1e3) / 1e9
        peak = measured_peak()
        n_sub_launches = sum(v.get("gpu_launches", 0) for v in sub.values())
        line = {
            "metric": METRIC, "value": round(r["value"], 2), "unit": UNIT,
            "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(r["ms_step"], 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {**c2_config(wl, r["n"], dist.world), "tiles_per_gpu": r["n_tiles"]},
            "p50_ms": latency["p50_ms"] if latency else None,
            "latency": latency,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak[0],
                         "unit": "GB/s", "frac": round(achieved / peak[0], 4),
                         "traffic": traffic, "peak_source": peak[1],
                         "kernel": "tp_tile (K2)", "kernel_ms": round(r["k2_ms"], 4),
                         "kernel_timing": "CUDA events around K back-to-back K2 launches, "
                                          "same stream and inputs, after the timed steps",
                         "bytes_per_launch": bytes_per_launch,
                         "bytes_full_image": int(wb["read_full"] + wb["write"]),
                         "peak_nominal_gbs": 8000.0,
                         "frac_of_nominal": round(achieved / 8000.0, 4),
                         "kernel_ms_smooth_content": round(r["k2_smooth_ms"], 4),
                         "frac_smooth_content": round(bytes_per_launch / (r["k2_smooth_ms"] / 1e3)
                                                      / 1e9 / peak[0], 4),
                         "content": "uniform-noise pixels (every value a fresh byte: the most "
                                    "exact-fp64 fallbacks); *_smooth_content = the same launch "
                                    "on smooth synthetic images"},
            "cpu_baseline": cpu,
            "e2e": r["e2e"],
            "e2e_jpeg": r["e2e_jpeg"],
            "e2e_png": r["e2e_png"],
            "gpu_launches": 2 * args.steps,
            "gpu_launches_sub_blocks": n_sub_launches,
            "clocks": r["clk"],
            **sub,
        }
        print(json.dumps(dist.tag(line)), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
