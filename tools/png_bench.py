"""Device PNG decode throughput (K8) on 64 corpus-like 1080p PNGs written by Pillow
(default settings, the reference's re-encode path imgproc.py:252-256) and on 16 noise
PNGs: end to end through PngDecoder.decode (host chunk walk + pinned staging + H2D + K8 +
status readback, host clock), the K8 kernels alone (CUDA events around relaunches), and
Pillow (the reference's decoder) on all host cores.

    python tools/png_bench.py
"""
import io
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from png_cases import content, pil_png  # noqa: E402
from paper_2603_16987_b200.png import PngDecoder  # noqa: E402

DEV = torch.device("cuda:0")


def _pil(p):
    from PIL import Image
    t0 = time.perf_counter()
    np.asarray(Image.open(io.BytesIO(p)).convert("RGB"))
    return time.perf_counter() - t0


def pil_rate(payloads):
    cores = len(os.sched_getaffinity(0))
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_pil, payloads[:cores])
        t0 = time.perf_counter()
        pool.map(_pil, payloads, chunksize=1)
        dt = time.perf_counter() - t0
    return len(payloads) / dt, cores


def run(name, payloads, iters=10):
    dec = PngDecoder(DEV)
    for _ in range(2):
        dec.decode(payloads)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        dec.decode(payloads)
    torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) / iters
    s = torch.cuda.current_stream(DEV)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(iters):
        dec.launch(s)
    b.record(s)
    torch.cuda.synchronize()
    k = a.elapsed_time(b) / iters
    st = dec.last_status()
    sl, n, totals, out = dec._last
    return {"set": name, "images": len(payloads),
            "avg_kb": round(sum(map(len, payloads)) / len(payloads) / 1e3, 1),
            "e2e_ms": round(e2e * 1e3, 3), "e2e_images_s": round(len(payloads) / e2e, 1),
            "kernel_ms": round(k, 3), "kernel_images_s": round(len(payloads) / (k / 1e3), 1),
            "units": int(totals[0]), "device_status_nonzero": int((st != 0).sum()),
            "fallback": dec.last_fallback, "h2d_bytes": dec.last_h2d_bytes}


def main():
    scenes = [pil_png(content("scene", 1920, 1080, 1000 + i)) for i in range(64)]
    noise = [pil_png(content("noise", 1920, 1080, 2000 + i)) for i in range(16)]
    res = [run("scene_1080p_x64", scenes), run("noise_1080p_x16", noise),
           run("scene_1080p_x1", scenes[:1])]
    for r, pl in zip(res, (scenes, noise, scenes[:1])):
        rate, cores = pil_rate(pl if len(pl) > 1 else pl * 16)
        r["pillow_images_s"] = round(rate, 1)
        r["pillow_cores"] = cores
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
