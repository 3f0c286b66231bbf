"""Device JPEG decode throughput (K7) on 64 corpus-like 1080p q85 JPEGs (and noise):
end to end through JpegDecoder.decode (host parse + pinned staging + H2D + K7 + status
readback, host clock) and the K7 kernels alone (CUDA events around relaunches), against
Pillow (the reference's decoder) on all host cores.

    python tools/jpeg_bench.py [sub_bits[:lead_bits] ...]   (default: the decoder's choice)
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
from jpeg_cases import encode, scene  # noqa: E402
from paper_2603_16987_b200.jpeg import JpegDecoder  # noqa: E402

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
        pool.map(_pil, payloads * 2, chunksize=1)
        dt = time.perf_counter() - t0
    return 2 * len(payloads) / dt, cores


def run(name, payloads, spec):
    sub_bits, _, lead = str(spec).partition(":")
    sub_bits, lead = int(sub_bits), int(lead or 0)  # 0: the decoder's choice
    dec = JpegDecoder(DEV, sub_bits=sub_bits, lead_bits=lead)
    for _ in range(3):
        dec.decode(payloads)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    iters = 10
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
    steps = int(dec._work[4092:4096].view(torch.int32).item())
    st = dec._work[3968:3968 + 40].view(torch.int64).cpu().numpy()
    cnt = dec._work[:4096].view(torch.int32).cpu().numpy()
    ts = dec._work[640 * 4: 640 * 4 + 64 * 8].view(torch.int64).cpu().numpy()
    rounds = [(h, int(cnt[512 + h]), int(cnt[h]), round((ts[h] - (ts[h - 1] if h > 2 else st[1])) / 1e3, 1),
               int(cnt[256 + h]), int(cnt[384 + h]))
              for h in range(2, steps + 1) if h < 64]
    phases = {"spec_us": (st[1] - st[0]) / 1e3, "rounds_us": (st[2] - st[1]) / 1e3,
              "scan_us": (st[3] - st[2]) / 1e3, "write_us": (st[4] - st[3]) / 1e3}
    return {"set": name, "sub_bits": sub_bits, "lead_bits": lead, "images": len(payloads),
            "avg_kb": round(sum(map(len, payloads)) / len(payloads) / 1e3, 1),
            "e2e_ms": round(e2e * 1e3, 3), "e2e_images_s": round(len(payloads) / e2e, 1),
            "kernel_ms": round(k, 3), "kernel_images_s": round(len(payloads) / (k / 1e3), 1),
            "half_rounds": steps, "rounds(h,decoded,changed,us,max_symbols,max_cycles)": rounds, "huff_phases": {k: round(float(v), 1) for k, v in phases.items()}, "fallback": dec.last_fallback,
            "h2d_bytes": dec.last_h2d_bytes}


def main():
    subs = sys.argv[1:] or ["0"]  # sub_bits[:lead_bits]; 0: the decoder's own choice by batch size
    sets = {"scene1080_q85": [encode(scene(1920, 1080, s)) for s in range(64)],
            "noise1080_q85": [encode(np.random.default_rng(s).integers(0, 256, (1080, 1920, 3),
                                                                        dtype=np.uint8)) for s in range(16)]}
    for name, pl in sets.items():
        rate, cores = pil_rate(pl)
        print(json.dumps({"set": name, "pillow_images_s": round(rate, 1), "cores": cores}), flush=True)
        for sb in subs:
            print(json.dumps(run(name, pl, sb)), flush=True)


if __name__ == "__main__":
    main()
