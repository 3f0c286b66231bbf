"""Batch-1 device JPEG decode latency (the drop-in preprocess path) over sub_bits /
lead-in: one corpus-like 1080p q85 JPEG, JpegDecoder.decode wall time (host parse +
H2D + K7 + status readback), p50 over 100 calls."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_16987_b200.jpeg import JpegDecoder  # noqa: E402
from paper_2603_16987_b200.workloads import jpeg_payloads  # noqa: E402

p = jpeg_payloads(1)
for spec in sys.argv[1:] or ["0", "4096", "2048:2048", "1024:1024", "512:1024"]:
    sb, _, lead = spec.partition(":")
    dec = JpegDecoder("cuda:0", sub_bits=int(sb), lead_bits=int(lead or 0))
    for _ in range(10):
        dec.decode(p)
    ts = []
    for _ in range(100):
        t0 = time.perf_counter()
        dec.decode(p)
        ts.append((time.perf_counter() - t0) * 1e3)
    s = torch.cuda.current_stream()
    ks = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dec.launch(s)
        b.record(s)
        b.synchronize()
        ks.append(a.elapsed_time(b))
    print(f"{spec}: decode() p50 {np.median(ts):.3f} ms p99 {np.percentile(ts, 99):.3f} ms; "
          f"K7 kernels alone p50 {np.median(ks):.3f} ms", flush=True)
