"""Decode the 64 corpus-like 1080p q85 JPEGs of the bench a few times (a driver for ncu
captures of the K7 kernels: `ncu --set full -k regex:k_jpeg_color -c 1 python
tools/jpeg_once.py`)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_16987_b200.jpeg import JpegDecoder  # noqa: E402
from paper_2603_16987_b200.workloads import jpeg_payloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
payloads = jpeg_payloads(n, seed=20260817)
dec = JpegDecoder(torch.device("cuda:0"))
for _ in range(reps):
    dec.decode(payloads)
torch.cuda.synchronize()
print("decoded", n, "x", reps, "fallbacks", dec.last_fallback)
