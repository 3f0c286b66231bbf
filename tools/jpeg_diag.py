"""Device JPEG decode diagnostics: half-rounds the parallel Huffman sync needed, host
fallbacks and decode time, over sub_bits, for corpus-like 1080p images and noise."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from jpeg_cases import encode, pil_rgb, scene  # noqa: E402
from paper_2603_16987_b200.jpeg import JpegDecoder  # noqa: E402

DEV = torch.device("cuda:0")
imgs = {"scene1080_q85": [encode(scene(1920, 1080, s)) for s in range(8)],
        "noise1080_q85": [encode(np.random.default_rng(s).integers(0, 256, (1080, 1920, 3), dtype=np.uint8))
                          for s in range(4)]}
for name, pl in imgs.items():
    for sb in (1024, 2048, 4096, 8192, 16384):
        dec = JpegDecoder(DEV, sub_bits=sb)
        pk = dec.decode(pl)
        steps = int(dec._work[4092:4096].view(torch.int32).item())
        ok = all(np.array_equal(pk.data[int(o): int(o) + 1920 * 1080 * 3].cpu().numpy().reshape(1080, 1920, 3),
                                pil_rgb(p)) for o, p in zip(pk.offsets_host, pl))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            dec.decode(pl)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 5 * 1e3
        print(f"{name} sub_bits={sb}: half-rounds {steps}, fallback {dec.last_fallback}, exact {ok}, "
              f"{ms:.2f} ms / {len(pl)} images (incl. host parse + H2D), {sum(map(len, pl)) / len(pl) / 1e3:.0f} KB avg",
              flush=True)
