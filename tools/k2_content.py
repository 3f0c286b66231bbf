"""K2 on the C2 batch (64 x 1080p, E=448, ImageNet, bf16 NCHW) by pixel content:
uniform noise (the bench headline's input), smooth synthetic (tp_synth kind 1) and
corpus-like scenes (smooth gradients + blocks + Gaussian noise sigma 10, the content model
of the reference's make_corpus.py).  CUDA events around back-to-back K2 launches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

from jpeg_cases import scene
from paper_2603_16987_b200.engine import TilePreprocessor, pack_images, synth_packed
from paper_2603_16987_b200.imgproc import PreprocessConfig
from paper_2603_16987_b200.workloads import c2

wl = c2(64)
cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                       std=wl.std, reduced_precision_normalize=wl.bf16)
dev = torch.device("cuda:0")
prep = TilePreprocessor(cfg, dev)
stream = torch.cuda.Stream(dev)
ALG = 561512448


def time_k2(images, iters=200):
    out = prep(images)
    torch.cuda.synchronize()
    for _ in range(5):
        prep.tile(images, out.plans, out.pixel_values, None, stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        prep.tile(images, out.plans, out.pixel_values, None, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return ms


res = {}
res["noise"] = time_k2(synth_packed(wl.wh, 3, dev, seed=wl.seed, kind=0))
res["smooth"] = time_k2(synth_packed(wl.wh, 3, dev, seed=wl.seed, kind=1))
arrs = [scene(int(w), int(h), 1000 + i) for i, (w, h) in enumerate(wl.wh)]
res["scene"] = time_k2(pack_images(arrs).to(dev))
for k, ms in res.items():
    print(f"{k:8s} K2 {ms * 1e3:7.1f} us  {ALG / ms / 1e6:7.1f} GB/s  frac {ALG / ms / 1e6 / 6551:.3f}")
