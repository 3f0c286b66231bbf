"""Batch-1 latency pieces (C3: 1 x 3840x2160, E=448, bf16): CUDA-graph replays of K1
alone, K2 alone and K1+K2, p50 over 500 replays each."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed  # noqa: E402
from paper_2603_16987_b200.imgproc import PreprocessConfig  # noqa: E402
from paper_2603_16987_b200.workloads import c1, c3  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for wl in (c3(), c1()):
    cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                           std=wl.std, reduced_precision_normalize=wl.bf16)
    img = synth_packed(wl.wh, 3, dev, seed=wl.seed, kind=0)
    prep = TilePreprocessor(cfg, dev)
    out = prep(img)
    s = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    graphs = {}
    for name, fn in (("k1", lambda: prep.plan(img, out.plans, s)),
                     ("k2", lambda: prep.tile(img, out.plans, out.pixel_values, None, s)),
                     ("k1k2", lambda: prep(img, out=out, stream=s))):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                fn()
        graphs[name] = g
    for name, g in graphs.items():
        ts = []
        for k in range(600):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                g.replay()
            b.record(s)
            b.synchronize()
            if k >= 100:
                ts.append(a.elapsed_time(b) * 1e3)
        res[f"{wl.name}_{name}_p50_us"] = round(float(np.median(ts)), 2)
    # empty graph-replay baseline (event overhead)
    g = torch.cuda.CUDAGraph()
    x = torch.zeros(1, device=dev)
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            x.add_(1)
    ts = []
    for k in range(600):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            g.replay()
        b.record(s)
        b.synchronize()
        if k >= 100:
            ts.append(a.elapsed_time(b) * 1e3)
    res["tiny_kernel_graph_p50_us"] = round(float(np.median(ts)), 2)
print(json.dumps(res))
