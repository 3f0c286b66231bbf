"""Where does a C2 step's time go?  Times K1 alone, K2 alone and K1+K2 back to back
(CUDA events around 200 launches each, device resident) so the gap between the bench's
ms_per_step and K2's event time can be attributed."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed  # noqa: E402
from paper_2603_16987_b200.imgproc import PreprocessConfig  # noqa: E402
from paper_2603_16987_b200.workloads import c2  # noqa: E402

wl = c2()
cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean, std=wl.std,
                       reduced_precision_normalize=wl.bf16)
dev = torch.device("cuda:0")
images = synth_packed(wl.wh, 3, dev, seed=wl.seed, kind=0)
prep = TilePreprocessor(cfg, dev)
out = prep(images)
stream = torch.cuda.Stream(dev)
torch.cuda.synchronize()


def timeit(fn, n=200):
    with torch.cuda.stream(stream):
        for _ in range(5):
            fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(n):
            fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


res = {
    "k1_us": timeit(lambda: prep.plan(images, out.plans, stream)),
    "k2_us": timeit(lambda: prep.tile(images, out.plans, out.pixel_values, None, stream)),
    "k1k2_us": timeit(lambda: (prep.plan(images, out.plans, stream),
                               prep.tile(images, out.plans, out.pixel_values, None, stream))),
}
# CUDA graph of K1+K2 (no host launch cost)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(stream):
    prep.plan(images, out.plans, stream)
    prep.tile(images, out.plans, out.pixel_values, None, stream)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        prep.plan(images, out.plans, stream)
        prep.tile(images, out.plans, out.pixel_values, None, stream)
res["k1k2_graph_us"] = timeit(lambda: g.replay())
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
