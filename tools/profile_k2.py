"""Small driver for ncu: C2 (64 x 1080p, E=448, bf16 NCHW) K1+K2, a few steps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed  # noqa: E402
from paper_2603_16987_b200.imgproc import PreprocessConfig  # noqa: E402
from paper_2603_16987_b200.workloads import c2  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "auto"
wl = c2()
cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean, std=wl.std,
                       reduced_precision_normalize=wl.bf16)
images = synth_packed(wl.wh, 3, "cuda:0", seed=wl.seed, kind=0)
prep = TilePreprocessor(cfg, "cuda:0", algo=algo)
out = prep(images)
for _ in range(4):
    prep(images, out=out)
torch.cuda.synchronize()
print("ok", out.num_tiles())
