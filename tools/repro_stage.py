"""Repro: staged upload (H2D) immediately followed by K1/K2."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np, torch
from golden_data import IMAGENET_MEAN, IMAGENET_STD, make_input
from paper_2603_16987_b200.engine import TilePreprocessor, pack_images
from paper_2603_16987_b200.imgproc import PreprocessConfig
from paper_2603_16987_b200.transfer import HostArena, stage_images, staged_bytes, upload_images

mode = sys.argv[1]
DEV = torch.device("cuda:0")
CFG = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                       reduced_precision_normalize=True)
rng = np.random.default_rng(3)
sizes = [(1080, 1920), (480, 640), (517, 333), (2160, 3840), (300, 700), (64, 64)]
imgs = [make_input(*sizes[int(rng.integers(len(sizes)))], 3, "random" if i % 2 else "smooth", 300 + i) for i in range(6)]
print([a.shape for a in imgs])
arena = HostArena(capacity=staged_bytes(imgs), alignment=256)
staged = stage_images(imgs, arena)
dest = torch.empty(staged_bytes(imgs), dtype=torch.uint8, device=DEV)
packed, done = upload_images(staged, dest)
if mode == "sync":
    torch.cuda.synchronize()
print("wh", packed.wh.cpu().numpy().tolist(), "off", packed.offsets.cpu().numpy().tolist() if mode == "sync" else "")
prep = TilePreprocessor(CFG, DEV)
out = prep(packed)
torch.cuda.synchronize()
print("tiles", out.num_tiles(), out.plans.plan.cpu().numpy().tolist())
if len(sys.argv) > 2:
    ref = prep(pack_images(imgs).to(DEV))
    torch.cuda.synchronize()
    T = ref.num_tiles()
    print("ref tiles", T, torch.equal(out.pixel_values[:T].view(torch.int16), ref.pixel_values[:T].view(torch.int16)))
