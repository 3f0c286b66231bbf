"""Probe: staged upload + engine (PDL K1->K2) vs reference path, repeated."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np, torch
from golden_data import IMAGENET_MEAN, IMAGENET_STD, make_input
from paper_2603_16987_b200.engine import TilePreprocessor, pack_images, PackedImages
from paper_2603_16987_b200.imgproc import PreprocessConfig
from paper_2603_16987_b200.transfer import HostArena, stage_images, staged_bytes, upload_images

mode = sys.argv[1]
DEV = torch.device("cuda:0")
CFG = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                       reduced_precision_normalize=True)
prep = TilePreprocessor(CFG, DEV)
sizes = [(1080, 1920), (480, 640), (517, 333), (2160, 3840), (300, 700), (64, 64)]
bad = 0
for it in range(int(sys.argv[2])):
    rng = np.random.default_rng(it)
    imgs = [make_input(*sizes[int(rng.integers(len(sizes)))], 3, "random", it * 10 + i) for i in range(int(rng.integers(1, 7)))]
    ref = prep(pack_images(imgs).to(DEV))
    arena = HostArena(capacity=staged_bytes(imgs), alignment=256)
    staged = stage_images(imgs, arena)
    dest = torch.empty(staged_bytes(imgs), dtype=torch.uint8, device=DEV)
    packed, done = upload_images(staged, dest)
    if mode == "separate":
        packed = PackedImages(dest, packed.offsets.clone(), packed.wh.clone(), packed.channels, packed.wh_host, packed.offsets_host)
    if mode == "split":
        out = prep.alloc_outputs(3, len(imgs) * 13)
        from paper_2603_16987_b200.engine import TileBatch
        tb = TileBatch(prep.alloc_plans(len(imgs)), out[0], out[1])
        prep.plan(packed, tb.plans)
        torch.cuda.synchronize()
        prep.tile(packed, tb.plans, tb.pixel_values, None, after_plan=False)
        o = tb
    else:
        o = prep(packed)
    torch.cuda.synchronize()
    T = ref.num_tiles()
    ok = o.num_tiles() == T and torch.equal(o.pixel_values[:T].view(torch.int16), ref.pixel_values[:T].view(torch.int16))
    if not ok:
        bad += 1
        if bad < 4:
            print("mismatch it", it, [a.shape for a in imgs], o.num_tiles(), T, o.plans.plan.cpu().numpy().tolist()[:3], ref.plans.plan.cpu().numpy().tolist()[:3], flush=True)
print(mode, "bad", bad)
