"""Randomized parity stress on the GPU (minutes, not a unit test): for random batches of
random sizes, tilings, dtypes and layouts, the fast K2 must equal the exact-fp64 K2 byte
for byte, the fused small-batch launch must equal the two-launch path, and touched-row
uploads must equal whole-image uploads.  Prints one JSON summary line.

    python tools/stress_parity.py [rounds] > gpurun_out/stress.json
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_16987_b200.engine import TilePreprocessor, pack_images  # noqa: E402
from paper_2603_16987_b200.imgproc import PreprocessConfig  # noqa: E402
from paper_2603_16987_b200.transfer import (HostArena, stage_images, staged_bytes,  # noqa: E402
                                            upload_images)

DEV = torch.device("cuda:0")


def same(a, b):
    T = int(a.plans.tile_off[-1])
    if T != int(b.plans.tile_off[-1]) or not torch.equal(a.plans.plan, b.plans.plan):
        return False
    for x, y in ((a.pixel_values, b.pixel_values), (a.pixel_u8, b.pixel_u8)):
        if x is not None and not torch.equal(x[:T].view(torch.uint8), y[:T].view(torch.uint8)):
            return False
    return True


def main(rounds: int):
    rng = np.random.default_rng(2026)
    stats = {"rounds": 0, "images": 0, "tiles": 0, "fast_vs_exact": 0, "fused_vs_two": 0,
             "touched_vs_full": 0, "failures": []}
    t0 = time.time()
    for r in range(rounds):
        n = int(rng.integers(1, 9))
        c = int(rng.choice([1, 3]))
        e = int(rng.choice([32, 224, 336, 448, 512]))
        mt = int(rng.integers(1, 13))
        kind = int(rng.integers(0, 2))
        imgs = []
        for _ in range(n):
            hi = 4200 if rng.random() < 0.2 else 1400
            w, h = int(rng.integers(1, hi)), int(rng.integers(1, hi))
            if kind:
                yy, xx = np.mgrid[0:h, 0:w]
                base = ((xx * 7 + yy * 3) % 256).astype(np.uint8)
                imgs.append(np.repeat(base[:, :, None], c, axis=2))
            else:
                imgs.append(rng.integers(0, 256, (h, w, c), dtype=np.uint8))
        bf16 = bool(rng.integers(0, 2))
        layout = str(rng.choice(["NCHW", "NHWC"]))
        cfg = PreprocessConfig(tile_edge=e, max_tiles=mt, mean=(0.48, 0.45, 0.41)[:c] if c == 3 else (0.5,),
                               std=(0.23, 0.22, 0.23)[:c] if c == 3 else (0.25,),
                               reduced_precision_normalize=bf16)
        packed = pack_images(imgs).to(DEV)
        fast = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=True)(packed)
        exact = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=True, algo="exact")(packed)
        two = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=True, fuse_small=False)(packed)
        nbytes = staged_bytes(imgs, touched=(e, mt))
        staged = stage_images(imgs, HostArena(nbytes, 256, pin=True), touched=(e, mt))
        rows, _ = upload_images(staged, torch.empty(nbytes, dtype=torch.uint8, device=DEV))
        via_rows = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=True)(rows)
        torch.cuda.synchronize()
        desc = {"round": r, "n": n, "c": c, "e": e, "mt": mt, "kind": kind, "bf16": bf16,
                "layout": layout}
        for key, a, b in (("fast_vs_exact", fast, exact), ("fused_vs_two", fast, two),
                          ("touched_vs_full", via_rows, fast)):
            if same(a, b):
                stats[key] += 1
            else:
                stats["failures"].append(dict(desc, check=key))
        stats["rounds"] += 1
        stats["images"] += n
        stats["tiles"] += int(fast.plans.tile_off[-1])
    stats["seconds"] = round(time.time() - t0, 1)
    from paper_2603_16987_b200 import _lib

    lib = _lib.load()
    if hasattr(lib, "tp_debug_checks"):  # bounds-checked build (TP_CHECKS=1)
        stats["check_bits"] = int(lib.tp_debug_checks(1))
    print(json.dumps(stats))
    return 0 if not stats["failures"] and not stats.get("check_bits") else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 200))
