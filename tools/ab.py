"""A/B timing of K2 builds in one GPU session: for each round, every variant library
(build/variants/<name>/libtileprep.so) runs in its own process and times K2 on C2
(64 x 1080p, 200 launches) and on the first 1024 C4 images (20 launches), CUDA events.
Rounds interleave the variants so clock/thermal drift hits all of them alike.

  python tools/ab.py [rounds] > gpurun_out/ab.log
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import json, sys, torch
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed
from paper_2603_16987_b200.imgproc import PreprocessConfig
from paper_2603_16987_b200.workloads import Workload, c2, c3, c4, workload_bytes
dev = torch.device("cuda:0")
res = {}
w3 = c3()
c3b = Workload("C3x32", "32 x 4K", np.repeat(w3.wh, 32, axis=0), w3.tile_edge, w3.max_tiles,
               w3.mean, w3.std, w3.bf16, w3.seed)
up = Workload("UP", "64 x 640x480 (3x4 upscaled)", np.repeat(np.array([[640, 480]], np.int32), 64, axis=0),
              448, 12, w3.mean, w3.std, True, 5)
tall = Workload("TALL", "64 x 1080x1920 portrait", np.repeat(np.array([[1080, 1920]], np.int32), 64, axis=0),
                448, 12, w3.mean, w3.std, True, 6)
import os
sel = os.environ.get("ABW", "c2,c4k,c3x32").split(",")
for name, wl, n in [x for x in (("c2", c2(), 200), ("c4k", c4(1024), 20), ("c3x32", c3b, 100),
                                ("up", up, 50), ("tall", tall, 100), ("c2s", c2(), 200))
                     if x[0] in sel]:
    cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                           std=wl.std, reduced_precision_normalize=wl.bf16)
    imgs = synth_packed(wl.wh, 3, dev, seed=wl.seed, kind=1 if name.endswith("s") else 0)
    prep = TilePreprocessor(cfg, dev)
    out = prep(imgs)
    torch.cuda.synchronize()  # synth + K1 ran on the default stream; the loops use s
    s = torch.cuda.Stream(dev)
    for _ in range(5):
        prep.tile(imgs, out.plans, out.pixel_values, None, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        prep.tile(imgs, out.plans, out.pixel_values, None, s)
    b.record(s)
    torch.cuda.synchronize()
    res[name + "_us"] = round(a.elapsed_time(b) / n * 1e3, 2)
    res[name + "_frac"] = round(workload_bytes(wl)["total"] / (res[name + "_us"] * 1e-6) / 6545.3e9, 4)
    a.record(s)
    for _ in range(n):
        prep.plan(imgs, out.plans, s, after_kernel=True)
        prep.tile(imgs, out.plans, out.pixel_values, None, s, after_plan=True)
    b.record(s)
    torch.cuda.synchronize()
    res[name + "_step_us"] = round(a.elapsed_time(b) / n * 1e3, 2)
    del imgs, out
print(json.dumps(res))
"""


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    # ABW=c2,c4k,c3x32,up,tall,c2s selects the workloads (default: c2,c4k,c3x32);
    # c2s is C2 on smooth synthetic content (kind 1), which flags more exact ties
    variants = sorted(p for p in (ROOT / "build" / "variants").glob("*/libtileprep.so"))
    if os.environ.get("ABV"):  # ABV=name,name selects the variants
        keep = os.environ["ABV"].split(",")
        variants = [p for p in variants if p.parent.name in keep]
    results = {p.parent.name: [] for p in variants}
    for r in range(rounds):
        for lib in variants:
            env = dict(os.environ, TILEPREP_LIB=str(lib))
            out = subprocess.run([sys.executable, "-c", CHILD % {"root": str(ROOT)}], env=env,
                                 capture_output=True, text=True, timeout=600)
            line = out.stdout.strip().splitlines()[-1] if out.returncode == 0 else None
            rec = json.loads(line) if line else {"error": out.stderr[-400:]}
            results[lib.parent.name].append(rec)
            print(json.dumps({"round": r, "variant": lib.parent.name, **rec}), flush=True)
    summary = {}
    for name, recs in results.items():
        ok = [x for x in recs if "error" not in x]
        if ok:
            summary[name] = {k: round(min(x[k] for x in ok), 2) for k in ok[0]}
    print(json.dumps({"summary_min": summary}))


if __name__ == "__main__":
    main()
