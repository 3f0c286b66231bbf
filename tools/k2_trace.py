"""Per-phase timing of K2 on C2 (or C3: K2_TRACE_WL=c3) from a TP_K2_TRACE=1 build (clock64 stamps, same SM):
how long consumers wait for data, whether waits cluster at item starts, producer
planning time.  TILEPREP_LIB must point at the trace build."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_16987_b200 import _lib  # noqa: E402
from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed  # noqa: E402
from paper_2603_16987_b200.imgproc import PreprocessConfig  # noqa: E402
from paper_2603_16987_b200.workloads import c2, c3  # noqa: E402

lib = _lib.load()
wl = c3() if os.environ.get("K2_TRACE_WL") == "c3" else c2()
cfg = PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean, std=wl.std,
                       reduced_precision_normalize=wl.bf16)
imgs = synth_packed(wl.wh, 3, "cuda:0", seed=wl.seed, kind=0)
prep = TilePreprocessor(cfg, "cuda:0")
out = prep(imgs)
for _ in range(3):
    prep(imgs, out=out)
torch.cuda.synchronize()
lib.tp_debug_k2_trace_clear()
prep(imgs, out=out)
torch.cuda.synchronize()
buf = np.zeros((296, 96, 6), dtype=np.uint64)
assert lib.tp_debug_k2_trace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int64(buf.nbytes)) == 0
t = buf.astype(np.float64)
valid = t[:, :, 5] > 0
flags = buf[:, :, 0]
first = (flags & 1) == 1
thumb = (flags & 2) == 2
nrows = (flags >> 8).astype(np.int64)
plan = (t[:, :, 2] - t[:, :, 1])[valid]
wait = (t[:, :, 4] - t[:, :, 3])[valid]
work = (t[:, :, 5] - t[:, :, 4])[valid]
start = t[:, 0, 3]
end = np.array([t[c, valid[c], 5].max() if valid[c].any() else t[c, 0, 3] for c in range(296)])
res = {
    "workload": wl.name,
    "phases": int(valid.sum()),
    "cycles_per_cta_p50": float(np.median(end - start)),
    "cta_span_min_max": [float((end - start).min()), float((end - start).max())],
    "wait_share": float(wait.sum() / (wait.sum() + work.sum())),
    "wait_p50_p90": [float(np.percentile(wait, 50)), float(np.percentile(wait, 90))],
    "work_p50_p90": [float(np.percentile(work, 50)), float(np.percentile(work, 90))],
    "plan_p50_p90": [float(np.percentile(plan, 50)), float(np.percentile(plan, 90))],
    "wait_first_phase_of_item_mean": float((t[:, :, 4] - t[:, :, 3])[valid & first].mean()),
    "wait_other_phases_mean": float((t[:, :, 4] - t[:, :, 3])[valid & ~first].mean()),
    "first_phase_wait_per_cta_mean": float((t[:, 0, 4] - t[:, 0, 3]).mean()),
    "lag_issue_to_ready_p50": float(np.percentile((t[:, :, 4] - t[:, :, 2])[valid], 50)),
}
span = end - start
thumb_rows = np.array([(nrows[c] * (thumb[c] & valid[c])).sum() for c in range(296)])
all_rows = np.array([(nrows[c] * valid[c]).sum() for c in range(296)])
nph = valid.sum(axis=1)
res["rows_per_cta_min_max"] = [int(all_rows.min()), int(all_rows.max())]
res["corr_span_thumbrows"] = float(np.corrcoef(span, thumb_rows)[0, 1])
res["corr_span_phases"] = float(np.corrcoef(span, nph)[0, 1])
res["phases_per_cta_min_max"] = [int(nph.min()), int(nph.max())]
res["thumb_work_per_row"] = float(((t[:, :, 5] - t[:, :, 4])[valid & thumb]).sum() / nrows[valid & thumb].sum())
res["tile_work_per_row"] = float(((t[:, :, 5] - t[:, :, 4])[valid & ~thumb]).sum() / nrows[valid & ~thumb].sum())
res["thumb_wait_per_phase"] = float((t[:, :, 4] - t[:, :, 3])[valid & thumb].mean())
res["tile_wait_per_phase"] = float((t[:, :, 4] - t[:, :, 3])[valid & ~thumb].mean())
cta = np.zeros((296, 3), dtype=np.uint64)
assert lib.tp_debug_k2_cta(ctypes.c_void_p(cta.ctypes.data), ctypes.c_int64(cta.nbytes)) == 0
smid = cta[:, 0].astype(np.int64)
t0 = cta[:, 1].astype(np.float64)
t1 = cta[:, 2].astype(np.float64)
base = t0.min()
res["cta_start_ns_spread"] = float(t0.max() - t0.min())
res["cta_end_ns_min_p50_max"] = [float(t1.min() - base), float(np.median(t1) - base), float(t1.max() - base)]
sm_end = {}
for s_, e_ in zip(smid, t1 - base):
    sm_end[s_] = max(sm_end.get(s_, 0), e_)
ends = np.array(list(sm_end.values()))
res["sm_end_ns_min_p50_max"] = [float(ends.min()), float(np.median(ends)), float(ends.max())]
res["n_sms"] = len(sm_end)
print(json.dumps(res))
