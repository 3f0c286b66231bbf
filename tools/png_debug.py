"""Diagnostics for K8 (device PNG decode): per-unit records and image status of one
batch, next to what zlib says about the stream."""
import sys
import zlib
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

from png_cases import bad_cases, custom_cases, pil_cases
from paper_2603_16987_b200 import png as P

names = sys.argv[1:] if __name__ == "__main__" else []
dec = P.PngDecoder(torch.device("cuda:0"))
for name in names:
    payload = dict(bad_cases() + custom_cases() + pil_cases())[name]
    info, offs, lens = P.parse(payload)
    z = b"".join(payload[o: o + n] for o, n in zip(offs.tolist(), lens.tolist()))
    try:
        d = zlib.decompressobj()
        raw = d.decompress(z)
        zs = f"zlib ok len {len(raw)} eof {d.eof} adler {zlib.adler32(raw):08x}"
    except Exception as e:
        zs = f"zlib: {e}"
    batch = dec.decode([payload], sync=False)
    sl, n, totals, out = dec._last
    torch.cuda.synchronize()
    st = sl.status[:n].cpu().numpy()
    U = int(totals[0])
    rec = sl.work[int(totals[3]): int(totals[3]) + U * 80].cpu().numpy().view(np.int64).reshape(U, 10)
    print(name, "status", st, zs, "trailer", z[-4:].hex(), "zlib_len", len(z))
    for u in range(U):
        r = rec[u]
        i32 = r[4:8].view(np.int32)
        print(f"  unit {u}: start {r[0]} end {r[1]} out_len {r[2]} out_off {r[3]} ntok {i32[0]} "
              f"status {i32[1]} final {i32[2]} dirty {i32[3]} stored {i32[4]} final_end {r[8]}")


def unit_stats(payload):
    """Valid units, and the longest unit (tokens, inflated bytes) of one payload."""
    dec.decode([payload], sync=False)
    sl, n, totals, out = dec._last
    torch.cuda.synchronize()
    U = int(totals[0])
    rec = sl.work[int(totals[3]): int(totals[3]) + U * 80].cpu().numpy().view(np.int64).reshape(U, 10)
    valid = rec[:, 0] >= 0
    i32 = rec[:, 4:8].view(np.int32).reshape(U, 8)
    runs = "".join("x" if v else "." for v in valid).split("x")
    return {"units": U, "valid": int(valid.sum()), "max_ntok": int(i32[:, 0].max()),
            "max_out": int(rec[:, 2].max()), "mean_out": float(rec[valid, 2].mean()),
            "stored_starts": int(i32[:, 4].sum()), "max_invalid_run": max(len(r) for r in runs),
            "fixups": int(i32[:, 6].sum()), "rounds": int(i32[:, 7].sum()),
            "markers": int(i32[:, 5].sum())}
