"""CPU oracle for the VLM preprocessing hot path — TEST INFRASTRUCTURE ONLY.

This module restates the reference algorithm (vlmfp, /root/reference/pkg/src)
in numpy so the CUDA path can be checked against it.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import it; the product package never does (it has no CPU fallback).

Pinning: tests/golden/make_golden.py runs the reference itself and commits its
outputs under tests/golden/; tests/test_oracle_golden.py checks every function
here against those vectors (and, where /root/reference is present, against
the live reference with hypothesis).  Each function cites the reference
file:line it restates.
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np

try:  # bf16 with round-to-nearest-even, as vlmfp/dtypes.py:41-43
    import ml_dtypes

    BF16 = np.dtype(ml_dtypes.bfloat16)
except ImportError:  # pragma: no cover - the image ships ml_dtypes
    BF16 = None


# ---------------------------------------------------------------------------
# planner

def plan_float(width: int, height: int, tile_edge: int, max_tiles: int) -> tuple:
    """select_tile_plan (imgproc.py:266-292): minimise the key
    (|log(w/h) - log(c/r)|, r*c, r) in float64 over all r*c <= max_tiles.
    Returns (rows, cols, tile_edge, thumb, resized_w, resized_h)."""
    if width < 1 or height < 1:
        raise ValueError("width and height must be >= 1")
    goal = math.log(width / height)
    best = None
    for r in range(1, max_tiles + 1):
        for c in range(1, max_tiles // r + 1):
            key = (abs(goal - math.log(c / r)), r * c, r)
            if best is None or key < best[0]:
                best = (key, r, c)
    _, r, c = best
    return (r, c, tile_edge, int(r * c > 1), c * tile_edge, r * tile_edge)


def plan_int(width: int, height: int, tile_edge: int, max_tiles: int) -> tuple:
    """The exact integer restatement K1 implements: compare log-ratios by
    cross-multiplying max(wr, hc)/min(wr, hc); same tie-break."""
    best = None
    for r in range(1, max_tiles + 1):
        for c in range(1, max_tiles // r + 1):
            a, b = width * r, height * c
            big, small = max(a, b), min(a, b)
            if best is None:
                best = (big, small, r, c)
                continue
            lhs, rhs = big * best[1], best[0] * small
            if lhs < rhs or (lhs == rhs and (r * c, r) < (best[2] * best[3], best[2])):
                best = (big, small, r, c)
    _, _, r, c = best
    return (r, c, tile_edge, int(r * c > 1), c * tile_edge, r * tile_edge)


def n_images(plan: Sequence[int]) -> int:
    return plan[0] * plan[1] + plan[3]


# ---------------------------------------------------------------------------
# resampling

def axis_weights(src: int, out: int):
    """_axis_weights (imgproc.py:298-306): half-pixel positions, clamped."""
    pos = (np.arange(out, dtype=np.float64) + 0.5) * (src / out) - 0.5
    pos = np.minimum(np.maximum(pos, 0.0), float(src - 1))
    i0 = np.minimum(np.floor(pos).astype(np.int64), src - 1)
    frac = pos - i0
    i1 = np.minimum(i0 + 1, src - 1)
    return i0, i1, frac


def _blend(img64: np.ndarray, ry, cx) -> np.ndarray:
    """Vertical then horizontal 2-tap blend in the reference's rounding order
    (imgproc.py:309-331): each product and each sum is a separately rounded
    float64 numpy op (numpy never contracts them into an FMA)."""
    y0, y1, fy = ry
    x0, x1, fx = cx
    wy = fy[:, None, None]
    vert = img64[y0] * (1.0 - wy) + img64[y1] * wy
    wx = fx[None, :, None]
    return vert[:, x0] * (1.0 - wx) + vert[:, x1] * wx


def _round_u8(vals: np.ndarray) -> np.ndarray:
    """_to_uint8 (imgproc.py:338-340): floor(v + 0.5) clipped to [0, 255]."""
    return np.clip(np.floor(vals + 0.5), 0.0, 255.0).astype(np.uint8)


def sample_window(arr: np.ndarray, resized_h: int, resized_w: int, oy0: int, ox0: int,
                  out_h: int, out_w: int) -> np.ndarray:
    """Rows [oy0, oy0+out_h) x cols [ox0, ox0+out_w) of the virtual
    resize of `arr` (H, W, C) to (resized_h, resized_w), as uint8."""
    h, w = arr.shape[:2]
    y0, y1, fy = axis_weights(h, resized_h)
    x0, x1, fx = axis_weights(w, resized_w)
    ys = slice(oy0, oy0 + out_h)
    xs = slice(ox0, ox0 + out_w)
    vals = _blend(arr.astype(np.float64), (y0[ys], y1[ys], fy[ys]), (x0[xs], x1[xs], fx[xs]))
    return _round_u8(vals)


def resize_u8(arr: np.ndarray, out_w: int, out_h: int) -> np.ndarray:
    """_resize_array (imgproc.py:352-358); the identity shortcut is exact anyway."""
    if arr.ndim == 2:
        arr = arr[:, :, None]
    return sample_window(arr, out_h, out_w, 0, 0, out_h, out_w)


def _vert_band(img64: np.ndarray, y0, y1, fy) -> np.ndarray:
    """_blend_vertical (imgproc.py:309-321) with its in-place updates: the same
    separately rounded fp64 ops as _blend, one band of output rows."""
    wy = fy[:, None, None]
    vert = img64[y0]
    vert *= 1.0 - wy
    lower = img64[y1]
    lower *= wy
    vert += lower
    return vert


def _horiz_into(vert: np.ndarray, x0, x1, fx, out: np.ndarray) -> None:
    """_blend_horizontal + _to_uint8_into (imgproc.py:324-349), in place."""
    wx = fx[None, :, None]
    vals = vert[:, x0]
    vals *= 1.0 - wx
    right = vert[:, x1]
    right *= wx
    vals += right
    vals += 0.5
    np.floor(vals, out=vals)
    np.clip(vals, 0.0, 255.0, out=vals)
    out[...] = vals


def tiles_u8(arr: np.ndarray, plan: Sequence[int]) -> np.ndarray:
    """_tile_fused with avoid_per_item_split (imgproc.py:373-404): row-major tiles,
    thumbnail last, as one (n_images, E, E, C) uint8 array.  Like the reference, the
    vertical blend of a grid row is computed once and shared by that row's tiles
    (imgproc.py:388-393), so this port costs what vlmfp's fused path costs."""
    if arr.ndim == 2:
        arr = arr[:, :, None]
    rows, cols, e, thumb, rw, rh = (int(v) for v in plan)
    h, w, c = arr.shape
    out = np.empty((rows * cols + thumb, e, e, c), dtype=np.uint8)
    img64 = arr.astype(np.float64)
    y0, y1, fy = axis_weights(h, rh)
    x0, x1, fx = axis_weights(w, rw)
    k = 0
    for r in range(rows):
        ys = slice(r * e, (r + 1) * e)
        band = _vert_band(img64, y0[ys], y1[ys], fy[ys])
        for cl in range(cols):
            xs = slice(cl * e, (cl + 1) * e)
            _horiz_into(band, x0[xs], x1[xs], fx[xs], out[k])
            k += 1
    if thumb:
        ty0, ty1, tfy = axis_weights(h, e)
        tx0, tx1, tfx = axis_weights(w, e)
        _horiz_into(_vert_band(img64, ty0, ty1, tfy), tx0, tx1, tfx, out[k])
    return out


def resize_scalar(arr: np.ndarray, out_w: int, out_h: int) -> np.ndarray:
    """Pure-Python quadruple loop straight from the definition, for tiny
    cases (restates the reference's own test oracle, tests/test_imgproc.py:30-55)."""
    if arr.ndim == 2:
        arr = arr[:, :, None]
    h, w, c = arr.shape
    out = np.empty((out_h, out_w, c), dtype=np.uint8)
    sy_scale, sx_scale = h / out_h, w / out_w
    for oy in range(out_h):
        sy = min(max((oy + 0.5) * sy_scale - 0.5, 0.0), float(h - 1))
        y0 = min(int(math.floor(sy)), h - 1)
        fy = sy - y0
        y1 = min(y0 + 1, h - 1)
        for ox in range(out_w):
            sx = min(max((ox + 0.5) * sx_scale - 0.5, 0.0), float(w - 1))
            x0 = min(int(math.floor(sx)), w - 1)
            fx = sx - x0
            x1 = min(x0 + 1, w - 1)
            for ch in range(c):
                left = float(arr[y0, x0, ch]) * (1.0 - fy) + float(arr[y1, x0, ch]) * fy
                right = float(arr[y0, x1, ch]) * (1.0 - fy) + float(arr[y1, x1, ch]) * fy
                out[oy, ox, ch] = int(math.floor(left * (1.0 - fx) + right * fx + 0.5))
    return out


# ---------------------------------------------------------------------------
# normalization

def normalize(u8: np.ndarray, mean, std, bf16: bool) -> np.ndarray:
    """_normalize_array (imgproc.py:471-478): (x_f32 / f32(255) - mean) / std in
    IEEE fp32, then optional bf16 RNE.  Channel-last input."""
    c = u8.shape[-1]
    m = np.asarray(tuple(mean)[:c], dtype=np.float32)
    s = np.asarray(tuple(std)[:c], dtype=np.float32)
    out = (u8.astype(np.float32) / np.float32(255.0) - m) / s
    return out.astype(BF16) if bf16 else out


def lut(mean, std, channels: int, bf16: bool) -> np.ndarray:
    """[C, 256] table of normalize() over every uint8 value."""
    vals = np.tile(np.arange(256, dtype=np.uint8)[:, None], (1, channels))
    return np.ascontiguousarray(normalize(vals, mean, std, bf16).T)


# ---------------------------------------------------------------------------
# token expansion

def expand(ids: Sequence[int], counts: Sequence[int], tpt: int, marker: int, ctx: int,
           asst: int):
    """expand_image_placeholders + _first_assistant (tokenizer.py:294-322).
    Returns (ids, spans, first_assistant_index); raises ValueError on the
    reference's ExpansionError / MalformedSequenceError conditions."""
    ids = list(ids)
    if sum(1 for t in ids if t == marker) != len(counts):
        raise ValueError("marker/count mismatch")
    out: list[int] = []
    spans: list[tuple[int, int]] = []
    k = 0
    for tok in ids:
        if tok == marker:
            n = counts[k] * tpt
            spans.append((len(out), n))
            out.extend([ctx] * n)
            k += 1
        else:
            out.append(tok)
    if asst not in out:
        raise ValueError("no assistant header")
    return out, spans, out.index(asst)


def supervision_mask(ids: Sequence[int], t: int, asst: int) -> np.ndarray:
    """build_supervision_mask law (tokenizer.py:410-418)."""
    a = np.asarray(ids, dtype=np.int64)
    return (np.arange(len(a)) >= t) & (a != asst)


# ---------------------------------------------------------------------------
# token reduction

def pixel_unshuffle(grid: np.ndarray, r: int) -> np.ndarray:
    """pixel_unshuffle (tokenred.py:80-103) on an (h, w, d) array: output cell (i, j)
    concatenates input cells (i*r + a, j*r + b), a outer, b inner."""
    h, w, d = grid.shape
    out = np.empty((h // r, w // r, d * r * r), dtype=grid.dtype)
    for a in range(r):
        for b in range(r):
            k = a * r + b
            out[:, :, k * d:(k + 1) * d] = grid[a::r, b::r, :]
    return out


# ---------------------------------------------------------------------------
# synthetic inputs: CPU twin of tp_synth (misc.cu)

_M32 = np.uint64(0xFFFFFFFF)


def _fmix32(h: np.ndarray) -> np.ndarray:
    h = h.astype(np.uint64) & _M32
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x85EBCA6B)) & _M32
    h ^= h >> np.uint64(13)
    h = (h * np.uint64(0xC2B2AE35)) & _M32
    h ^= h >> np.uint64(16)
    return h


def synth_image(seed: int, k: int, width: int, height: int, channels: int = 3,
                kind: int = 0) -> np.ndarray:
    """Image k of a tp_synth batch, as (H, W, C) uint8."""
    nbytes = width * height * channels
    q = np.arange(nbytes, dtype=np.uint64)
    if kind == 0:
        lo, hi = np.uint64(seed & 0xFFFFFFFF), np.uint64((seed >> 32) & 0xFFFFFFFF)
        inner = (hi + np.uint64(k) * np.uint64(0x9E3779B9) + np.uint64(0x7F4A7C15)) & _M32
        key = _fmix32(lo ^ _fmix32(np.array(inner)))
        q4 = q >> np.uint64(2)
        word = _fmix32(key ^ ((q4 * np.uint64(0x9E3779B1) + np.uint64(0x632BE5AB)) & _M32))
        vals = (word >> (np.uint64(8) * (q & np.uint64(3)))) & np.uint64(0xFF)
    else:
        qi = q.astype(np.int64)
        row = width * channels
        y = qi // row
        rem = qi - y * row
        x = rem // channels
        c = rem - x * channels
        t = (3 * x + 2 * y + 40 * c + 17 * k) % 510
        vals = np.where(t < 256, t, 509 - t)
    return vals.astype(np.uint8).reshape(height, width, channels)


# ---------------------------------------------------------------------------
# the full per-image CPU path (cpu_baseline / --impl reference)

def preprocess_image(arr: np.ndarray, tile_edge: int, max_tiles: int, mean, std,
                     bf16: bool) -> tuple:
    """plan -> fused tiles -> normalize, the reference's fastest recipe path
    (imgproc.py:556-590 with fused_transform / avoid_per_item_split)."""
    h, w = arr.shape[:2]
    plan = plan_float(w, h, tile_edge, max_tiles)
    tiles = tiles_u8(arr, plan)
    return plan, normalize(tiles, mean, std, bf16)


# ---------------------------------------------------------------------------
# greedy tokenizer (tokenizer.py:72-158)

def parse_vocab(text: str):
    """(id_to_token, byte_ids[256], match_table {bytes: id}, max_token_bytes) of a vocab
    file's contents: JSON header line, then one token per line, id = line index
    (tokenizer.py:72-129; validation lives in the product's load_vocab)."""
    import re

    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    toks = lines[1:]
    byte_ids = [-1] * 256
    table = {}
    max_len = 1
    for i, tok in enumerate(toks):
        m = re.match(r"^<0x([0-9A-F]{2})>$", tok)
        if m:
            byte_ids[int(m.group(1), 16)] = i
        else:
            b = tok.encode("utf-8")
            table[b] = i
            max_len = max(max_len, len(b))
    return toks, byte_ids, table, max_len


def tokenize(text: str, byte_ids, table, max_len: int) -> list:
    """Greedy longest match, byte fallback (tokenizer.py:135-158)."""
    data = text.encode("utf-8")
    out, pos, n = [], 0, len(data)
    while pos < n:
        for stop in range(min(pos + max_len, n), pos, -1):
            tid = table.get(data[pos:stop])
            if tid is not None:
                out.append(tid)
                pos = stop
                break
        else:
            bid = byte_ids[data[pos]]
            if bid < 0:
                raise ValueError(f"no token or byte fallback for byte 0x{data[pos]:02X}")
            out.append(bid)
            pos += 1
    return out
