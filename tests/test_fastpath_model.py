"""CPU model of K2's fp32 fast path (csrc/tile_tma.cu, DESIGN.md §K2 error bound).

Emulates the packed-fp32 arithmetic in numpy (fp32 rounding after every operation;
fma as an fp64 product-sum rounded once to fp32, exact for these magnitudes) and checks
the two facts bit-exactness rests on, against the oracle's fp64 reference values:
  * |T' - v| <= 6.9e-5 for every value;
  * whenever the window test does not flag a value, round(T') is the reference byte;
  * the affine path's form of the test (|T' - round(T')| >= 1/2 - 3/16384, TP_K2_DWIN)
    flags nearly the same values (the window edges differ by < 1/16384) and is
    sufficient on its own.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import tileprep_oracle as O

F32 = np.float32


def _fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(F32)


def _fast_path(arr: np.ndarray, out_h: int, out_w: int):
    """(T', flagged, reference uint8) for a full-frame resize of arr."""
    h, w = arr.shape[:2]
    y0, y1, fy = O.axis_weights(h, out_h)
    x0, x1, fx = O.axis_weights(w, out_w)
    a = arr[y0][:, x0].astype(F32)
    b = arr[y1][:, x0].astype(F32)
    c = arr[y0][:, x1].astype(F32)
    d = arr[y1][:, x1].astype(F32)
    fy32 = fy.astype(F32)[:, None, None]
    fx32 = fx.astype(F32)[None, :, None]
    L = _fma32(fy32, (b - a).astype(F32), a)  # a + fy (b - a); the differences are exact
    R = _fma32(fy32, (d - c).astype(F32), c)
    D = (R - L).astype(F32)
    T = _fma32(fx32, D, L)
    N = _fma32(T, F32(8192), F32(12587008)).astype(np.int64)  # 1.5*2^23 + 4096 + round(8192 t)
    flagged = ((N + 1) & 8191) <= 2
    ref = O.resize_u8(arr, out_w, out_h)
    # the exact real value with the fp64 weights (the fp64 reference is within 2e-13)
    wy = fy[:, None, None]
    wx = fx[None, :, None]
    a64, b64, c64, d64 = (v.astype(np.float64) for v in (a, b, c, d))
    v = (1 - wx) * (a64 + wy * (b64 - a64)) + wx * (c64 + wy * (d64 - c64))
    return T, flagged, ref, v


@pytest.mark.parametrize("h,w,oh,ow,kind", [
    (1080, 1920, 448, 896, "random"),   # C2 tiles (rational 135/56 x 15/7 weights)
    (1080, 1920, 448, 448, "random"),   # C2 thumbnail
    (480, 640, 1344, 1792, "smooth"),   # 2.8x upscale
    (517, 333, 896, 448, "random"),
    (128, 128, 64, 64, "random"),       # exact 2x: every weight is 1/2, many exact ties
])
def test_fast_path_error_bound_and_window(h, w, oh, ow, kind):
    rng = np.random.default_rng(h * 7 + w)
    if kind == "random":
        arr = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    else:
        yy, xx = np.mgrid[0:h, 0:w]
        arr = np.stack([(xx * 255 // max(w - 1, 1)), (yy * 255 // max(h - 1, 1)),
                        ((xx + yy) % 256)], axis=2).astype(np.uint8)
    T, flagged, ref, v = _fast_path(arr, oh, ow)
    assert float(np.abs(T.astype(np.float64) - v).max()) <= 6.9e-5
    fast_byte = np.floor(T.astype(np.float64) + 0.5).clip(0, 255).astype(np.uint8)
    ok = ~flagged
    assert np.array_equal(fast_byte[ok], ref[ok])
    # affine path (TP_K2_DWIN): d = T - rint(T) exact in fp32, flagged when |d| >= 8189/16384
    kf = (T + F32(12582912.0)).astype(F32) - F32(12582912.0)
    d = (T - kf).astype(F32)
    flagged_d = np.abs(d) >= F32(8189.0 / 16384.0)
    ok_d = ~flagged_d
    assert np.array_equal(kf[ok_d].astype(np.int64), ref[ok_d].astype(np.int64))
    # the same window up to its edges: N = round(8192 t) moves the edge by < 1/16384
    assert int(flagged_d.sum()) <= 1.1 * int(flagged.sum()) + 8
    # on random content the flagged share stays small except on exact-tie grids
    # (smooth content with rational weights hits exact k + 1/2 more often: 2.4% here)
    if kind == "random" and (h, w) != (128, 128):
        assert flagged.mean() < 0.01
