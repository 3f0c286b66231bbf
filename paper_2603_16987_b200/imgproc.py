"""Drop-in image preprocessing API backed by the sm_100a kernels.

Same types, signatures, validation and error behaviour as vlmfp.imgproc
(imgproc.py:29-598); the arithmetic runs on the GPU:

  select_tile_plan  -> K1 tp_plan      (warp-level exact planner)
  tile_image        -> K2 tp_tile      (fused fp64-exact resample/crop/thumbnail)
  resize_bilinear   -> K2 tp_resize
  normalize(_tiles) -> K0 tp_build_lut + K4 tp_normalize
  preprocess        -> host decode, then K1 + K2 with normalize fused into K2

Inputs and outputs stay host numpy ``ImageBuffer``s (the reference contract),
so every call pays one H2D and one D2H; the batch engine
(paper_2603_16987_b200.engine) is the device-resident fast path.
Recipe toggles are latency-only in the reference and change no output; here
they only select whether returned tiles share one backing array
(avoid_per_item_split, imgproc.py:400-404) and whether a "mask" stage key is
reported (skip_pixel_mask, the mask is an all-ones no-op, imgproc.py:516-532).
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._decode import decode_rgb
from .dtypes import FLOAT16_WIDE, FLOAT32, UINT8, to_numpy
from .runtime import (dtype_code, normalize_lut, normalize_tables, require_device, stream_handle,
                      torch_dtype)


@dataclass
class ImageBuffer:
    """Contiguous row-major (H, W, C) raster (imgproc.py:29-61)."""

    width: int
    height: int
    channels: int
    elem: str
    data: np.ndarray

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be >= 1")
        if self.channels not in (1, 3):
            raise ValueError(f"channels must be 1 or 3, got {self.channels}")
        want = (self.height, self.width, self.channels)
        if self.data.shape != want:
            raise ValueError(f"data shape {self.data.shape} != {want}")
        if self.data.dtype != to_numpy(self.elem):
            raise ValueError(f"dtype {self.data.dtype} does not match elem {self.elem!r}")
        if not self.data.flags.c_contiguous:
            raise ValueError("data must be C-contiguous")

    @classmethod
    def from_array(cls, arr: np.ndarray, elem: str = UINT8) -> "ImageBuffer":
        if arr.ndim == 2:
            arr = arr[:, :, None]
        h, w, c = arr.shape
        return cls(w, h, c, elem, np.ascontiguousarray(arr, dtype=to_numpy(elem)))


@dataclass(frozen=True)
class TilePlan:
    """Chosen tiling grid for one image (imgproc.py:64-81)."""

    rows: int
    cols: int
    tile_edge: int
    include_thumbnail: bool
    resized_width: int
    resized_height: int

    @property
    def n_tiles(self) -> int:
        return self.rows * self.cols

    @property
    def n_images(self) -> int:
        return self.n_tiles + (1 if self.include_thumbnail else 0)

    def as_record(self) -> np.ndarray:
        return np.array([self.rows, self.cols, self.tile_edge, int(self.include_thumbnail),
                         self.resized_width, self.resized_height], dtype=np.int32)

    @classmethod
    def from_record(cls, rec) -> "TilePlan":
        r = [int(v) for v in rec]
        return cls(rows=r[0], cols=r[1], tile_edge=r[2], include_thumbnail=bool(r[3]),
                   resized_width=r[4], resized_height=r[5])


@dataclass(frozen=True)
class PreprocessConfig:
    """Geometry, normalization constants and recipe toggles (imgproc.py:84-120)."""

    tile_edge: int = 448
    max_tiles: int = 12
    mean: tuple[float, float, float] = (0.5, 0.5, 0.5)
    std: tuple[float, float, float] = (0.5, 0.5, 0.5)
    normalize_precision: str = FLOAT32
    fused_transform: bool = False
    contiguous_tensor_path: bool = False
    decode_once: bool = False
    reduced_precision_normalize: bool = False
    simd_decode: bool = False
    skip_pixel_mask: bool = False
    avoid_per_item_split: bool = False

    def __post_init__(self):
        if self.tile_edge < 1:
            raise ValueError("tile_edge must be positive")
        if self.max_tiles < 1:
            raise ValueError("max_tiles must be >= 1")
        if any(s <= 0 for s in self.std):
            raise ValueError("std components must be strictly positive")
        if self.normalize_precision not in (FLOAT32, FLOAT16_WIDE):
            raise ValueError(f"bad normalize_precision {self.normalize_precision!r}")

    @property
    def effective_precision(self) -> str:
        return FLOAT16_WIDE if self.reduced_precision_normalize else self.normalize_precision


@dataclass
class PreprocessResult:
    tiles: list[ImageBuffer]
    plan: TilePlan
    stage_timings_ns: dict[str, int]
    deferred: bool


# ---------------------------------------------------------------------------
# decode (host; outside the GPU path)

def decode_image(payload: bytes, cfg: PreprocessConfig) -> ImageBuffer:
    """Decode a JPEG or PNG payload to a 3-channel uint8 buffer (imgproc.py:245-260).
    The reference's decode toggles only add redundant work; one decode here."""
    arr = decode_rgb(payload)
    h, w, c = arr.shape
    return ImageBuffer(w, h, c, UINT8, arr)


# ---------------------------------------------------------------------------
# helpers

def _check_plan_args(width: int, height: int, cfg: PreprocessConfig) -> None:
    if width < 1 or height < 1:
        raise ValueError("width and height must be >= 1")
    if width > _lib.TP_MAX_EDGE or height > _lib.TP_MAX_EDGE:
        raise ValueError(f"image edge above {_lib.TP_MAX_EDGE} is outside the exact planner domain")


def _upload(arr: np.ndarray, device: torch.device) -> torch.Tensor:
    host = torch.from_numpy(np.require(arr, requirements=("C", "W")))  # copies read-only views
    return host.to(device, non_blocking=False)


def _split(backing: np.ndarray, e: int, c: int, elem: str, shared: bool) -> list[ImageBuffer]:
    if shared:
        return [ImageBuffer(e, e, c, elem, backing[i]) for i in range(backing.shape[0])]
    return [ImageBuffer(e, e, c, elem, backing[i].copy()) for i in range(backing.shape[0])]


def _to_numpy(t: torch.Tensor, elem: str) -> np.ndarray:
    host = t.cpu()
    if elem == FLOAT16_WIDE:
        return host.view(torch.int16).numpy().view(to_numpy(FLOAT16_WIDE))
    return host.numpy()


class _Run:
    """One single-image device pass: image upload + plan + K2 on one stream."""

    def __init__(self, img: ImageBuffer):
        self.device = require_device()
        self.stream = torch.cuda.current_stream(self.device)
        self.handle = stream_handle(self.device, self.stream)
        self.img = img
        self.src = _upload(img.data.reshape(-1), self.device)
        self.off = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.wh = torch.tensor([[img.width, img.height]], dtype=torch.int32, device=self.device)

    def tile(self, plan_rec: torch.Tensor, tile_off: torch.Tensor, e: int, n_tiles: int,
             lut: Optional[torch.Tensor], dtype: int, layout: int, want_u8: bool,
             affine: bool = False):
        c = self.img.channels
        out = None
        if dtype != _lib.TP_DTYPE_NONE:
            out = torch.empty((n_tiles, e, e, c), dtype=torch_dtype(dtype), device=self.device)
        u8 = torch.empty((n_tiles, e, e, c), dtype=torch.uint8, device=self.device) \
            if want_u8 else None
        algo = _lib.TP_TILE_ALGO_AUTO | (_lib.TP_TILE_NORM_AFFINE if affine else 0)
        _lib.call("tp_tile_ex", _lib.ptr(self.src), _lib.ptr(self.off), _lib.ptr(self.wh), 1, c,
                  _lib.ptr(plan_rec), _lib.ptr(tile_off), e, _lib.ptr(lut), dtype, layout,
                  _lib.ptr(out), _lib.ptr(u8), n_tiles, algo, self.handle)
        return out, u8


# ---------------------------------------------------------------------------
# tile planning (K1)

def select_tile_plan(width: int, height: int, cfg: PreprocessConfig) -> TilePlan:
    """Grid whose aspect ratio is log-closest to the image's; ties go to fewer
    tiles, then fewer rows; thumbnail iff more than one tile (imgproc.py:266-292).
    Computed by the warp-level planner K1 with exact integer comparisons."""
    _check_plan_args(width, height, cfg)
    device = require_device()
    wh = torch.tensor([[width, height]], dtype=torch.int32, device=device)
    plan = torch.empty((1, _lib.TP_PLAN_FIELDS), dtype=torch.int32, device=device)
    n_img = torch.empty((1,), dtype=torch.int32, device=device)
    tile_off = torch.empty((2,), dtype=torch.int32, device=device)
    _lib.call("tp_plan", _lib.ptr(wh), 1, cfg.tile_edge, cfg.max_tiles, _lib.ptr(plan),
              _lib.ptr(n_img), _lib.ptr(tile_off), stream_handle(device))
    return TilePlan.from_record(plan.cpu().numpy()[0])


# ---------------------------------------------------------------------------
# resampling (K2)

def resize_bilinear(img: ImageBuffer, out_w: int, out_h: int) -> ImageBuffer:
    """Half-pixel bilinear resize, bit-exact with imgproc.py:352-367."""
    if img.elem != UINT8:
        raise ValueError("resize_bilinear expects a uint8 buffer")
    if out_w < 1 or out_h < 1:
        raise ValueError("output dimensions must be >= 1")
    device = require_device()
    src = _upload(img.data.reshape(-1), device)
    dst = torch.empty((out_h, out_w, img.channels), dtype=torch.uint8, device=device)
    _lib.call("tp_resize", _lib.ptr(src), img.width, img.height, img.channels, out_w, out_h,
              _lib.ptr(dst), stream_handle(device))
    return ImageBuffer(out_w, out_h, img.channels, UINT8, dst.cpu().numpy())


def _validate_plan(plan: TilePlan) -> None:
    if plan.rows < 1 or plan.cols < 1 or plan.tile_edge < 1:
        raise ValueError("plan needs rows, cols, tile_edge >= 1")
    if plan.resized_width < 1 or plan.resized_height < 1:
        raise ValueError("plan resized size must be >= 1")
    if plan.resized_width < plan.cols * plan.tile_edge or \
            plan.resized_height < plan.rows * plan.tile_edge:
        raise ValueError("plan resized size smaller than its tile grid")


def tile_image(img: ImageBuffer, plan: TilePlan, cfg: PreprocessConfig) -> list[ImageBuffer]:
    """Row-major tiles of the aspect-resized image, thumbnail last (imgproc.py:449-465),
    sampled straight from the source by K2 (byte-identical to resize-then-crop)."""
    if img.elem != UINT8:
        raise ValueError("tile_image expects a uint8 buffer")
    _validate_plan(plan)
    run = _Run(img)
    rec = torch.from_numpy(plan.as_record()[None, :]).to(run.device)
    tile_off = torch.tensor([0, plan.n_images], dtype=torch.int32, device=run.device)
    _, u8 = run.tile(rec, tile_off, plan.tile_edge, plan.n_images, None, _lib.TP_DTYPE_NONE,
                     _lib.TP_LAYOUT_NHWC, True)
    return _split(u8.cpu().numpy(), plan.tile_edge, img.channels, UINT8,
                  cfg.avoid_per_item_split)


# ---------------------------------------------------------------------------
# normalization (K0 + K4)

def _normalize_batch(stack: np.ndarray, channels: int, cfg: PreprocessConfig) -> np.ndarray:
    device = require_device()
    dtype = dtype_code(cfg.effective_precision)
    lut = normalize_lut(cfg.mean, cfg.std, channels, dtype, device)
    src = _upload(stack.reshape(-1), device)
    out = torch.empty(stack.shape, dtype=torch_dtype(dtype), device=device)
    n_img = stack.shape[0] if stack.ndim == 4 else 1
    ppi = stack.size // (channels * n_img) if stack.size else 0
    _lib.call("tp_normalize", _lib.ptr(src), n_img, ppi, channels, _lib.ptr(lut), dtype,
              _lib.TP_LAYOUT_NHWC, _lib.ptr(out), stream_handle(device))
    return _to_numpy(out, cfg.effective_precision)


def normalize(img: ImageBuffer, cfg: PreprocessConfig) -> ImageBuffer:
    """Per-channel (x/255 - mean)/std in float32 or float16-wide (imgproc.py:481-486),
    as the exact 3x256 lookup table built on device by K0."""
    if img.elem != UINT8:
        raise ValueError("normalize expects a uint8 buffer")
    out = _normalize_batch(img.data, img.channels, cfg)
    return ImageBuffer(img.width, img.height, img.channels, cfg.effective_precision, out)


def normalize_tiles(tiles: list[ImageBuffer], cfg: PreprocessConfig) -> list[ImageBuffer]:
    """Normalize a tile batch in one device pass (imgproc.py:496-513); with
    avoid_per_item_split the results are views of one backing array."""
    if not tiles:
        return tiles
    for t in tiles:
        if t.elem != UINT8:
            raise ValueError("normalize expects a uint8 buffer")
    shape0 = tiles[0].data.shape
    if any(t.data.shape != shape0 for t in tiles):
        return [normalize(t, cfg) for t in tiles]
    stack = np.stack([t.data for t in tiles])
    out = _normalize_batch(stack, shape0[2], cfg)
    prec = cfg.effective_precision
    return [ImageBuffer(t.width, t.height, t.channels, prec,
                        out[i] if cfg.avoid_per_item_split else out[i].copy())
            for i, t in enumerate(tiles)]


# ---------------------------------------------------------------------------
# full preprocessing pass

class _Session:
    """Per-thread, per-device state of the drop-in ``preprocess``: the device JPEG decoder,
    one batch preprocessor per tiling / output configuration, and grow-only pinned and
    device buffers, so a request costs no allocation beyond its result arrays."""

    def __init__(self, device: torch.device):
        self.device = device
        self.jpeg = None
        self.png = None
        self.preps: dict = {}
        self.host = None  # pinned staging for host-decoded pixels
        self.dev = None

    def prep(self, cfg: PreprocessConfig, defer: bool):
        from .engine import TilePreprocessor

        key = (cfg.tile_edge, cfg.max_tiles, tuple(cfg.mean), tuple(cfg.std),
               cfg.effective_precision, defer)
        p = self.preps.get(key)
        if p is None:
            p = TilePreprocessor(cfg, self.device, layout="NHWC", emit_uint8=defer,
                                 normalize=not defer)
            self.preps[key] = p
        return p

    def upload(self, arr: np.ndarray, stream):
        """Host pixels -> a 1-image device batch through the pinned slab."""
        from .engine import PackedImages

        nbytes = arr.size
        if self.host is None or self.host.numel() < nbytes:
            cap = (nbytes * 5 // 4 + (1 << 20)) & ~((1 << 20) - 1)
            self.host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self.dev = torch.empty(cap, dtype=torch.uint8, device=self.device)
        stream.synchronize()  # the previous request's upload no longer reads the slab
        self.host[:nbytes].numpy()[:] = arr.reshape(-1)
        with torch.cuda.stream(stream):
            self.dev[:nbytes].copy_(self.host[:nbytes], non_blocking=True)
        wh = np.array([[arr.shape[1], arr.shape[0]]], dtype=np.int32)
        off = np.zeros(1, dtype=np.int64)
        return PackedImages(self.dev, torch.zeros(1, dtype=torch.int64, device=self.device),
                            torch.from_numpy(wh).to(self.device), 3, wh, off)


_tls = threading.local()


def _session(device: torch.device) -> _Session:
    s = getattr(_tls, "session", None)
    if s is None or s.device != device:
        s = _Session(device)
        _tls.session = s
    return s


def preprocess(payload: bytes, cfg: PreprocessConfig, *,
               defer_normalize: bool = False) -> PreprocessResult:
    """decode -> plan -> resize -> tile -> normalize (or defer) -> mask
    (imgproc.py:538-598).  Stage keys are the reference's.  On the device path:
    "decode" is the device decode of baseline JPEGs (K7) and 8-bit L / RGB / P PNGs (K8):
    host marker / chunk parse, upload of the compressed bytes, device decode -- or, for
    the payloads neither takes, the reference's Pillow decode on the host plus the pixel
    upload; "plan"
    is K1's exact rule on the host (the TilePlan the result carries); "resize" is empty
    (fused into K2); "tile" is K1 + K2 in one launch (resample + crop + thumbnail, with
    normalize fused unless deferred); "normalize"/"defer" is the readback into
    ImageBuffers."""
    from .jpeg import TP_JPEG_OK, JpegDecoder, parse
    from . import png as _png

    timings: dict[str, int] = {}
    device = require_device()
    stream = torch.cuda.current_stream(device)
    sess = _session(device)
    t0 = time.perf_counter_ns()
    if payload[:2] == b"\xff\xd8" and parse(payload).status == TP_JPEG_OK:
        if sess.jpeg is None:
            sess.jpeg = JpegDecoder(device)
        images = sess.jpeg.decode([payload], stream=stream)  # host fallback inside
        width, height = (int(v) for v in images.wh_host[0])
    elif payload[:8] == _png.PNG_SIGNATURE and _png.parse(payload)[0].status == _png.TP_PNG_OK:
        if sess.png is None:
            sess.png = _png.PngDecoder(device)
        images = sess.png.decode([payload], stream=stream)  # host fallback inside
        width, height = (int(v) for v in images.wh_host[0])
    else:
        arr = decode_rgb(payload)
        height, width = arr.shape[:2]
        _check_plan_args(width, height, cfg)
        images = sess.upload(arr, stream)
    timings["decode"] = time.perf_counter_ns() - t0

    t0 = time.perf_counter_ns()
    _check_plan_args(width, height, cfg)
    plan_rec = np.zeros(_lib.TP_PLAN_FIELDS, dtype=np.int32)
    _lib.check(_lib.load().tp_plan_host(width, height, cfg.tile_edge, cfg.max_tiles,
                                        plan_rec.ctypes.data), "tp_plan_host")
    plan = TilePlan.from_record(plan_rec)
    timings["plan"] = time.perf_counter_ns() - t0

    timings["resize"] = 0  # fused into K2
    prep = sess.prep(cfg, defer_normalize)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(stream)
    with torch.cuda.stream(stream):
        out = prep(images, capacity=plan.n_images, stream=stream)
    ev[1].record(stream)
    dev_tiles = out.pixel_u8 if defer_normalize else out.pixel_values
    elem = UINT8 if defer_normalize else cfg.effective_precision
    backing = _to_numpy(dev_tiles[: plan.n_images], elem)
    ev[2].record(stream)
    ev[2].synchronize()
    timings["tile"] = int(ev[0].elapsed_time(ev[1]) * 1e6)
    timings["defer" if defer_normalize else "normalize"] = int(ev[1].elapsed_time(ev[2]) * 1e6)
    if not cfg.skip_pixel_mask:
        timings["mask"] = 0  # all-ones validity mask: values unchanged, no work
    tiles = _split(backing, cfg.tile_edge, 3, elem, cfg.avoid_per_item_split)
    return PreprocessResult(tiles, plan, timings, deferred=defer_normalize)


__all__ = [
    "ImageBuffer",
    "PreprocessConfig",
    "PreprocessResult",
    "TilePlan",
    "decode_image",
    "normalize",
    "normalize_tiles",
    "preprocess",
    "resize_bilinear",
    "select_tile_plan",
    "tile_image",
]
