"""Batch fast path: packed uint8 images in HBM -> plans + vision-encoder input.

This is the serving-side API the drop-in functions are built on.  One call
runs, on one CUDA stream and without any host round trip:

    K1 tp_plan    -> plan [n,6], n_images [n], tile_off [n+1]
    K2 tp_tile    -> pixel_values [tiles, C, E, E] (bf16/fp32 NCHW) and/or
                     uint8 tiles [tiles, E, E, C]

so the whole step is CUDA-graph capturable.  Output buffers are sized by an
upper bound (n * (max_tiles + 1) tiles) unless the caller passes a capacity;
``TileBatch.num_tiles()`` reads the exact count back when the host needs it.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .dtypes import FLOAT16_WIDE, FLOAT32
from .runtime import dtype_code, normalize_tables, require_device, stream_handle, torch_dtype

IMAGE_ALIGN = 256


@dataclass
class PackedImages:
    """HWC uint8 images packed into one buffer (host-pinned or device).

    ``wh_host`` keeps the sizes on the host: whoever packed the images knows
    them, and buffer sizing needs them without a device round trip."""

    data: torch.Tensor  # uint8 [bytes]
    offsets: torch.Tensor  # int64 [n]
    wh: torch.Tensor  # int32 [n, 2] (width, height)
    channels: int
    wh_host: np.ndarray  # int32 [n, 2]
    offsets_host: np.ndarray  # int64 [n]
    # touched-row input (transfer.stage_images(touched=...)): each image block holds only
    # the source rows K2 reads; row_map / row_map_off as tp_tile_rows takes them
    row_map: Optional[torch.Tensor] = None  # int32
    row_map_off: Optional[torch.Tensor] = None  # int64 [n]
    touched_for: Optional[tuple] = None  # (tile_edge, max_tiles) the rows were chosen for

    @property
    def n(self) -> int:
        return int(self.wh_host.shape[0])

    @property
    def device(self) -> torch.device:
        return self.data.device

    def nbytes(self) -> int:
        return int(self.data.numel())

    def to(self, device, non_blocking: bool = True) -> "PackedImages":
        device = torch.device(device)
        return PackedImages(
            data=self.data.to(device, non_blocking=non_blocking),
            offsets=self.offsets.to(device, non_blocking=non_blocking),
            wh=self.wh.to(device, non_blocking=non_blocking),
            channels=self.channels,
            wh_host=self.wh_host,
            offsets_host=self.offsets_host,
            row_map=None if self.row_map is None else self.row_map.to(
                device, non_blocking=non_blocking),
            row_map_off=None if self.row_map_off is None else self.row_map_off.to(
                device, non_blocking=non_blocking),
            touched_for=self.touched_for,
        )

    def copy_from_(self, other: "PackedImages", non_blocking: bool = True) -> "PackedImages":
        """In-place refill (same layout) — the per-step H2D of a serving loop.  A
        touched-row batch (row maps) refills only a touched-row batch of the same tiling
        and map size, a whole-image batch only a whole-image one: K2 would otherwise read
        one layout as the other."""
        if (self.row_map is None) != (other.row_map is None):
            raise ValueError("copy_from_: one batch is touched-row staged and the other is not")
        if self.row_map is not None:
            if self.touched_for != other.touched_for:
                raise ValueError(f"copy_from_: batches staged for tilings {self.touched_for} "
                                 f"and {other.touched_for}")
            if (self.row_map.numel() != other.row_map.numel()
                    or self.row_map_off.numel() != other.row_map_off.numel()):
                raise ValueError("copy_from_: row maps differ in size")
        self.data.copy_(other.data, non_blocking=non_blocking)
        self.offsets.copy_(other.offsets, non_blocking=non_blocking)
        self.wh.copy_(other.wh, non_blocking=non_blocking)
        if self.row_map is not None:
            self.row_map.copy_(other.row_map, non_blocking=non_blocking)
            self.row_map_off.copy_(other.row_map_off, non_blocking=non_blocking)
        self.wh_host = other.wh_host
        self.offsets_host = other.offsets_host
        return self


def layout_offsets(wh: np.ndarray, channels: int, align: int = IMAGE_ALIGN):
    wh = np.asarray(wh, dtype=np.int64).reshape(-1, 2)
    sizes = wh[:, 0] * wh[:, 1] * channels
    padded = (sizes + align - 1) // align * align
    offsets = np.zeros(len(sizes), dtype=np.int64)
    if len(sizes) > 1:
        offsets[1:] = np.cumsum(padded)[:-1]
    total = int(padded.sum()) if len(sizes) else 0
    return offsets, max(total, align)


def empty_packed(wh, channels: int, device, pin: bool = False) -> PackedImages:
    wh = np.ascontiguousarray(np.asarray(wh, dtype=np.int32).reshape(-1, 2))
    offsets, total = layout_offsets(wh, channels)
    device = torch.device(device)
    if device.type == "cpu":
        data = torch.empty(total, dtype=torch.uint8, pin_memory=pin)
        off_t = torch.from_numpy(offsets.copy())
        wh_t = torch.from_numpy(wh.copy())
        if pin:
            off_t, wh_t = off_t.pin_memory(), wh_t.pin_memory()
    else:
        data = torch.empty(total, dtype=torch.uint8, device=device)
        off_t = torch.from_numpy(offsets).to(device)
        wh_t = torch.from_numpy(wh).to(device)
    return PackedImages(data, off_t, wh_t, channels, wh, offsets)


def pack_images(arrays: Sequence[np.ndarray], pin: bool = True) -> PackedImages:
    """Pack HWC uint8 numpy images into one (pinned) host buffer."""
    if not arrays:
        raise ValueError("no images")
    arrs = [a[:, :, None] if a.ndim == 2 else a for a in arrays]
    channels = arrs[0].shape[2]
    for a in arrs:
        if a.dtype != np.uint8 or a.ndim != 3 or a.shape[2] != channels:
            raise ValueError("images must be HWC uint8 with a common channel count")
    wh = np.array([[a.shape[1], a.shape[0]] for a in arrs], dtype=np.int32)
    packed = empty_packed(wh, channels, "cpu", pin=pin)
    buf = packed.data.numpy()
    for a, off in zip(arrs, packed.offsets_host):
        flat = np.ascontiguousarray(a).reshape(-1)
        buf[off: off + flat.size] = flat
    return packed


def synth_packed(wh, channels: int, device, seed: int, kind: int = 0) -> PackedImages:
    """Synthetic images generated on device by tp_synth (bench/test inputs)."""
    device = require_device(device)
    packed = empty_packed(wh, channels, device)
    max_bytes = int((packed.wh_host[:, 0].astype(np.int64) * packed.wh_host[:, 1]).max()) * channels
    with torch.cuda.device(device):
        _lib.call("tp_synth", _lib.ptr(packed.data), _lib.ptr(packed.offsets),
                  _lib.ptr(packed.wh), packed.n, channels, seed & (2**64 - 1), kind, max_bytes,
                  stream_handle(device))
    return packed


@dataclass
class PlanBatch:
    plan: torch.Tensor  # int32 [n, 6] TilePlan records
    n_images: torch.Tensor  # int32 [n]
    tile_off: torch.Tensor  # int32 [n+1]

    def host(self):
        """(plan [n,6], tile_off [n+1]) as numpy; synchronises the stream."""
        return self.plan.cpu().numpy(), self.tile_off.cpu().numpy()


@dataclass
class TileBatch:
    plans: PlanBatch
    pixel_values: Optional[torch.Tensor]  # [cap, C, E, E] or [cap, E, E, C]
    pixel_u8: Optional[torch.Tensor]  # [cap, E, E, C] uint8

    def num_tiles(self) -> int:
        t = int(self.plans.tile_off[-1].item())
        if t < 0:
            raise ValueError("invalid image size in batch (width/height outside [1, 65536])")
        return t


class TilePreprocessor:
    """Batched, device-resident equivalent of tile_image + normalize_tiles.

    cfg            PreprocessConfig (tile_edge, max_tiles, mean, std, precision)
    layout         "NCHW" (vision-encoder input) or "NHWC" (reference layout)
    emit_uint8     also write the uint8 HWC tiles (deferred-normalize payload)
    normalize      write normalized tiles (False = uint8 tiles only)
    fuse_small     batches of <= TP_PLAN_TILE_MAX_IMAGES images run K1 inside K2
                   (tp_plan_tile: one launch, same plans and tiles; batch-1 latency)
    """

    def __init__(self, cfg, device=None, layout: str = "NCHW", emit_uint8: bool = False,
                 normalize: bool = True, algo: str = "auto", fuse_small: bool = True):
        self.cfg = cfg
        self.fuse_small = fuse_small
        algos = {"auto": _lib.TP_TILE_ALGO_AUTO, "fast": _lib.TP_TILE_ALGO_FAST,
                 "exact": _lib.TP_TILE_ALGO_EXACT}
        if algo not in algos:
            raise ValueError(f"algo must be one of {sorted(algos)}, got {algo!r}")
        self.algo = algos[algo]
        self.device = require_device(device)
        if layout not in ("NCHW", "NHWC"):
            raise ValueError(f"layout must be NCHW or NHWC, got {layout!r}")
        if not normalize and not emit_uint8:
            raise ValueError("nothing to emit")
        self.layout = _lib.TP_LAYOUT_NCHW if layout == "NCHW" else _lib.TP_LAYOUT_NHWC
        self.emit_uint8 = emit_uint8
        self.normalize = normalize
        self.dtype = dtype_code(cfg.effective_precision) if normalize else _lib.TP_DTYPE_NONE
        self._luts: dict[int, tuple] = {}

    @property
    def tile_edge(self) -> int:
        return self.cfg.tile_edge

    def capacity_for(self, n: int) -> int:
        return n * (self.cfg.max_tiles + 1)

    def lut(self, channels: int) -> Optional[torch.Tensor]:
        return self._norm(channels)[0]

    def _norm(self, channels: int):
        """(table, affine_ok) from K0; affine_ok lets K2 normalize by fma (same bits)."""
        if self.dtype == _lib.TP_DTYPE_NONE:
            return None, False
        if channels not in self._luts:
            self._luts[channels] = normalize_tables(self.cfg.mean, self.cfg.std, channels,
                                                    self.dtype, self.device)
        return self._luts[channels]

    def alloc_plans(self, n: int) -> PlanBatch:
        d = self.device
        return PlanBatch(
            plan=torch.empty((n, _lib.TP_PLAN_FIELDS), dtype=torch.int32, device=d),
            n_images=torch.empty((n,), dtype=torch.int32, device=d),
            tile_off=torch.empty((n + 1,), dtype=torch.int32, device=d),
        )

    def alloc_outputs(self, channels: int, capacity: int):
        E = self.cfg.tile_edge
        d = self.device
        pv = None
        if self.dtype != _lib.TP_DTYPE_NONE:
            shape = (capacity, channels, E, E) if self.layout == _lib.TP_LAYOUT_NCHW else (
                capacity, E, E, channels)
            pv = torch.empty(shape, dtype=torch_dtype(self.dtype), device=d)
        u8 = torch.empty((capacity, E, E, channels), dtype=torch.uint8, device=d) \
            if self.emit_uint8 else None
        return pv, u8

    def plan(self, images: PackedImages, out: Optional[PlanBatch] = None,
             stream: Optional[torch.cuda.Stream] = None, after_kernel: bool = False) -> PlanBatch:
        """K1.  ``after_kernel``: the last operation enqueued on ``stream`` is a kernel
        (e.g. the previous batch's tile()), so K1 may start under its tail."""
        out = out or self.alloc_plans(images.n)
        with torch.cuda.device(self.device):
            _lib.call("tp_plan_ex", _lib.ptr(images.wh), images.n, self.cfg.tile_edge,
                      self.cfg.max_tiles, _lib.ptr(out.plan), _lib.ptr(out.n_images),
                      _lib.ptr(out.tile_off),
                      _lib.TP_PLAN_AFTER_KERNEL if after_kernel else 0,
                      stream_handle(self.device, stream))
        return out

    def tile(self, images: PackedImages, plans: PlanBatch, pixel_values=None, pixel_u8=None,
             stream: Optional[torch.cuda.Stream] = None, after_plan: bool = False) -> None:
        """K2 over a planned batch into caller-provided buffers.  ``after_plan``: the
        last operation enqueued on ``stream`` is the plan() of this batch, so K2 may be
        launched as K1's programmatic dependent."""
        lut, affine = self._norm(images.channels)
        algo = self.algo | (_lib.TP_TILE_NORM_AFFINE if affine else 0) | (
            _lib.TP_TILE_AFTER_PLAN if after_plan else 0)
        caps = [t.shape[0] for t in (pixel_values, pixel_u8) if t is not None]
        if not caps:
            raise ValueError("no output buffer")
        args = (_lib.ptr(images.data), _lib.ptr(images.offsets), _lib.ptr(images.wh), images.n,
                images.channels, _lib.ptr(plans.plan), _lib.ptr(plans.tile_off),
                self.cfg.tile_edge, _lib.ptr(lut), self.dtype, self.layout,
                _lib.ptr(pixel_values), _lib.ptr(pixel_u8), min(caps), algo)
        with torch.cuda.device(self.device):
            if images.row_map is not None:  # touched rows only (transfer.stage_images)
                if images.touched_for != (self.cfg.tile_edge, self.cfg.max_tiles):
                    raise ValueError(f"images were staged with the rows of tiling "
                                     f"{images.touched_for}, preprocessor tiles with "
                                     f"{(self.cfg.tile_edge, self.cfg.max_tiles)}")
                _lib.call("tp_tile_rows", *args, _lib.ptr(images.row_map),
                          _lib.ptr(images.row_map_off), stream_handle(self.device, stream))
            else:
                _lib.call("tp_tile_ex", *args, stream_handle(self.device, stream))

    def __call__(self, images: PackedImages, capacity: Optional[int] = None,
                 out: Optional[TileBatch] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> TileBatch:
        if images.device != self.device:
            raise ValueError(f"images are on {images.device}, preprocessor on {self.device}")
        if out is None:
            cap = capacity if capacity is not None else self.capacity_for(images.n)
            pv, u8 = self.alloc_outputs(images.channels, cap)
            out = TileBatch(self.alloc_plans(images.n), pv, u8)
        self._norm(images.channels)  # K0 (first use only) before K1, so K2 follows K1 directly
        if (self.fuse_small and 0 < images.n <= _lib.TP_PLAN_TILE_MAX_IMAGES
                and self.algo != _lib.TP_TILE_ALGO_EXACT and images.row_map is None):
            self.plan_tile(images, out, stream)
            return out
        self.plan(images, out.plans, stream)
        self.tile(images, out.plans, out.pixel_values, out.pixel_u8, stream, after_plan=True)
        return out

    def plan_tile(self, images: PackedImages, out: TileBatch,
                  stream: Optional[torch.cuda.Stream] = None) -> None:
        """K1 + K2 as one launch (tp_plan_tile) for a batch of at most
        TP_PLAN_TILE_MAX_IMAGES images: the same plans, counts, offsets and tiles."""
        if images.row_map is not None:
            # a touched-row block is not a W*H*C image: tp_plan_tile would read it as one
            # (wrong tiles, and past the slab for the last image); plan() + tile() route
            # through tp_tile_rows
            raise ValueError("plan_tile takes whole-image batches; touched-row batches "
                             "(stage_images(touched=...)) go through plan() + tile()")
        lut, affine = self._norm(images.channels)
        algo = self.algo | (_lib.TP_TILE_NORM_AFFINE if affine else 0)
        caps = [t.shape[0] for t in (out.pixel_values, out.pixel_u8) if t is not None]
        if not caps:
            raise ValueError("no output buffer")
        p = out.plans
        with torch.cuda.device(self.device):
            _lib.call("tp_plan_tile", _lib.ptr(images.data), _lib.ptr(images.offsets),
                      _lib.ptr(images.wh), images.n, images.channels, self.cfg.tile_edge,
                      self.cfg.max_tiles, _lib.ptr(p.plan), _lib.ptr(p.n_images),
                      _lib.ptr(p.tile_off), _lib.ptr(lut), self.dtype, self.layout,
                      _lib.ptr(out.pixel_values), _lib.ptr(out.pixel_u8), min(caps), algo,
                      stream_handle(self.device, stream))


__all__ = [
    "PackedImages",
    "PlanBatch",
    "TileBatch",
    "TilePreprocessor",
    "empty_packed",
    "layout_offsets",
    "pack_images",
    "synth_packed",
    "FLOAT16_WIDE",
    "FLOAT32",
]
