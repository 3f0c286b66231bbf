"""Pinned host arena, packed uint8 staging and one-copy H2D.

Mirrors the reference's host staging API (vlmfp/transfer.py:1-272): ``HostArena``
(bump allocator over one slab, transfer.py:62-110), ``Region``, ``CostModel``,
``BatchEntry`` / ``TransferBatch`` (:131-158), ``payload_bytes`` (:167-180),
``pack`` / ``stage_individually`` (:187-236), ``transfer`` (:239-261) and ``unpack``
(:264-272), with the same layouts, errors and modeled duration.  What the reference
only models, this module does for real:

* the slab is page-locked host memory (``torch.empty(pin_memory=True)``) when CUDA is
  present, so a device copy is a true asynchronous DMA;
* ``transfer(batch, model, dest=<CUDA tensor>, stream=...)`` issues one
  ``cudaMemcpyAsync`` per copy span (one for a packed batch) and returns at once;
* ``stage_images`` packs a whole image batch *and* its K1/K2 metadata (sizes,
  offsets) into one region, so a batch reaches the GPU in exactly one copy;
* ``PipelinedPreprocessor`` double-buffers pinned and device slabs so the copy of
  batch i+1 overlaps K1+K2 of batch i on another stream.

Host staging is plumbing, not arithmetic: the bytes are copied, never transformed.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .dtypes import ITEMSIZE, tag_of, to_numpy
from .errors import ArenaFullError, DataError, DomainError, ShapeError

__all__ = [
    "DEFAULT_ALIGNMENT",
    "ArenaFullError",
    "CostModel",
    "HostArena",
    "Region",
    "BatchEntry",
    "TransferBatch",
    "TransferResult",
    "payload_bytes",
    "pack",
    "stage_individually",
    "transfer",
    "unpack",
    "StagedImages",
    "stage_images",
    "upload_images",
    "PipelinedPreprocessor",
]

DEFAULT_ALIGNMENT = 64
IMAGE_ALIGNMENT = 256  # K2 reads rows from 16-byte multiples; images start 256-aligned


def _round_up(n: int, alignment: int) -> int:
    return ((n + alignment - 1) // alignment) * alignment


@dataclass(frozen=True)
class Region:
    """An aligned window into an arena's slab (transfer.py:52-58)."""

    offset: int
    size: int
    view: np.ndarray


class HostArena:
    """Bump allocator over one slab allocated at construction (transfer.py:62-110).

    ``pin`` (default: when CUDA is available) makes the slab page-locked so device
    copies from it are asynchronous DMA transfers."""

    def __init__(self, capacity: int, alignment: int = DEFAULT_ALIGNMENT,
                 pin: Optional[bool] = None) -> None:
        if capacity <= 0:
            raise DomainError(f"arena capacity must be positive, got {capacity}")
        if alignment <= 0:
            raise DomainError(f"arena alignment must be positive, got {alignment}")
        if pin is None:
            pin = torch.cuda.is_available()
        self._tensor = torch.zeros(capacity, dtype=torch.uint8, pin_memory=bool(pin))
        self._slab = self._tensor.numpy()
        self._capacity = capacity
        self._alignment = alignment
        self._mark = 0
        self._alloc_count = 0
        self.pinned = bool(pin)

    @property
    def capacity(self) -> int:
        return self._capacity

    @property
    def alignment(self) -> int:
        return self._alignment

    @property
    def mark(self) -> int:
        return self._mark

    @property
    def allocation_count(self) -> int:
        return self._alloc_count

    @property
    def remaining(self) -> int:
        return max(0, self._capacity - self._mark)

    @property
    def tensor(self) -> torch.Tensor:
        """The slab as a (pinned) torch uint8 tensor, for device copies."""
        return self._tensor

    def alloc(self, size: int) -> Region:
        if size <= 0:
            raise DomainError(f"allocation size must be positive, got {size}")
        if self._mark + size > self._capacity:
            raise ArenaFullError(requested=size, remaining=self.remaining)
        offset = self._mark
        self._mark = _round_up(offset + size, self._alignment)
        self._alloc_count += 1
        return Region(offset=offset, size=size, view=self._slab[offset: offset + size])

    def reset(self) -> None:
        self._mark = 0


@dataclass(frozen=True)
class CostModel:
    """Copy-engine model: fixed per-copy latency plus a bandwidth term (:113-125)."""

    latency_per_copy: float
    bytes_per_second: float

    def __post_init__(self) -> None:
        if not self.latency_per_copy > 0:
            raise DomainError("latency_per_copy must be positive")
        if not self.bytes_per_second > 0:
            raise DomainError("bytes_per_second must be positive")


@dataclass(frozen=True)
class BatchEntry:
    """One logical buffer inside a staged payload (:128-135)."""

    offset: int
    length: int
    dtype: str
    shape: tuple


@dataclass(frozen=True)
class TransferBatch:
    """Staged buffers plus the copy spans needed to move them (:138-158).

    ``slab`` / ``base`` locate the payload in its arena's torch tensor so device
    copies can come straight from the pinned slab."""

    payload: np.ndarray
    entries: tuple
    copies: tuple
    slab: Optional[torch.Tensor] = field(default=None, repr=False, compare=False)
    base: int = 0

    @property
    def n_copies(self) -> int:
        return len(self.copies)

    @property
    def data_bytes(self) -> int:
        return sum(entry.length for entry in self.entries)

    def payload_tensor(self) -> torch.Tensor:
        """The payload as a torch uint8 tensor (a view of the pinned slab if staged in one)."""
        if self.slab is not None:
            return self.slab[self.base: self.base + len(self.payload)]
        return torch.from_numpy(self.payload)


@dataclass(frozen=True)
class TransferResult:
    duration_s: float
    dest: object  # numpy array, or the CUDA tensor the copies were issued to
    done: Optional[torch.cuda.Event] = None  # recorded after the device copies


def payload_bytes(shape: Sequence[int], dtype: str) -> int:
    """Bytes needed for ``shape`` elements of the tagged dtype (:167-180)."""
    dims = tuple(shape)
    if any(d <= 0 for d in dims):
        raise ShapeError(f"shape dims must be positive, got {dims}")
    try:
        itemsize = ITEMSIZE[dtype]
    except KeyError:
        raise DataError(f"unknown dtype tag {dtype!r}") from None
    total = itemsize
    for d in dims:
        total *= d
    return total


def _empty_batch() -> TransferBatch:
    return TransferBatch(payload=np.empty(0, dtype=np.uint8), entries=(), copies=())


def _stage(buffers: Sequence[np.ndarray], arena: HostArena, *, packed: bool) -> TransferBatch:
    if not buffers:
        return _empty_batch()
    sizes = [int(buf.nbytes) for buf in buffers]
    alignment = arena.alignment
    rel_offsets = []
    mark = 0
    for size in sizes:
        rel_offsets.append(mark)
        mark = _round_up(mark + size, alignment)
    total = mark
    if packed:
        region = arena.alloc(total)
        base = region.offset
    else:
        # sequential allocations land back to back: one contiguous window
        regions = [arena.alloc(size) for size in sizes]
        base = regions[0].offset
    payload = arena._slab[base: base + total]
    entries = []
    for buf, rel, size in zip(buffers, rel_offsets, sizes):
        flat = np.ascontiguousarray(buf).view(np.uint8).reshape(-1)
        payload[rel: rel + size] = flat
        entries.append(BatchEntry(offset=rel, length=size, dtype=tag_of(buf), shape=buf.shape))
    if packed:
        copies = ((0, total),)
    else:
        copies = tuple((rel, size) for rel, size in zip(rel_offsets, sizes))
    return TransferBatch(payload=payload, entries=tuple(entries), copies=copies,
                         slab=arena.tensor, base=base)


def pack(buffers: Sequence[np.ndarray], arena: HostArena) -> TransferBatch:
    """Stage buffers back to back in one arena region: one copy total (:226-228)."""
    return _stage(buffers, arena, packed=True)


def stage_individually(buffers: Sequence[np.ndarray], arena: HostArena) -> TransferBatch:
    """Stage each buffer as its own region: one copy per buffer (:231-233)."""
    return _stage(buffers, arena, packed=False)


def transfer(batch: TransferBatch, cost_model: CostModel, dest=None,
             stream: Optional[torch.cuda.Stream] = None) -> TransferResult:
    """Copy the batch to ``dest`` and return the modeled duration (:239-261).

    ``dest`` None or a numpy array: a host byte copy, as in the reference.  ``dest`` a
    CUDA uint8 tensor: one asynchronous H2D copy per span on ``stream`` (default: the
    current stream) from the pinned slab; ``done`` is an event recorded after them.
    The returned duration is the model's ``latency * n_copies + bytes / bandwidth``."""
    n = len(batch.payload)
    duration = 0.0 if batch.n_copies == 0 else (
        cost_model.latency_per_copy * batch.n_copies + batch.data_bytes / cost_model.bytes_per_second)
    if isinstance(dest, torch.Tensor) and dest.is_cuda:
        if dest.dtype != torch.uint8 or dest.numel() < n:
            raise ShapeError(f"destination holds {dest.numel()} bytes, payload needs {n}")
        src = batch.payload_tensor()
        stream = stream or torch.cuda.current_stream(dest.device)
        with torch.cuda.stream(stream):
            for offset, length in batch.copies:
                dest[offset: offset + length].copy_(src[offset: offset + length],
                                                    non_blocking=True)
            done = torch.cuda.Event()
            done.record(stream)
        return TransferResult(duration_s=duration, dest=dest, done=done)
    if dest is None:
        dest = np.empty(n, dtype=np.uint8)
    elif len(dest) < n:
        raise ShapeError(f"destination holds {len(dest)} bytes, payload needs {n}")
    for offset, length in batch.copies:
        dest[offset: offset + length] = batch.payload[offset: offset + length]
    return TransferResult(duration_s=duration, dest=dest)


def unpack(batch: TransferBatch, source=None) -> List[np.ndarray]:
    """Reconstruct the staged buffers bit-exactly from a payload image (:264-272);
    ``source`` may be the CUDA tensor a batch was transferred to."""
    buf = batch.payload if source is None else source
    if isinstance(buf, torch.Tensor):
        buf = buf[: len(batch.payload)].cpu().numpy()
    out = []
    for entry in batch.entries:
        raw = buf[entry.offset: entry.offset + entry.length].tobytes()
        arr = np.frombuffer(raw, dtype=to_numpy(entry.dtype)).reshape(entry.shape)
        out.append(arr.copy())
    return out


# ---------------------------------------------------------------------------
# image batches: pixels and K1/K2 metadata in one region, one copy

@dataclass(frozen=True)
class StagedImages:
    """An image batch staged for one H2D copy.  Payload layout (byte offsets):
    [wh int32 n x 2][offsets int64 n][pad][image 0][pad][image 1]... with every image
    at a multiple of IMAGE_ALIGNMENT; ``offsets`` are payload-relative, so the device
    copy of the payload is directly K2's packed source buffer."""

    batch: TransferBatch
    n: int
    channels: int
    wh: np.ndarray  # int32 [n, 2]
    offsets: np.ndarray  # int64 [n], payload-relative
    wh_at: int
    offsets_at: int
    # touched-row staging: [row-map offsets int64 n][row maps int32] after the offsets
    row_map_at: Optional[int] = None
    row_map_len: int = 0
    row_map_off_at: Optional[int] = None
    touched_for: Optional[tuple] = None  # (tile_edge, max_tiles)


def _image_layout(wh: np.ndarray, channels: int):
    n = len(wh)
    wh_at = 0
    offsets_at = _round_up(8 * n, 8)
    mark = _round_up(offsets_at + 8 * n, IMAGE_ALIGNMENT)
    offs = np.empty(n, dtype=np.int64)
    for k in range(n):
        offs[k] = mark
        mark = _round_up(mark + int(wh[k, 0]) * int(wh[k, 1]) * channels, IMAGE_ALIGNMENT)
    return wh_at, offsets_at, offs, max(mark, IMAGE_ALIGNMENT)


def touched_row_maps(wh: np.ndarray, tile_edge: int, max_tiles: int):
    """Per image, the source rows and columns K2's stencil reads under its plan
    (tp_plan_host + tp_touched_rows / tp_touched_cols, host C code with the device's
    arithmetic): a list of int32 maps [n_rows, idx(y) for each y, n_cols, idx(x) for
    each x] (idx -1 = not read), the layout tp_tile_rows reads."""
    lib = _lib.load()
    maps = []
    plan = np.zeros(_lib.TP_PLAN_FIELDS, dtype=np.int32)
    for w, h in np.asarray(wh, dtype=np.int64).reshape(-1, 2):
        _lib.check(lib.tp_plan_host(int(w), int(h), tile_edge, max_tiles, plan.ctypes.data),
                   "tp_plan_host")
        m = np.empty(int(h) + int(w) + 2, dtype=np.int32)
        rows = m[: int(h) + 1]
        cols = m[int(h) + 1:]
        for fn, part in (("tp_touched_rows", rows), ("tp_touched_cols", cols)):
            n = getattr(lib, fn)(int(w), int(h), plan.ctypes.data, part.ctypes.data)
            if n < 0:
                _lib.check(int(n), fn)
        maps.append(m)
    return maps


def _touched_dims(m: np.ndarray, h: int) -> tuple:
    """(n_rows, n_cols) of a touched map."""
    return int(m[0]), int(m[h + 1])


_map_cache: dict = {}


def staging_map(w: int, h: int, tile_edge: int, max_tiles: int) -> np.ndarray:
    """The map stage_images(touched=...) stages image (w, h) through: the touched-row
    map of touched_row_maps, then an identity column map (n_cols = w: columns are
    staged whole, a column gather saves 3% of a 1080p image for a 3-byte-run copy).
    Depends only on (w, h, tile_edge, max_tiles), so it is cached (read-only)."""
    key = (int(w), int(h), int(tile_edge), int(max_tiles))
    m = _map_cache.get(key)
    if m is None:
        rows = touched_row_maps(np.array([[w, h]], dtype=np.int32), tile_edge, max_tiles)[0]
        m = np.empty(int(h) + int(w) + 2, dtype=np.int32)
        m[: int(h) + 1] = rows[: int(h) + 1]
        m[int(h) + 1] = int(w)
        m[int(h) + 2:] = np.arange(int(w), dtype=np.int32)
        m.setflags(write=False)
        if len(_map_cache) > 4096:
            _map_cache.clear()
        _map_cache[key] = m
    return m


def _hwc(images: Sequence[np.ndarray]):
    """(arrays as HWC views, channels, wh int32 [n, 2]) with validation."""
    if not images:
        raise DataError("no images to stage")
    arrs = [a[:, :, None] if a.ndim == 2 else a for a in images]
    channels = arrs[0].shape[2]
    for a in arrs:
        if a.dtype != np.uint8 or a.ndim != 3 or a.shape[2] != channels:
            raise DataError("images must be HWC uint8 with a common channel count")
    wh = np.array([[a.shape[1], a.shape[0]] for a in arrs], dtype=np.int32)
    return arrs, channels, wh


def _native_pack(arrs, wh, channels, view: np.ndarray, offs: np.ndarray, maps_all=None,
                 map_off=None, threads: int = 0) -> None:
    """Copy every image's pixels (all rows, or only the mapped rows) into ``view`` at
    ``offs`` with tp_stage_pack (multithreaded host C++; the GIL is released)."""
    n = len(arrs)
    keep = []
    ptrs = np.empty(n, dtype=np.uint64)
    strides = np.empty(n, dtype=np.int64)
    for k, a in enumerate(arrs):
        if a.strides[2] != 1 or a.strides[1] != channels or a.strides[0] < a.shape[1] * channels:
            a = np.ascontiguousarray(a)
            keep.append(a)
        ptrs[k] = a.ctypes.data
        strides[k] = a.strides[0]
    base = view.ctypes.data
    _lib.call("tp_stage_pack", n, ptrs.ctypes.data, strides.ctypes.data, wh.ctypes.data,
              channels, None if maps_all is None else maps_all.ctypes.data,
              None if map_off is None else map_off.ctypes.data, base, offs.ctypes.data,
              int(threads))
    del keep


def stage_images(images: Sequence[np.ndarray], arena: HostArena,
                 touched: Optional[tuple] = None, threads: int = 0) -> StagedImages:
    """Pack HWC uint8 images and their sizes/offsets into one arena region.

    The pixels are copied by tp_stage_pack on the library's host thread pool
    (``threads`` <= 0: all of it).  ``touched=(tile_edge, max_tiles)`` stages only the
    source rows K2 will read for that tiling (every tile and thumbnail output's two row
    taps; 83% of a 1080p image at E=448, 41% of a 4K one) plus the maps K2 reads them
    through (tp_tile_rows): fewer bytes on the H2D link, the same tiles."""
    arrs, channels, wh = _hwc(images)
    if touched is not None:
        return _stage_touched(arrs, wh, channels, arena, *touched, threads=threads)
    wh_at, offsets_at, offs, total = _image_layout(wh, channels)
    if arena.alignment % IMAGE_ALIGNMENT and IMAGE_ALIGNMENT % arena.alignment:
        raise DomainError("arena alignment must divide or be a multiple of 256")
    region = arena.alloc(total)
    if region.offset % IMAGE_ALIGNMENT:
        raise DomainError("image batches need 256-byte aligned regions (arena alignment 256)")
    view = region.view
    view[wh_at: wh_at + wh.nbytes] = wh.reshape(-1).view(np.uint8)
    view[offsets_at: offsets_at + offs.nbytes] = offs.view(np.uint8)
    entries = [BatchEntry(wh_at, wh.nbytes, "int32", wh.shape),
               BatchEntry(offsets_at, offs.nbytes, "int64", offs.shape)]
    _native_pack(arrs, wh, channels, view, offs, threads=threads)
    for a, off in zip(arrs, offs):
        entries.append(BatchEntry(int(off), int(a.size), "uint8", a.shape))
    batch = TransferBatch(payload=view[:total], entries=tuple(entries), copies=((0, total),),
                          slab=arena.tensor, base=region.offset)
    return StagedImages(batch, len(arrs), channels, wh, offs, wh_at, offsets_at)


def _touched_layout(wh, channels, tile_edge: int, max_tiles: int):
    """(maps, map_off, maps_all, offsets_at, map_off_at, map_at, image offsets, total)."""
    n = len(wh)
    maps = [staging_map(int(w), int(h), tile_edge, max_tiles) for w, h in wh]
    sizes = np.fromiter((m.size for m in maps), dtype=np.int64, count=n)
    map_off = np.zeros(n, dtype=np.int64)
    if n > 1:
        map_off[1:] = np.cumsum(sizes)[:-1]
    offsets_at = _round_up(8 * n, 8)
    map_off_at = offsets_at + 8 * n
    map_at = map_off_at + 8 * n
    mark = _round_up(map_at + 4 * int(sizes.sum()), IMAGE_ALIGNMENT)
    offs = np.empty(n, dtype=np.int64)
    for k in range(n):
        offs[k] = mark
        nr = int(maps[k][0])
        mark = _round_up(mark + nr * int(wh[k, 0]) * channels, IMAGE_ALIGNMENT)
    return maps, map_off, offsets_at, map_off_at, map_at, offs, max(mark, IMAGE_ALIGNMENT)


def _stage_touched(arrs, wh, channels, arena, tile_edge: int, max_tiles: int,
                   threads: int = 0) -> StagedImages:
    n = len(arrs)
    maps, map_off, offsets_at, map_off_at, map_at, offs, total = _touched_layout(
        wh, channels, tile_edge, max_tiles)
    wh_at = 0
    if arena.alignment % IMAGE_ALIGNMENT and IMAGE_ALIGNMENT % arena.alignment:
        raise DomainError("arena alignment must divide or be a multiple of 256")
    region = arena.alloc(total)
    if region.offset % IMAGE_ALIGNMENT:
        raise DomainError("image batches need 256-byte aligned regions (arena alignment 256)")
    view = region.view
    view[wh_at: wh_at + wh.nbytes] = wh.reshape(-1).view(np.uint8)
    view[offsets_at: offsets_at + offs.nbytes] = offs.view(np.uint8)
    view[map_off_at: map_off_at + map_off.nbytes] = map_off.view(np.uint8)
    maps_view = view[map_at: map_at + 4 * int(map_off[-1] + maps[-1].size)].view(np.int32)
    for m, o in zip(maps, map_off):
        maps_view[o: o + m.size] = m
    entries = [BatchEntry(wh_at, wh.nbytes, "int32", wh.shape),
               BatchEntry(offsets_at, offs.nbytes, "int64", offs.shape),
               BatchEntry(map_off_at, map_off.nbytes, "int64", map_off.shape),
               BatchEntry(map_at, maps_view.nbytes, "int32", maps_view.shape)]
    _native_pack(arrs, wh, channels, view, offs, maps_view, map_off, threads=threads)
    for a, m, off in zip(arrs, maps, offs):
        nr = int(m[0])
        entries.append(BatchEntry(int(off), nr * a.shape[1] * channels, "uint8",
                                  (nr, a.shape[1], channels)))
    batch = TransferBatch(payload=view[:total], entries=tuple(entries), copies=((0, total),),
                          slab=arena.tensor, base=region.offset)
    return StagedImages(batch, n, channels, wh, offs, wh_at, offsets_at, map_at,
                        int(maps_view.size), map_off_at, (int(tile_edge), int(max_tiles)))


def upload_images(staged: StagedImages, dest: torch.Tensor,
                  stream: Optional[torch.cuda.Stream] = None):
    """One asynchronous H2D copy of a staged batch into ``dest`` (CUDA uint8, at least
    the payload size); returns (PackedImages viewing ``dest``, event after the copy)."""
    from .engine import PackedImages  # engine imports nothing from here

    n = staged.n
    res = transfer(staged.batch, _COPY_MODEL, dest=dest, stream=stream)
    wh_t = dest[staged.wh_at: staged.wh_at + 8 * n].view(torch.int32).view(n, 2)
    off_t = dest[staged.offsets_at: staged.offsets_at + 8 * n].view(torch.int64)
    packed = PackedImages(dest, off_t, wh_t, staged.channels, staged.wh, staged.offsets)
    if staged.row_map_at is not None:
        packed.row_map = dest[staged.row_map_at: staged.row_map_at + 4 * staged.row_map_len].view(
            torch.int32)
        packed.row_map_off = dest[staged.row_map_off_at: staged.row_map_off_at + 8 * n].view(
            torch.int64)
        packed.touched_for = staged.touched_for
    return packed, res.done


_COPY_MODEL = CostModel(latency_per_copy=1e-5, bytes_per_second=5e10)


def staged_bytes(images: Sequence[np.ndarray], touched: Optional[tuple] = None) -> int:
    """Payload bytes ``stage_images`` needs for these images (same ``touched``)."""
    arrs, channels, wh = _hwc(images)
    if touched is None:
        return _image_layout(wh, channels)[3]
    return _touched_layout(wh, channels, *touched)[-1]


class PipelinedPreprocessor:
    """Host packing + one H2D copy per batch, overlapped with K1+K2 of the previous
    batch.

    ``depth`` pinned slabs and device slabs rotate: while the copy engine uploads batch
    i and the compute stream runs K1+K2 on it, the library's host thread pool
    (tp_stage_pack, the GIL released) packs batch i+1 into the next pinned slab; the
    compute stream waits only on that batch's copy event.  A pinned slab is reused
    after its copy has completed, a device slab after the K2 that read it has
    completed.  ``touched`` stages only the source rows the preprocessor's tiling reads
    (stage_images(touched=...)).  ``threads``: host packing threads (<= 0: all)."""

    def __init__(self, prep, slab_bytes: int, depth: int = 2, touched: bool = False,
                 threads: int = 0):
        if depth < 2:
            raise DomainError("depth must be >= 2 for overlap")
        self.prep = prep
        self.touched = (prep.cfg.tile_edge, prep.cfg.max_tiles) if touched else None
        self.device = prep.device
        self.depth = depth
        self.threads = int(threads)
        self.slab_bytes = _round_up(int(slab_bytes), IMAGE_ALIGNMENT)
        self.host = [HostArena(self.slab_bytes, IMAGE_ALIGNMENT, pin=True) for _ in range(depth)]
        self.dev = [torch.empty(self.slab_bytes, dtype=torch.uint8, device=self.device)
                    for _ in range(depth)]
        self.copy_stream = torch.cuda.Stream(self.device)
        self.compute_stream = torch.cuda.Stream(self.device)
        self._copied: list = [None] * depth  # event: copy from host slab k finished
        self._consumed: list = [None] * depth  # event: K2 reading device slab k finished
        self._i = 0
        self.last_bytes = 0  # payload bytes of the last submitted batch

    def submit(self, images: Sequence[np.ndarray], capacity: Optional[int] = None, out=None):
        """Pack ``images`` (HWC uint8 host arrays), upload them and enqueue K1+K2;
        returns the TileBatch (``out`` when given: reused buffers; its previous contents
        must no longer be needed).  Returns once the batch is packed and enqueued."""
        k = self._i % self.depth
        self._i += 1
        if self._copied[k] is not None:
            self._copied[k].synchronize()  # host slab k free again
        self.host[k].reset()
        staged = stage_images(images, self.host[k], touched=self.touched, threads=self.threads)
        self.last_bytes = len(staged.batch.payload)
        if self._consumed[k] is not None:
            self.copy_stream.wait_event(self._consumed[k])  # device slab k free again
        packed, copied = upload_images(staged, self.dev[k], self.copy_stream)
        self._copied[k] = copied
        self.compute_stream.wait_event(copied)
        with torch.cuda.stream(self.compute_stream):  # outputs belong to this stream
            res = self.prep(packed, capacity=capacity, out=out, stream=self.compute_stream)
        done = torch.cuda.Event()
        done.record(self.compute_stream)
        self._consumed[k] = done
        return res

    def run(self, batches: Iterable[Sequence[np.ndarray]], capacity: Optional[int] = None):
        """Preprocess each batch; returns one TileBatch per batch (device tensors, all
        work enqueued on the compute stream; synchronise or wait on it before use)."""
        return [self.submit(images, capacity=capacity) for images in batches]

    def synchronize(self) -> None:
        self.compute_stream.synchronize()
