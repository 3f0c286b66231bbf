"""Device PNG decode (K8, csrc/png.cu): compressed payloads in, packed RGB HWC images in
HBM out -- the input layout of K1/K2 (engine.PackedImages).

The reference decodes every image with Pillow on the host (vlmfp/imgproc.py:213-229).
For 8-bit greyscale, RGB and palette PNGs (modes "L", "RGB", "P": the reference's
accepted modes, imgproc.py:26) the inflate, the scanline unfiltering and the L/P -> RGB
expansion run on the B200 instead; PNG is lossless, so the pixels are Pillow's by
construction.  Only the IDAT bytes cross PCIe.  Payloads the host parser leaves to
Pillow (other bit depths, interlacing, chunks whose Pillow handlers can raise, bad
header CRCs -- csrc/png_host.cu) and streams the device finds unclean (corrupt,
truncated, a block chain the finder could not close) are decoded on the host with
Pillow, the reference's own decoder, so the pixels (or the DecodeError) are the
reference's.

    dec = PngDecoder(device)
    batch = dec.decode(payloads)          # engine.PackedImages on the device
    tiles = TilePreprocessor(cfg, device)(batch)
"""

from __future__ import annotations

import ctypes
from ctypes import c_char, c_int32, c_int64, c_uint8
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .engine import PackedImages, layout_offsets
from .jpeg import JpegBatch, _host_decode, _round_up, _Slot
from .runtime import require_device, stream_handle

TP_PNG_OK = 0
TP_PNG_UNSUPPORTED = 1
PNG_SIGNATURE = b"\x89PNG\r\n\x1a\n"


class TpPngInfo(ctypes.Structure):
    """include/tileprep.h TpPngInfo."""

    _fields_ = [
        ("status", c_int32), ("width", c_int32), ("height", c_int32), ("bit_depth", c_int32),
        ("color_type", c_int32), ("interlace", c_int32), ("pal_n", c_int32), ("n_idat", c_int32),
        ("zlib_len", c_int64), ("pal", c_uint8 * 768), ("message", c_char * 96),
    ]


def parse(payload: bytes, info: Optional[TpPngInfo] = None, cap: int = 256):
    """tp_png_parse of one payload (host): the header fields, whether the device decoder
    takes it (``status``), and the IDAT data extents (offsets, lengths) in the payload."""
    info = info if info is not None else TpPngInfo()
    buf = ctypes.c_char_p(payload)
    while True:
        offs = np.zeros(cap, dtype=np.int64)
        lens = np.zeros(cap, dtype=np.int64)
        _lib.call("tp_png_parse", ctypes.cast(buf, ctypes.c_void_p), len(payload),
                  ctypes.byref(info), offs.ctypes.data, lens.ctypes.data, cap)
        if info.n_idat <= cap:
            return info, offs[: info.n_idat], lens[: info.n_idat]
        cap = int(info.n_idat)


class PngDecoder:
    """Batched device PNG decode into a packed RGB batch.

    ``depth`` buffer sets rotate, so with ``sync=False`` the host work of batch i+1
    (chunk walk, packing the IDAT data into the pinned slab) overlaps the upload and
    decode of batch i.  Buffers grow on demand and are reused."""

    def __init__(self, device=None, depth: int = 2, max_work_bytes: int = 8 << 30):
        self.device = require_device(device)
        self.max_work_bytes = int(max_work_bytes)
        self._debug_flags = 0  # tests only: bit 0 plants false finder starts
        self.lib = _lib.load()
        self.desc_bytes = int(self.lib.tp_png_desc_bytes())
        self.slots = [_Slot() for _ in range(max(1, depth))]
        self._i = 0
        self.last_fallback: list[int] = []
        self.last_h2d_bytes = 0
        self._last = None
        self._copy_stream = torch.cuda.Stream(self.device)

    def _buffers(self, sl: _Slot, payload_bytes: int, work_bytes: int, n: int):
        if sl.host is None or sl.host.numel() < payload_bytes:
            cap = _round_up(int(payload_bytes * 1.25) + 4096, 1 << 20)
            sl.host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            sl.dev = torch.empty(cap, dtype=torch.uint8, device=self.device)
        if sl.work is None or sl.work.numel() < work_bytes:
            sl.work = torch.empty(_round_up(int(work_bytes * 1.25) + 4096, 1 << 20),
                                  dtype=torch.uint8, device=self.device)
        if sl.status is None or sl.status.numel() < n:
            cap = _round_up(n, 256)
            sl.status = torch.empty(cap, dtype=torch.int32, device=self.device)
            sl.status_host = torch.empty(cap, dtype=torch.int32, pin_memory=True)

    def decode(self, payloads: Sequence[bytes], out: Optional[PackedImages] = None,
               stream: Optional[torch.cuda.Stream] = None, sync: bool = True):
        """Decode every payload to RGB uint8 HWC in one packed device batch (the
        engine.layout_offsets layout).  sync=True: returns the PackedImages with host
        fallbacks patched in; sync=False: returns a batch handle (call finish())."""
        n = len(payloads)
        if n == 0:
            raise ValueError("no payloads")
        infos = (TpPngInfo * n)()
        extents = [None] * n
        host_arrays: dict[int, np.ndarray] = {}
        wh = np.zeros((n, 2), dtype=np.int32)
        for k, p in enumerate(payloads):
            if p[:8] == PNG_SIGNATURE:
                _, offs, lens = parse(p, infos[k])
                extents[k] = (offs, lens)
            else:
                infos[k].status = TP_PNG_UNSUPPORTED
            if infos[k].status == TP_PNG_OK:
                wh[k] = (infos[k].width, infos[k].height)
            else:  # the reference's decoder; raises DecodeError like the reference
                a = _host_decode(p)
                host_arrays[k] = a
                wh[k] = (a.shape[1], a.shape[0])
        out_off, out_total = layout_offsets(wh, 3)
        ok = np.array([infos[k].status == TP_PNG_OK for k in range(n)])
        zlen = np.array([infos[k].zlib_len for k in range(n)], dtype=np.int64)
        # workspace per device image (csrc/png_host.cu tp_png_describe): tokens 16 B per
        # compressed byte (indexed by bit / 2), T + R + marker lists 7 B per pixel byte,
        # token staging per 48 KB unit; large batches decode in sub-batches that fit
        est = np.where(ok, 16 * zlen + 7 * wh[:, 0].astype(np.int64) * wh[:, 1] * 3
                       + (zlen // 49152 + 1) * 73728, 0)
        if n > 1 and int(est.sum()) > self.max_work_bytes:
            return self._decode_chunked(payloads, est, wh, out_off, out_total, out, stream, sync)
        mark = _round_up(n * self.desc_bytes, 256)
        sizes = np.where(ok, (zlen + 64 + 15) // 16 * 16, 0)  # 64 readable bytes after
        in_off = mark + np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        in_off[~ok] = -1
        payload_bytes = _round_up(int(mark + sizes.sum()) + 64, 256)
        totals = np.zeros(16, dtype=np.int64)
        sl = self.slots[self._i % len(self.slots)]
        self._i += 1
        if sl.copied is not None:
            sl.copied.synchronize()
        if sl.done is not None:
            sl.done.synchronize()
        desc_host = (ctypes.c_uint8 * (n * self.desc_bytes))()
        work_bytes = int(self.lib.tp_png_describe(
            ctypes.byref(infos), n, in_off.ctypes.data, out_off.ctypes.data,
            ctypes.cast(desc_host, ctypes.c_void_p), totals.ctypes.data))
        if work_bytes < 0:
            _lib.check(-work_bytes, "tp_png_describe")
        totals[15] = self._debug_flags  # test hooks (csrc/png_common.cuh)
        self._buffers(sl, payload_bytes, max(work_bytes, 4096), n)
        ctypes.memmove(sl.host.data_ptr(), desc_host, n * self.desc_bytes)
        dev_idx = np.nonzero(ok)[0]
        if len(dev_idx):  # IDAT data back to back per image, on the host thread pool
            keep, src, rows, dst = [], [], [], []
            for k in dev_idx:
                a = np.frombuffer(payloads[k], dtype=np.uint8)
                keep.append(a)
                offs, lens = extents[k]
                d = int(in_off[k])
                for o, ln in zip(offs.tolist(), lens.tolist()):
                    if ln:
                        src.append(a.ctypes.data + o)
                        rows.append(ln)
                        dst.append(d)
                    d += ln
            if src:
                m = len(src)
                src_a = np.array(src, dtype=np.uint64)
                wh_a = np.stack([np.array(rows, np.int32), np.ones(m, np.int32)], 1).astype(np.int32)
                stride = np.array(rows, dtype=np.int64)
                dst_a = np.array(dst, dtype=np.int64)
                _lib.call("tp_stage_pack", m, src_a.ctypes.data, stride.ctypes.data,
                          wh_a.ctypes.data, 1, None, None, sl.host.data_ptr(), dst_a.ctypes.data, 0)
        self.last_h2d_bytes = payload_bytes
        stream = stream or torch.cuda.current_stream(self.device)
        if out is None:
            data = torch.empty(out_total, dtype=torch.uint8, device=self.device)
            if sl.meta_host is None or sl.meta_host.numel() < 3 * n:
                sl.meta_host = torch.empty(3 * _round_up(n, 64), dtype=torch.int64, pin_memory=True)
            if sl.meta_copied is not None:
                sl.meta_copied.synchronize()
            mh = sl.meta_host.numpy()
            mh[:n] = out_off
            mh[n: 3 * n] = wh.reshape(-1)
            meta = torch.empty(3 * n, dtype=torch.int64, device=self.device)
            with torch.cuda.stream(stream):
                meta.copy_(sl.meta_host[: 3 * n], non_blocking=True)
                sl.meta_copied = torch.cuda.Event()
                sl.meta_copied.record(stream)
                wh_dev = meta[n:].to(torch.int32).view(n, 2)
            out = PackedImages(data, meta[:n], wh_dev, 3, wh, out_off)
        cs = self._copy_stream
        with torch.cuda.stream(cs):
            sl.dev[:payload_bytes].copy_(sl.host[:payload_bytes], non_blocking=True)
            sl.copied = torch.cuda.Event()
            sl.copied.record(cs)
        stream.wait_event(sl.copied)
        self._last = (sl, n, totals, out)
        self.launch(stream)
        with torch.cuda.stream(stream):
            sl.status_host[:n].copy_(sl.status[:n], non_blocking=True)
            sl.done = torch.cuda.Event()
            sl.done.record(stream)
        batch = JpegBatch(self, sl, payloads, out, host_arrays, wh, out_off, n)
        if not sync:
            return batch
        batch.finish()
        return out

    def _decode_chunked(self, payloads, est, wh, out_off, out_total, out, stream, sync):
        """Sub-batches of at most max_work_bytes of workspace, decoded in turn into one
        output batch (the layout of a run of images is the batch layout shifted by the
        run's first offset)."""
        n = len(payloads)
        if out is None:
            out = PackedImages(torch.empty(out_total, dtype=torch.uint8, device=self.device),
                               torch.as_tensor(out_off, device=self.device),
                               torch.as_tensor(wh, device=self.device), 3, wh, out_off)
        parts, i = [], 0
        while i < n:
            j, acc = i, 0
            while j < n and (j == i or acc + int(est[j]) <= self.max_work_bytes):
                acc += int(est[j])
                j += 1
            o0 = int(out_off[i])
            sub_off = out_off[i:j] - o0
            end = int(out_off[j]) if j < n else out_total
            view = PackedImages(out.data[o0:end], out.offsets[i:j] - o0, out.wh[i:j], 3,
                                wh[i:j], sub_off)
            parts.append((i, self.decode(payloads[i:j], out=view, stream=stream, sync=False)))
            i = j
        batch = _ChunkedBatch(self, parts, out)
        if not sync:
            return batch
        batch.finish()
        return out

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """(Re)launch the device decode of the last uploaded batch (K8 only: no host
        work, no copies) -- what the bench times as the decode kernels."""
        sl, n, totals, out = self._last
        stream = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            _lib.call("tp_png_decode", sl.dev.data_ptr(), sl.dev.data_ptr(), n,
                      totals.ctypes.data, sl.work.data_ptr(), sl.work.numel(),
                      out.data.data_ptr(), sl.status.data_ptr(),
                      stream_handle(self.device, stream))

    def last_status(self) -> np.ndarray:
        """Device status of the last batch (0: decoded on the device); synchronises."""
        sl, n, _, _ = self._last
        sl.done.synchronize()
        return sl.status_host[:n].numpy().copy()


class _ChunkedBatch:
    """Sub-batches of one decode: ``images`` is the whole output, ``finish()`` finishes
    every part and returns the host-decoded indices of the whole batch."""

    def __init__(self, dec, parts, images):
        self._dec, self._parts, self.images = dec, parts, images
        self.fallback: Optional[list] = None

    def finish(self) -> list:
        if self.fallback is None:
            self.fallback = sorted(i0 + k for i0, b in self._parts for k in b.finish())
            self._dec.last_fallback = self.fallback
        return self.fallback


def decode_images(payloads: Sequence[bytes], device=None) -> list[np.ndarray]:
    """Convenience: device decode, then copy every image back as an (H, W, 3) array."""
    dec = PngDecoder(device)
    pk = dec.decode(payloads)
    host = pk.data.cpu().numpy()
    return [host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            for o, (w, h) in zip(pk.offsets_host, pk.wh_host)]


__all__ = ["PngDecoder", "TpPngInfo", "decode_images", "parse", "TP_PNG_OK",
           "TP_PNG_UNSUPPORTED"]
