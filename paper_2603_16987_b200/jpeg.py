"""Device JPEG decode (K7, csrc/jpeg.cu): compressed payloads in, packed RGB HWC images
in HBM out -- the input layout of K1/K2 (engine.PackedImages).

The reference decodes every image with Pillow on the host (vlmfp/imgproc.py:213-229);
for the baseline JPEGs Pillow itself writes (and the reference corpus holds,
pkg/scripts/make_corpus.py:139-142) the decode runs on the B200 instead, bit-exact with
Pillow's libjpeg-turbo.  Only the compressed bytes cross PCIe (a corpus-like 1080p q85
JPEG is ~0.5 MB against 6.2 MB of pixels).  Payloads the device decoder does not take
(PNG, progressive / arithmetic / 12-bit JPEG, CMYK, unusual sampling) and streams it
finds unclean are decoded on the host with Pillow -- the reference's own decoder, so the
pixels (or the DecodeError) are the reference's.

    dec = JpegDecoder(device)
    batch = dec.decode(payloads)          # engine.PackedImages on the device
    tiles = TilePreprocessor(cfg, device)(batch)
"""

from __future__ import annotations

import ctypes
from ctypes import c_char, c_int32, c_int64, c_uint8, c_uint16
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .engine import PackedImages, layout_offsets
from .runtime import require_device, stream_handle

TP_JPEG_OK = 0
TP_JPEG_UNSUPPORTED = 1
TP_JPEG_CORRUPT = 2
DEFAULT_SUB_BITS = 0  # 0: by batch size (small batches: short subsequences, more threads)


class TpJpegInfo(ctypes.Structure):
    """include/tileprep.h TpJpegInfo."""

    _fields_ = [
        ("status", c_int32), ("width", c_int32), ("height", c_int32), ("ncomp", c_int32),
        ("comp_id", c_int32 * 3), ("comp_h", c_int32 * 3), ("comp_v", c_int32 * 3),
        ("comp_tq", c_int32 * 3), ("comp_td", c_int32 * 3), ("comp_ta", c_int32 * 3),
        ("restart_interval", c_int32), ("qt_mask", c_int32), ("dc_mask", c_int32),
        ("ac_mask", c_int32), ("scan_off", c_int64), ("scan_len", c_int64),
        ("qt", (c_uint16 * 64) * 4), ("dc_bits", (c_uint8 * 16) * 2),
        ("dc_vals", (c_uint8 * 256) * 2), ("ac_bits", (c_uint8 * 16) * 2),
        ("ac_vals", (c_uint8 * 256) * 2), ("message", c_char * 96),
    ]


def parse(payload: bytes, info: Optional[TpJpegInfo] = None) -> TpJpegInfo:
    """tp_jpeg_parse of one payload (host): frame, tables, scan extent, and whether the
    device decoder takes it (``status``)."""
    info = info if info is not None else TpJpegInfo()
    if len(payload) < 4 or payload[:2] != b"\xff\xd8":
        info.status = TP_JPEG_UNSUPPORTED  # PNG or not an image: the host decoder decides
        return info
    _lib.call("tp_jpeg_parse", ctypes.cast(ctypes.c_char_p(payload), ctypes.c_void_p),
              len(payload), ctypes.byref(info))
    return info


def _host_decode(payload: bytes) -> np.ndarray:
    """The reference's decode (Pillow) of one payload the device does not take."""
    from ._decode import decode_rgb

    return decode_rgb(payload)


def _round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


class _Slot:
    """One in-flight batch's buffers: pinned staging, device payload, workspace, status."""

    def __init__(self):
        self.host = None
        self.dev = None
        self.work = None
        self.status = None
        self.status_host = None
        self.copied = None  # event: the upload out of `host` finished
        self.done = None    # event: the decode (and the status copy) finished
        self.meta_host = None  # pinned image offsets / sizes of the output batch
        self.meta_copied = None


class JpegBatch:
    """A submitted batch: ``images`` (device, filled by the decode enqueued on the
    stream) and ``finish()``, which waits for the decode and patches in the images the
    host decoder must take (returns their indices; the caller re-runs anything it
    enqueued on ``images`` when the list is not empty)."""

    def __init__(self, dec, slot, payloads, images, host_arrays, wh, out_off, n):
        self._dec, self._slot, self._payloads = dec, slot, payloads
        self.images = images
        self._host_arrays, self._wh, self._out_off, self._n = host_arrays, wh, out_off, n
        self.fallback: Optional[list] = None

    def finish(self) -> list:
        if self.fallback is not None:
            return self.fallback
        sl = self._slot
        sl.done.synchronize()
        st = sl.status_host[: self._n].numpy()
        fb = sorted(set(self._host_arrays) | {k for k in range(self._n) if st[k] != 0})
        for k in fb:
            a = self._host_arrays.get(k)
            if a is None:
                a = _host_decode(self._payloads[k])
                if (a.shape[1], a.shape[0]) != tuple(self._wh[k]):
                    raise RuntimeError("host decode size differs from the JPEG frame header")
            o = int(self._out_off[k])
            self.images.data[o: o + a.size].copy_(
                torch.from_numpy(np.ascontiguousarray(a).reshape(-1).copy()))
        self.fallback = fb
        self._dec.last_fallback = fb
        return fb


class JpegDecoder:
    """Batched device JPEG decode into a packed RGB batch.

    ``sub_bits``: subsequence length of the parallel Huffman decode (bits per thread).
    ``depth`` buffer sets rotate, so with ``sync=False`` the host work of batch i+1
    (marker parse, descriptors, packing the scans into the pinned slab) overlaps the
    upload and decode of batch i.  Buffers grow on demand and are reused."""

    def __init__(self, device=None, sub_bits: int = DEFAULT_SUB_BITS, depth: int = 2,
                 lead_bits: int = 0):
        self.device = require_device(device)
        self.sub_bits = int(sub_bits)    # 0: chosen per batch (_pick)
        self.lead_bits = int(lead_bits)  # speculative lead-in per subsequence (0: sub_bits)
        self.lib = _lib.load()
        self.desc_bytes = int(self.lib.tp_jpeg_desc_bytes())
        self.slots = [_Slot() for _ in range(max(1, depth))]
        self._i = 0
        self.last_fallback: list[int] = []  # images decoded on the host in the last call
        self.last_h2d_bytes = 0
        self._last = None
        # uploads run on their own stream, so batch i+1's H2D overlaps batch i's decode
        self._copy_stream = torch.cuda.Stream(self.device)

    @property
    def _work(self):  # diagnostics (tools/jpeg_bench.py): the last batch's workspace
        return self._last[0].work

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
        fallbacks patched in; sync=False: returns a JpegBatch (call finish())."""
        n = len(payloads)
        if n == 0:
            raise ValueError("no payloads")
        infos = (TpJpegInfo * n)()
        host_arrays: dict[int, np.ndarray] = {}
        wh = np.zeros((n, 2), dtype=np.int32)
        for k, p in enumerate(payloads):
            parse(p, infos[k])
            if infos[k].status == TP_JPEG_OK and infos[k].scan_len < 1:
                infos[k].status = TP_JPEG_CORRUPT
            if infos[k].status == TP_JPEG_OK:
                wh[k] = (infos[k].width, infos[k].height)
            else:  # the reference's decoder; raises DecodeError like the reference
                a = _host_decode(p)
                host_arrays[k] = a
                wh[k] = (a.shape[1], a.shape[0])
        out_off, out_total = layout_offsets(wh, 3)
        # staged payload: [descriptors][scan bytes of every device-decoded image]
        desc_at = 0
        mark = _round_up(n * self.desc_bytes, 256)
        raw_off = np.zeros(n, dtype=np.int64)
        scan_len = np.array([infos[k].scan_len for k in range(n)], dtype=np.int64)
        ok = np.array([infos[k].status == TP_JPEG_OK for k in range(n)])
        sizes = np.where(ok, (scan_len + 64 + 15) // 16 * 16, 0)
        raw_off[:] = mark + np.concatenate([[0], np.cumsum(sizes)[:-1]]) if n else 0
        raw_off[~ok] = 0
        payload_bytes = _round_up(int(mark + sizes.sum()), 256)
        totals = np.zeros(8, dtype=np.int64)
        pixels = sum(int(infos[k].width) * int(infos[k].height) for k in range(n) if ok[k])
        sub_bits, lead_bits = self._pick(int(8 * scan_len[ok].sum()), pixels)
        sl = self.slots[self._i % len(self.slots)]
        self._i += 1
        if sl.copied is not None:
            sl.copied.synchronize()  # the slot's previous upload no longer reads the slab
        if sl.done is not None:
            sl.done.synchronize()  # nor its decode the workspace / status
        desc_host = (ctypes.c_uint8 * (n * self.desc_bytes))()
        work_bytes = int(self.lib.tp_jpeg_describe(
            ctypes.byref(infos), n, raw_off.ctypes.data, out_off.ctypes.data, sub_bits,
            ctypes.cast(desc_host, ctypes.c_void_p), totals.ctypes.data))
        if work_bytes < 0:
            _lib.check(-work_bytes, "tp_jpeg_describe")
        totals[7] = lead_bits
        self._buffers(sl, payload_bytes, max(work_bytes, 4096), n)
        ctypes.memmove(sl.host.data_ptr() + desc_at, desc_host, n * self.desc_bytes)
        dev_idx = np.nonzero(ok)[0]
        if len(dev_idx):  # scan bytes into the pinned slab on the host thread pool
            keep = [np.frombuffer(payloads[k], dtype=np.uint8) for k in dev_idx]
            src = np.array([a.ctypes.data + int(infos[k].scan_off) for a, k in zip(keep, dev_idx)],
                           dtype=np.uint64)
            lens = np.stack([scan_len[dev_idx], np.ones(len(dev_idx), np.int64)], 1).astype(np.int32)
            stride = scan_len[dev_idx].copy()
            dst_off = raw_off[dev_idx].copy()
            _lib.call("tp_stage_pack", len(dev_idx), src.ctypes.data, stride.ctypes.data,
                      lens.ctypes.data, 1, None, None, sl.host.data_ptr(), dst_off.ctypes.data, 0)
        self.last_h2d_bytes = payload_bytes
        stream = stream or torch.cuda.current_stream(self.device)
        if out is None:
            data = torch.empty(out_total, dtype=torch.uint8, device=self.device)
            # offsets and sizes ride in the slot's pinned slab (no per-call pinning)
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
        # the slot's previous decode finished (sl.done above), so the upload may start at
        # once on the copy stream; the decode waits for it on `stream`
        cs = self._copy_stream
        with torch.cuda.stream(cs):
            sl.dev[:payload_bytes].copy_(sl.host[:payload_bytes], non_blocking=True)
            sl.copied = torch.cuda.Event()
            sl.copied.record(cs)
        stream.wait_event(sl.copied)
        self._last = (sl, desc_at, n, totals, out, sub_bits)
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

    def _pick(self, scan_bits: int, pixels: int = 0) -> tuple:
        """(sub_bits, lead_bits) for a batch of `scan_bits` entropy-coded bits.  Measured on
        corpus-like 1080p JPEGs (profiles/r02/jpeg/): one image decodes fastest with short
        subsequences and a long lead-in (1024 + 2048: K7 0.69 ms, decode() 1.0 ms; 4096:
        1.71 ms per call), 64 images with 4096-bit subsequences and a 2048-bit lead-in
        (2.47 ms; 2.56 ms with a 4096-bit lead-in, profiles/r02/jpeg/lead_sweep.log), and a
        6144-bit lead-in for noise-like content."""
        if self.sub_bits:
            return self.sub_bits, self.lead_bits
        if scan_bits < 32 * 2**20:  # fewer than ~8 corpus-like 1080p images
            return 1024, 2048
        if pixels and scan_bits >= 4 * pixels:
            # high-entropy content (>= 4 coded bits per pixel, noise-like): longer lead-ins
            # cut the re-decode half-rounds (16 noise 1080p JPEGs: 2.75 -> 2.63 ms)
            return 4096, 6144
        return 4096, 2048

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """(Re)launch the device decode of the last uploaded batch (K7 only: no host work,
        no copies) -- what tools/jpeg_bench.py times as the decode kernels."""
        sl, desc_at, n, totals, out, sub_bits = self._last
        stream = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            _lib.call("tp_jpeg_decode", sl.dev.data_ptr(), sl.dev.data_ptr() + desc_at, n,
                      totals.ctypes.data, sub_bits, sl.work.data_ptr(),
                      sl.work.numel(), out.data.data_ptr(), sl.status.data_ptr(),
                      stream_handle(self.device, stream))


def decode_images(payloads: Sequence[bytes], device=None) -> list[np.ndarray]:
    """Convenience: device decode, then copy every image back as an (H, W, 3) array."""
    dec = JpegDecoder(device)
    pk = dec.decode(payloads)
    host = pk.data.cpu().numpy()
    return [host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            for o, (w, h) in zip(pk.offsets_host, pk.wh_host)]


__all__ = ["JpegBatch", "JpegDecoder", "TpJpegInfo", "decode_images", "parse",
           "TP_JPEG_OK", "TP_JPEG_UNSUPPORTED", "TP_JPEG_CORRUPT"]
