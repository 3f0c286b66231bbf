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
DEFAULT_SUB_BITS = 2048


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


class JpegDecoder:
    """Batched device JPEG decode into a packed RGB batch.

    ``sub_bits``: subsequence length of the parallel Huffman decode (bits per thread).
    Pinned staging, device payload and workspace buffers grow on demand and are reused
    across calls (one decoder per stream)."""

    def __init__(self, device=None, sub_bits: int = DEFAULT_SUB_BITS):
        self.device = require_device(device)
        self.sub_bits = int(sub_bits)
        self.lib = _lib.load()
        self.desc_bytes = int(self.lib.tp_jpeg_desc_bytes())
        self._host = None
        self._dev = None
        self._work = None
        self.last_fallback: list[int] = []  # images decoded on the host in the last call
        self.last_h2d_bytes = 0
        self._copied = None  # event: the last upload out of the pinned slab finished

    def _buffers(self, payload_bytes: int, work_bytes: int):
        if self._host is None or self._host.numel() < payload_bytes:
            cap = _round_up(int(payload_bytes * 1.25) + 4096, 1 << 20)
            self._host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self._dev = torch.empty(cap, dtype=torch.uint8, device=self.device)
        if self._work is None or self._work.numel() < work_bytes:
            self._work = torch.empty(_round_up(int(work_bytes * 1.25) + 4096, 1 << 20),
                                     dtype=torch.uint8, device=self.device)

    def decode(self, payloads: Sequence[bytes], out: Optional[PackedImages] = None,
               stream: Optional[torch.cuda.Stream] = None, sync: bool = True) -> PackedImages:
        """Decode every payload to RGB uint8 HWC in one packed device batch (the
        engine.layout_offsets layout).  Host fallbacks are patched in before returning."""
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
        for k in range(n):
            if infos[k].status == TP_JPEG_OK:
                raw_off[k] = mark
                mark = _round_up(mark + int(infos[k].scan_len) + 64, 16)
        payload_bytes = _round_up(mark, 256)
        totals = np.zeros(5, dtype=np.int64)
        desc_host = (ctypes.c_uint8 * (n * self.desc_bytes))()
        work_bytes = int(self.lib.tp_jpeg_describe(
            ctypes.byref(infos), n, raw_off.ctypes.data, out_off.ctypes.data, self.sub_bits,
            ctypes.cast(desc_host, ctypes.c_void_p), totals.ctypes.data))
        if work_bytes < 0:
            _lib.check(-work_bytes, "tp_jpeg_describe")
        if self._copied is not None:
            self._copied.synchronize()  # the previous upload no longer reads the slab
        self._buffers(payload_bytes, max(work_bytes, 4096))
        hv = self._host.numpy()
        hv[desc_at: desc_at + n * self.desc_bytes] = np.frombuffer(desc_host, dtype=np.uint8)
        dev_idx = [k for k in range(n) if infos[k].status == TP_JPEG_OK]
        if dev_idx:  # scan bytes into the pinned slab on the host thread pool
            keep = [np.frombuffer(payloads[k], dtype=np.uint8) for k in dev_idx]
            src = np.array([a.ctypes.data + int(infos[k].scan_off) for a, k in zip(keep, dev_idx)],
                           dtype=np.uint64)
            lens = np.array([[int(infos[k].scan_len), 1] for k in dev_idx], dtype=np.int32)
            stride = lens[:, 0].astype(np.int64).copy()
            dst_off = raw_off[dev_idx].copy()
            _lib.call("tp_stage_pack", len(dev_idx), src.ctypes.data, stride.ctypes.data,
                      lens.ctypes.data, 1, None, None, self._host.data_ptr(), dst_off.ctypes.data, 0)
        self.last_h2d_bytes = payload_bytes
        if out is None:
            data = torch.empty(out_total, dtype=torch.uint8, device=self.device)
            out = PackedImages(data, torch.from_numpy(out_off).to(self.device),
                               torch.from_numpy(wh.copy()).to(self.device), 3, wh, out_off)
        stream = stream or torch.cuda.current_stream(self.device)
        status = torch.empty(n, dtype=torch.int32, device=self.device)
        with torch.cuda.stream(stream):
            self._dev[:payload_bytes].copy_(self._host[:payload_bytes], non_blocking=True)
            self._copied = torch.cuda.Event()
            self._copied.record(stream)
        self._launch_args = (desc_at, n, totals, out, status)
        self.launch(stream)
        self._status = status
        if not sync:
            return out
        st = status.cpu().numpy()  # synchronises the stream (the host slab is reusable)
        self.last_fallback = sorted(set(host_arrays) | {k for k in range(n) if st[k] != 0})
        for k in self.last_fallback:
            a = host_arrays.get(k)
            if a is None:
                a = _host_decode(payloads[k])
                if (a.shape[1], a.shape[0]) != tuple(wh[k]):
                    raise RuntimeError("host decode size differs from the JPEG frame header")
            o = int(out_off[k])
            out.data[o: o + a.size].copy_(torch.from_numpy(np.ascontiguousarray(a).reshape(-1)))
        return out


    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """(Re)launch the device decode of the last uploaded batch (K7 only: no host work,
        no copies) -- what bench.py times as the decode kernels."""
        desc_at, n, totals, out, status = self._launch_args
        stream = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            _lib.call("tp_jpeg_decode", self._dev.data_ptr(), self._dev.data_ptr() + desc_at, n,
                      totals.ctypes.data, self.sub_bits, self._work.data_ptr(),
                      self._work.numel(), out.data.data_ptr(), status.data_ptr(),
                      stream_handle(self.device, stream))


def decode_images(payloads: Sequence[bytes], device=None) -> list[np.ndarray]:
    """Convenience: device decode, then copy every image back as an (H, W, 3) array."""
    dec = JpegDecoder(device)
    pk = dec.decode(payloads)
    host = pk.data.cpu().numpy()
    return [host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            for o, (w, h) in zip(pk.offsets_host, pk.wh_host)]


__all__ = ["JpegDecoder", "TpJpegInfo", "decode_images", "parse",
           "TP_JPEG_OK", "TP_JPEG_UNSUPPORTED", "TP_JPEG_CORRUPT"]
