"""Mixed batches of compressed images decoded on the device: baseline JPEGs through K7
(`jpeg.JpegDecoder`), 8-bit L / RGB / P PNGs through K8 (`png.PngDecoder`), everything
else through Pillow on the host (the reference's decoder, vlmfp/imgproc.py:213-229) --
into one packed RGB batch in the caller's order, the input layout of K1/K2.

    dec = ImageDecoder("cuda")
    images = dec.decode(payloads)          # engine.PackedImages on the device
    tiles = TilePreprocessor(cfg, "cuda")(images)

Single-format batches go straight to their decoder (no extra copy); mixed ones are
decoded per format and gathered into the caller's order with device copies.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from .engine import PackedImages, layout_offsets
from .jpeg import JpegDecoder, _host_decode
from .png import PNG_SIGNATURE, PngDecoder
from .runtime import require_device


class ImageDecoder:
    """Batched device decode of mixed JPEG / PNG payloads (host Pillow for the rest)."""

    def __init__(self, device=None):
        self.device = require_device(device)
        self.jpeg = JpegDecoder(self.device)
        self.png = PngDecoder(self.device)
        self.last_fallback: list[int] = []  # indices Pillow decoded on the host

    def decode(self, payloads: Sequence[bytes],
               stream: Optional[torch.cuda.Stream] = None) -> PackedImages:
        n = len(payloads)
        if n == 0:
            raise ValueError("no payloads")
        stream = stream or torch.cuda.current_stream(self.device)
        jpg = [i for i, p in enumerate(payloads) if p[:2] == b"\xff\xd8"]
        png = [i for i, p in enumerate(payloads) if p[:8] == PNG_SIGNATURE]
        other = sorted(set(range(n)) - set(jpg) - set(png))
        if len(jpg) == n or (len(png) == 0 and other):
            out = self.jpeg.decode(payloads, stream=stream)  # the rest via Pillow inside
            self.last_fallback = list(self.jpeg.last_fallback)
            return out
        if len(png) == n:
            out = self.png.decode(payloads, stream=stream)
            self.last_fallback = list(self.png.last_fallback)
            return out
        parts = []  # (indices, PackedImages or None for host arrays, host arrays)
        fallback = []
        if jpg:
            parts.append((jpg, self.jpeg.decode([payloads[i] for i in jpg], stream=stream)))
            fallback += [jpg[k] for k in self.jpeg.last_fallback]
        if png:
            parts.append((png, self.png.decode([payloads[i] for i in png], stream=stream)))
            fallback += [png[k] for k in self.png.last_fallback]
        host = {i: _host_decode(payloads[i]) for i in other}  # raises like the reference
        fallback += other
        wh = np.zeros((n, 2), dtype=np.int32)
        for idx, pk in parts:
            wh[idx] = pk.wh_host
        for i, a in host.items():
            wh[i] = (a.shape[1], a.shape[0])
        out_off, total = layout_offsets(wh, 3)
        data = torch.empty(total, dtype=torch.uint8, device=self.device)
        with torch.cuda.stream(stream):
            for idx, pk in parts:
                for k, i in enumerate(idx):
                    size = int(wh[i, 0]) * int(wh[i, 1]) * 3
                    o, so = int(out_off[i]), int(pk.offsets_host[k])
                    data[o: o + size].copy_(pk.data[so: so + size], non_blocking=True)
            for i, a in host.items():
                o = int(out_off[i])
                data[o: o + a.size].copy_(torch.from_numpy(np.ascontiguousarray(a).reshape(-1)),
                                          non_blocking=False)
            offsets = torch.as_tensor(out_off, device=self.device)
            wh_dev = torch.as_tensor(wh, device=self.device)
        self.last_fallback = sorted(fallback)
        return PackedImages(data, offsets, wh_dev, 3, wh, out_off)


def decode_images(payloads: Sequence[bytes], device=None) -> list[np.ndarray]:
    """Convenience: device decode of a mixed batch, copied back as (H, W, 3) arrays."""
    pk = ImageDecoder(device).decode(payloads)
    host = pk.data.cpu().numpy()
    return [host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            for o, (w, h) in zip(pk.offsets_host, pk.wh_host)]


__all__ = ["ImageDecoder", "decode_images"]
