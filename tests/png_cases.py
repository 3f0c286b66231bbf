"""PNG test inputs shared by the CPU and GPU decode tests: payloads written by Pillow (the
encoder of the reference's own PNG paths: decode_image's re-encode, imgproc.py:252-256,
and the PNG fixtures of pkg/tests/test_imgproc.py:269-283) and by a small encoder here
that picks every scanline filter (PNG §9.2) and zlib strategy explicitly, so the inflate
sees stored, fixed and dynamic blocks and the unfilter sees all five filter types."""

from __future__ import annotations

import io
import struct
import zlib

import numpy as np
from PIL import Image

from jpeg_cases import scene


def pil_png(arr: np.ndarray, mode: str = "RGB", **kw) -> bytes:
    im = Image.fromarray(arr)
    if mode != im.mode:
        im = im.convert(mode)
    buf = io.BytesIO()
    im.save(buf, format="PNG", **kw)
    return buf.getvalue()


def _chunk(t: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + t + data + struct.pack(">I", zlib.crc32(t + data) & 0xFFFFFFFF)


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = np.abs(p - a), np.abs(p - b), np.abs(p - c)
    return np.where((pa <= pb) & (pa <= pc), a, np.where(pb <= pc, b, c))


def filter_rows(raw: np.ndarray, bpp: int, filters) -> bytes:
    """Scanlines (h, rowbytes) uint8 -> filtered stream with the given filter per row."""
    h, rb = raw.shape
    out = bytearray()
    prev = np.zeros(rb, dtype=np.int32)
    for y in range(h):
        cur = raw[y].astype(np.int32)
        ft = int(filters[y % len(filters)])
        a = np.concatenate([np.zeros(bpp, np.int32), cur[:-bpp]]) if rb > bpp else np.zeros(rb, np.int32)
        if rb <= bpp:
            a = np.zeros(rb, np.int32)
        c = np.concatenate([np.zeros(bpp, np.int32), prev[:-bpp]]) if rb > bpp else np.zeros(rb, np.int32)
        b = prev
        pred = {1: a, 2: b, 3: (a + b) >> 1, 4: _paeth(a, b, c)}.get(ft, 0)
        out.append(ft)
        out += ((cur - pred) & 255).astype(np.uint8).tobytes()
        prev = cur
    return bytes(out)


def custom_png(arr: np.ndarray, ctype: int, filters=(0, 1, 2, 3, 4), level: int = 6,
               strategy: int = zlib.Z_DEFAULT_STRATEGY, idat: int = 8192, palette=None,
               trns: bytes | None = None, pre_chunks=(), post_chunks=(), wbits: int = 15,
               mem_level: int = 8) -> bytes:
    """A PNG of colour type 0 (arr HxW), 2 (HxWx3) or 3 (HxW indices + palette)."""
    h, w = arr.shape[:2]
    bpp = 3 if ctype == 2 else 1
    raw = np.ascontiguousarray(arr, dtype=np.uint8).reshape(h, w * bpp)
    data = filter_rows(raw, bpp, filters)
    co = zlib.compressobj(level, zlib.DEFLATED, wbits, mem_level, strategy)
    z = co.compress(data) + co.flush()
    out = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, ctype, 0, 0, 0))
    for t, d in pre_chunks:
        out += _chunk(t, d)
    if palette is not None:
        out += _chunk(b"PLTE", bytes(palette))
    if trns is not None:
        out += _chunk(b"tRNS", trns)
    for i in range(0, len(z), idat):
        out += _chunk(b"IDAT", z[i: i + idat])
    for t, d in post_chunks:
        out += _chunk(t, d)
    return out + _chunk(b"IEND", b"")


def content(kind: str, w: int, h: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "noise":
        return rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    if kind == "scene":
        return scene(w, h, seed)
    if kind == "flat":
        a = np.zeros((h, w, 3), np.uint8)
        a[:, : w // 2] = (200, 30, 90)
        a[h // 3:, w // 3:] = 17
        return a
    if kind == "smooth":
        return scene(w, h, seed, noise=0.0)
    raise ValueError(kind)


def pil_cases():
    """(name, payload) pairs written by Pillow: modes L / RGB / P, sizes, compress levels."""
    out = []
    for i, (w, h) in enumerate([(1, 1), (7, 3), (64, 64), (333, 517), (640, 480)]):
        for kind in ("scene", "noise", "flat"):
            a = content(kind, w, h, 100 + i)
            out.append((f"rgb_{kind}_{w}x{h}", pil_png(a)))
            out.append((f"l_{kind}_{w}x{h}", pil_png(a, "L")))
            out.append((f"p_{kind}_{w}x{h}", pil_png(a, "P")))
    a = content("scene", 320, 200, 7)
    for lvl in (0, 1, 3, 9):
        out.append((f"rgb_scene_level{lvl}", pil_png(a, compress_level=lvl)))
    out.append(("rgb_scene_optimize", pil_png(a, optimize=True)))
    return out


def custom_cases():
    """(name, payload) pairs from custom_png: every filter, zlib strategies, IDAT splits."""
    out = []
    a = content("scene", 257, 131, 3)
    g = np.ascontiguousarray(a[..., 1])
    for f in (0, 1, 2, 3, 4):
        out.append((f"filter{f}_rgb", custom_png(a, 2, filters=(f,))))
        out.append((f"filter{f}_l", custom_png(g, 0, filters=(f,))))
    for name, st in (("filtered", zlib.Z_FILTERED), ("huffman", zlib.Z_HUFFMAN_ONLY),
                     ("rle", zlib.Z_RLE), ("fixed", zlib.Z_FIXED)):
        out.append((f"strategy_{name}", custom_png(a, 2, strategy=st)))
    out.append(("level0_stored", custom_png(a, 2, level=0)))
    out.append(("idat_1byte", custom_png(a[:9, :11], 2, idat=1)))
    out.append(("wbits9", custom_png(a, 2, wbits=9)))
    out.append(("memlevel1", custom_png(a, 2, mem_level=1)))
    pal = np.random.default_rng(5).integers(0, 256, 3 * 200, dtype=np.uint8)
    idx = np.random.default_rng(6).integers(0, 200, (97, 61), dtype=np.uint8)
    out.append(("palette", custom_png(idx, 3, palette=pal)))
    out.append(("palette_trns", custom_png(idx, 3, palette=pal, trns=bytes([0, 128, 255]))))
    out.append(("gray_trns", custom_png(g, 0, trns=b"\x00\x10")))
    out.append(("rgb_ancillary", custom_png(a, 2, pre_chunks=[(b"gAMA", struct.pack(">I", 45455)),
                                                            (b"pHYs", b"\0\0\x0b\x13\0\0\x0b\x13\x01"),
                                                            (b"tEXt", b"Comment\0hello"),
                                                            (b"prVt", b"private data")],
                                              post_chunks=[(b"prVt", b"after")])))
    big = content("noise", 1920, 1080, 11)
    out.append(("noise_1080p_mixed_filters", custom_png(big, 2)))
    return out


def bad_cases():
    """Payloads the reference rejects or decodes specially: every one must come out of
    the device path exactly as the host decoder (Pillow) gives it -- pixels or error."""
    a = content("scene", 120, 80, 9)
    good = pil_png(a)
    out = []
    # corrupt deflate data (bit flips inside the IDAT data, CRCs left as they are)
    for pos in (60, 400, len(good) // 2, len(good) - 40):
        b = bytearray(good)
        b[pos] ^= 0x55
        out.append((f"flip_{pos}", bytes(b)))
    out.append(("truncated_half", good[: len(good) // 2]))
    out.append(("truncated_tail", good[:-20]))
    b = bytearray(good)
    b[20] ^= 1  # IHDR body: CRC mismatch
    out.append(("ihdr_crc", bytes(b)))
    out.append(("rgba", pil_png(np.dstack([a, a[..., :1]]), "RGBA")))
    out.append(("la", pil_png(np.dstack([a[..., :1], a[..., :1]])[..., :2].copy(), "LA")))
    out.append(("bad_filter", custom_png(a, 2, filters=(5,))))
    pal = bytes(range(30))  # 10 entries; indices up to 50
    idx = (np.arange(40 * 30).reshape(30, 40) % 50).astype(np.uint8)
    out.append(("palette_index_oob", custom_png(idx, 3, palette=pal)))
    out.append(("short_stream", custom_png(a, 2)[:-30] + _chunk(b"IEND", b"")))
    return out


def fuzzed(n: int, seed: int = 20261019):
    """n damaged PNGs as (t, kind, payload): kind 0 flips bits after the first IDAT tag,
    1 drops 1-4 bytes there, 2 truncates the file.  Single- and multi-unit streams (the
    finder, the chain and the re-decode rounds see the damage), Pillow and custom encodes."""
    rng = np.random.default_rng(seed)
    base = [pil_png(content("scene", 96, 64, 1)), pil_png(content("noise", 80, 48, 2)),
            pil_png(content("flat", 120, 90, 3)), pil_png(content("scene", 64, 40, 4), "P"),
            custom_png(content("scene", 70, 30, 5), 2, level=0),
            custom_png(content("scene", 70, 30, 6), 2, strategy=zlib.Z_FIXED),
            pil_png(content("scene", 640, 480, 7)), pil_png(content("noise", 400, 300, 8))]
    out = []
    for t in range(n):
        p = bytearray(base[t % len(base)])
        start = p.find(b"IDAT") + 4
        kind = t % 3
        if kind == 0:
            for _ in range(1 + t % 4):
                i = int(rng.integers(start, len(p) - 16))
                p[i] ^= 1 << int(rng.integers(0, 8))
        elif kind == 1:
            i = int(rng.integers(start, len(p) - 16))
            del p[i: i + int(rng.integers(1, 5))]
        else:
            p = p[: int(rng.integers(start, len(p)))]
        out.append((t, kind, bytes(p)))
    return out
