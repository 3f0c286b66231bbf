"""CPU restatement of the PNG decode the reference reaches through Pillow (test
infrastructure only: imported by tests/, never by the product path).

The reference decodes payloads with ``Image.open(...).convert("RGB")``
(/root/reference/pkg/src/vlmfp/imgproc.py:213-229; accepted modes L, P, RGB at
imgproc.py:26).  For PNG that is Pillow's PngImagePlugin (chunk walk, Pillow 12.2 in this
image, not in /root/reference; ``pillow>=9.0`` at pkg/pyproject.toml:12) over zlib's
inflate.  This module restates the pieces from their specifications:

* ``inflate``      RFC 1950 (zlib header, Adler-32) + RFC 1951 (stored, fixed and dynamic
                   Huffman blocks, LZ77 back references), canonical codes as in
                   RFC 1951 §3.2.2;
* ``unfilter``     PNG specification §9 (filter types 0-4, Paeth predictor §9.4);
* ``decode_rgb``   8-bit L / RGB / P, non-interlaced: IHDR, PLTE, the IDAT run, then
                   Pillow's convert("RGB") (L replicated, P through the palette).

It is pinned to Pillow by tests/test_png_oracle.py (bit-exact on every case there) and is
meant for small inputs: the inflate is a pure-Python loop.
"""

from __future__ import annotations

import struct

import numpy as np

_CL_ORDER = (16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15)
_LEN_BASE = (3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31, 35, 43, 51, 59, 67, 83,
             99, 115, 131, 163, 195, 227, 258)
_LEN_EXTRA = (0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5,
              5, 0)
_DIST_BASE = (1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193, 257, 385, 513, 769,
              1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577)
_DIST_EXTRA = (0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11,
               11, 12, 12, 13, 13)


class InflateError(ValueError):
    pass


class _Bits:
    """LSB-first bit reader (RFC 1951 §3.1.1)."""

    def __init__(self, data: bytes, pos: int = 0):
        self.data, self.pos = data, pos * 8

    def bits(self, n: int) -> int:
        v = 0
        for i in range(n):
            byte = self.pos >> 3
            if byte >= len(self.data):
                raise InflateError("stream ends early")
            v |= ((self.data[byte] >> (self.pos & 7)) & 1) << i
            self.pos += 1
        return v

    def align(self) -> None:
        self.pos = (self.pos + 7) & ~7


def _huffman(lengths):
    """Canonical code (RFC 1951 §3.2.2) as {(length, code): symbol}."""
    maxl = max(lengths, default=0)
    count = [0] * (maxl + 2)
    for l in lengths:
        if l:
            count[l] += 1
    code, nxt = 0, [0] * (maxl + 2)
    for l in range(1, maxl + 1):
        code = (code + count[l - 1]) << 1
        nxt[l] = code
    table = {}
    for sym, l in enumerate(lengths):
        if l:
            table[(l, nxt[l])] = sym
            nxt[l] += 1
    return table, maxl


def _decode_sym(br: _Bits, table, maxl) -> int:
    code = 0
    for l in range(1, maxl + 1):
        code = (code << 1) | br.bits(1)  # Huffman codes are packed MSB first
        sym = table.get((l, code))
        if sym is not None:
            return sym
    raise InflateError("invalid code")


def inflate(z: bytes) -> bytes:
    """zlib stream -> bytes (RFC 1950 / 1951).  The Adler-32 trailer is checked when the
    stream holds it (Pillow's zlib raises on a wrong one, and says nothing when the
    stream ends before it)."""
    if len(z) < 2 or (z[0] & 15) != 8 or ((z[0] << 8) | z[1]) % 31 or (z[1] & 0x20):
        raise InflateError("bad zlib header")
    br, out = _Bits(z, 2), bytearray()
    fixed_lit = _huffman([8] * 144 + [9] * 112 + [7] * 24 + [8] * 8)
    fixed_dist = _huffman([5] * 30)
    while True:
        final, btype = br.bits(1), br.bits(2)
        if btype == 0:
            br.align()
            n, nn = br.bits(16), br.bits(16)
            if n ^ nn != 0xFFFF:
                raise InflateError("stored block length")
            start = br.pos >> 3
            if start + n > len(z):
                raise InflateError("stream ends early")
            out += z[start: start + n]
            br.pos += 8 * n
        elif btype in (1, 2):
            if btype == 1:
                lit, dist = fixed_lit, fixed_dist
            else:
                hlit, hdist, hclen = br.bits(5) + 257, br.bits(5) + 1, br.bits(4) + 4
                cl = [0] * 19
                for i in range(hclen):
                    cl[_CL_ORDER[i]] = br.bits(3)
                pre = _huffman(cl)
                lens = []
                while len(lens) < hlit + hdist:
                    sym = _decode_sym(br, *pre)
                    if sym < 16:
                        lens.append(sym)
                    elif sym == 16:
                        if not lens:
                            raise InflateError("repeat with no previous length")
                        lens += [lens[-1]] * (3 + br.bits(2))
                    elif sym == 17:
                        lens += [0] * (3 + br.bits(3))
                    else:
                        lens += [0] * (11 + br.bits(7))
                if len(lens) > hlit + hdist:
                    raise InflateError("too many lengths")
                lit, dist = _huffman(lens[:hlit]), _huffman(lens[hlit:])
            while True:
                sym = _decode_sym(br, *lit)
                if sym < 256:
                    out.append(sym)
                elif sym == 256:
                    break
                else:
                    i = sym - 257
                    if i >= 29:
                        raise InflateError("invalid length symbol")
                    n = _LEN_BASE[i] + br.bits(_LEN_EXTRA[i])
                    d = _decode_sym(br, *dist)
                    if d >= 30:
                        raise InflateError("invalid distance symbol")
                    dd = _DIST_BASE[d] + br.bits(_DIST_EXTRA[d])
                    if dd > len(out):
                        raise InflateError("distance too far back")
                    for _ in range(n):  # byte by byte: overlapping copies repeat
                        out.append(out[-dd])
        else:
            raise InflateError("invalid block type")
        if final:
            break
    at = (br.pos + 7) >> 3
    if at + 4 <= len(z):
        a, b = 1, 0
        for v in out:
            a = (a + v) % 65521
            b = (b + a) % 65521
        if struct.unpack(">I", z[at: at + 4])[0] != (b << 16) | a:
            raise InflateError("incorrect data check")
    return bytes(out)


def unfilter(raw: bytes, width: int, height: int, bpp: int) -> np.ndarray:
    """Filtered scanlines -> (height, width * bpp) uint8 (PNG §9)."""
    rb = width * bpp
    a = np.frombuffer(raw, dtype=np.uint8)[: height * (rb + 1)].reshape(height, rb + 1)
    out = np.zeros((height, rb), dtype=np.uint8)
    prior = np.zeros(rb, dtype=np.int32)
    for y in range(height):
        ft, f = int(a[y, 0]), a[y, 1:].astype(np.int32)
        cur = np.zeros(rb, dtype=np.int32)
        if ft in (0, 2):
            cur = (f + (prior if ft == 2 else 0)) & 255
        elif ft in (1, 3, 4):
            for x in range(rb):  # left neighbour dependency: serial along the row
                left = cur[x - bpp] if x >= bpp else 0
                up = prior[x]
                ul = prior[x - bpp] if x >= bpp else 0
                if ft == 1:
                    pred = left
                elif ft == 3:
                    pred = (left + up) >> 1
                else:  # Paeth (§9.4)
                    p = left + up - ul
                    pa, pb, pc = abs(p - left), abs(p - up), abs(p - ul)
                    pred = left if pa <= pb and pa <= pc else (up if pb <= pc else ul)
                cur[x] = (f[x] + pred) & 255
        else:
            raise ValueError(f"unknown filter type {ft}")
        out[y] = cur
        prior = cur
    return out


def decode_rgb(payload: bytes) -> np.ndarray:
    """8-bit L / RGB / P PNG -> (H, W, 3) uint8, as Pillow's convert("RGB") gives it."""
    if payload[:8] != b"\x89PNG\r\n\x1a\n":
        raise ValueError("not a PNG")
    pos, idat, pal, ihdr = 8, bytearray(), None, None
    seen_idat = False
    while pos + 8 <= len(payload):
        n = struct.unpack(">I", payload[pos: pos + 4])[0]
        t, body = payload[pos + 4: pos + 8], payload[pos + 8: pos + 8 + n]
        if t == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body[:13])
        elif t == b"PLTE":
            pal = np.frombuffer(body, dtype=np.uint8).reshape(-1, 3)
        elif t == b"IDAT":
            idat += body
            seen_idat = True
        elif seen_idat or t == b"IEND":
            break  # Pillow reads image data up to the first non-IDAT chunk
        pos += 12 + n
    w, h, depth, ctype, _, _, interlace = ihdr
    if depth != 8 or interlace or ctype not in (0, 2, 3):
        raise ValueError("outside the restated subset")
    bpp = 3 if ctype == 2 else 1
    raw = inflate(bytes(idat))
    if len(raw) < h * (w * bpp + 1):
        raise ValueError("image file is truncated")
    px = unfilter(raw, w, h, bpp)
    if ctype == 2:
        return px.reshape(h, w, 3)
    if ctype == 0:
        return np.repeat(px.reshape(h, w, 1), 3, axis=2)
    full = np.zeros((256, 3), dtype=np.uint8)
    full[: len(pal)] = pal
    return full[px.reshape(h, w)]
