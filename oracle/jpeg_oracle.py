"""CPU restatement of baseline JPEG decoding as the reference performs it -- TEST
INFRASTRUCTURE ONLY (imported by tests/ and the CPU legs of bench.py, never by the
product package).

The reference decodes with Pillow (vlmfp/imgproc.py:213-229, `_decode_pass`:
`Image.open(...)`, `.convert("RGB")`, `np.asarray`), i.e. with the libjpeg-turbo that
Pillow bundles (Pillow 12.2.0 / libjpeg-turbo 3.1.4.1 in this image; a third-party
dependency absent from /root/reference, `pillow>=9.0` at pkg/pyproject.toml:12).  Its
default decompression settings are the IJG defaults: JDCT_ISLOW and fancy upsampling.
This module restates that published algorithm so the device decoder (csrc/jpeg.cu) can
be checked stage by stage; parity is pinned to Pillow itself in tests/test_jpeg_oracle.py
(every case bit-exact against `np.asarray(Image.open(...).convert("RGB"))`).

  * entropy decoding: ITU-T T.81 Annex F (baseline sequential Huffman, restart markers);
    coefficients stored as int16 (libjpeg's JCOEF), DC prediction per component,
    reset at each restart marker (jdhuff.c)
  * inverse DCT: jidctint.c jpeg_idct_islow (CONST_BITS 13, PASS1_BITS 2, 64-bit JLONG
    arithmetic; the sample limit saturates as libjpeg-turbo's x86-64 SIMD IDCT does, which
    equals jdmaster.c's range-limit table wherever that table does not wrap; blocks
    outside the SIMD version's exact 16-bit range raise SimdRange)
  * upsampling: jdsample.c h2v1 / h1v2 / h2v2 fancy (triangle) filters, with the context
    rows of jdmainct.c (the row above the first row is the first row, rows below the last
    real row repeat it); plain replication when the downsampled width is <= 2
  * colour: jdcolor.c ycc_rgb_convert (SCALEBITS 16 tables), grayscale replicated to RGB
    (Pillow's L -> RGB convert)
"""

from __future__ import annotations

import numpy as np

ZIGZAG = np.array([
    0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6, 7, 14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63], dtype=np.int64)


class Unsupported(Exception):
    """A JPEG variant the device decoder does not take (progressive, arithmetic,
    12-bit, CMYK / RGB colour space, exotic sampling): decoded on the host instead."""


class Corrupt(Exception):
    pass


def parse(data: bytes) -> dict:
    """Markers up to the first SOS (T.81 B.2): frame, tables, restart interval, colour
    space hints; the entropy-coded segment runs from the end of the SOS header to EOI."""
    if data[:2] != b"\xff\xd8":
        raise Corrupt("no SOI")
    pos = 2
    info = {"qt": {}, "dc": {}, "ac": {}, "dri": 0, "jfif": False, "adobe": None}
    n = len(data)
    while pos < n:
        if data[pos] != 0xFF:
            raise Corrupt(f"expected marker at {pos}")
        while pos < n and data[pos] == 0xFF:
            pos += 1
        m = data[pos]
        pos += 1
        if m == 0xD8 or 0xD0 <= m <= 0xD7 or m == 0x01:
            continue
        if m == 0xD9:
            raise Corrupt("EOI before SOS")
        seg_len = int.from_bytes(data[pos:pos + 2], "big")
        seg = data[pos + 2: pos + seg_len]
        if m in (0xC0, 0xC1):
            prec = seg[0]
            h = int.from_bytes(seg[1:3], "big")
            w = int.from_bytes(seg[3:5], "big")
            nc = seg[5]
            comps = []
            for i in range(nc):
                cid, hv, tq = seg[6 + 3 * i: 9 + 3 * i]
                comps.append({"id": cid, "h": hv >> 4, "v": hv & 15, "tq": tq})
            if prec != 8:
                raise Unsupported(f"{prec}-bit samples")
            info.update(width=w, height=h, comps=comps)
        elif 0xC2 <= m <= 0xCF and m not in (0xC4, 0xC8, 0xCC):
            raise Unsupported(f"SOF{m - 0xC0} (not baseline Huffman)")
        elif m == 0xDB:
            p = 0
            while p < len(seg):
                pq, tq = seg[p] >> 4, seg[p] & 15
                p += 1
                if pq:
                    q = np.frombuffer(seg[p: p + 128], dtype=">u2").astype(np.int64)
                    p += 128
                else:
                    q = np.frombuffer(seg[p: p + 64], dtype=np.uint8).astype(np.int64)
                    p += 64
                nat = np.zeros(64, dtype=np.int64)
                nat[ZIGZAG] = q
                info["qt"][tq] = nat
        elif m == 0xC4:
            p = 0
            while p < len(seg):
                tc, th = seg[p] >> 4, seg[p] & 15
                bits = list(seg[p + 1: p + 17])
                cnt = sum(bits)
                vals = list(seg[p + 17: p + 17 + cnt])
                p += 17 + cnt
                (info["ac"] if tc else info["dc"])[th] = (bits, vals)
        elif m == 0xDD:
            info["dri"] = int.from_bytes(seg[0:2], "big")
        elif m == 0xE0 and seg[:5] == b"JFIF\x00":
            info["jfif"] = True
        elif m == 0xEE and seg[:5] == b"Adobe":
            info["adobe"] = seg[11] if len(seg) > 11 else None
        elif m == 0xDA:
            ns = seg[0]
            sc = []
            for i in range(ns):
                cs, t = seg[1 + 2 * i], seg[2 + 2 * i]
                sc.append((cs, t >> 4, t & 15))
            if "comps" not in info:
                raise Corrupt("SOS before SOF")
            if ns != len(info["comps"]):
                raise Unsupported("multi-scan (non-interleaved) sequential JPEG")
            ss, se, ahal = seg[1 + 2 * ns], seg[2 + 2 * ns], seg[3 + 2 * ns]
            if ss != 0 or se != 63 or ahal != 0:
                raise Unsupported("spectral selection in a baseline frame")
            for (cs, td, ta), comp in zip(sc, info["comps"]):
                if cs != comp["id"]:
                    raise Unsupported("scan component order differs from the frame")
                comp["td"], comp["ta"] = td, ta
            info["scan_start"] = pos + seg_len
            end = data.rfind(b"\xff\xd9")
            if end < info["scan_start"]:  # Pillow: "image file is truncated"
                raise Corrupt("no EOI after the scan")
            info["scan_end"] = end
            _check_supported(info)
            return info
        pos += seg_len
    raise Corrupt("no SOS")


def _check_supported(info: dict) -> None:
    comps = info["comps"]
    if len(comps) not in (1, 3):
        raise Unsupported(f"{len(comps)} components")
    if len(comps) == 1:
        if (comps[0]["h"], comps[0]["v"]) != (1, 1):
            raise Unsupported("subsampled single-component scan")
        return
    if info["adobe"] is not None and not info["jfif"] and info["adobe"] != 1:
        raise Unsupported("Adobe transform != 1 (RGB / YCCK colour space)")
    if not info["jfif"] and info["adobe"] is None and \
            [c["id"] for c in comps] == [82, 71, 66]:
        raise Unsupported("RGB colour space")
    y, cb, cr = comps
    if (cb["h"], cb["v"], cr["h"], cr["v"]) != (1, 1, 1, 1) or y["h"] not in (1, 2) or \
            y["v"] not in (1, 2):
        raise Unsupported("sampling factors other than 4:4:4 / 4:2:2 / 4:2:0 / 4:4:0")


def unstuff(data: bytes, start: int, end: int):
    """Entropy-coded bytes with stuffing removed and restart markers cut out: a list of
    segments (bytes), one per restart interval."""
    segs, cur = [], bytearray()
    i = start
    while i < end:
        b = data[i]
        if b == 0xFF:
            nxt = data[i + 1] if i + 1 < end else 0xD9
            if nxt == 0x00:
                cur.append(0xFF)
                i += 2
                continue
            if 0xD0 <= nxt <= 0xD7:
                if nxt != 0xD0 + (len(segs) & 7):  # jdmarker.c read_restart_marker resyncs
                    raise Corrupt(f"RST{nxt - 0xD0} where RST{len(segs) & 7} is due")
                segs.append(bytes(cur))
                cur = bytearray()
                i += 2
                continue
            if nxt == 0xFF:
                i += 1
                continue
            # any other marker inside the scan: libjpeg stops the scan there and conceals
            # the rest; the device decoder hands such streams to Pillow (not restated)
            raise Corrupt(f"marker FF{nxt:02X} inside the entropy-coded data")
        cur.append(b)
        i += 1
    segs.append(bytes(cur))
    return segs


def _huff_lookup(spec):
    """(code length, code) -> symbol for a DHT table (T.81 C.2, the canonical codes)."""
    bits, vals = spec
    table = {}
    code, k = 0, 0
    for length in range(1, 17):
        for _ in range(bits[length - 1]):
            table[(length, code)] = vals[k]
            k += 1
            code += 1
        code <<= 1
    return table


class _Bits:
    def __init__(self, seg: bytes):
        self.v = int.from_bytes(seg, "big") if seg else 0
        self.n = 8 * len(seg)
        self.p = 0

    def bit(self):
        if self.p >= self.n:
            raise Corrupt("entropy data ran out")
        b = (self.v >> (self.n - 1 - self.p)) & 1
        self.p += 1
        return b

    def bits(self, k):
        r = 0
        for _ in range(k):
            r = (r << 1) | self.bit()
        return r


def _decode_sym(br: _Bits, table) -> int:
    code = 0
    for length in range(1, 17):
        code = (code << 1) | br.bit()
        s = table.get((length, code))
        if s is not None:
            return s
    raise Corrupt("bad Huffman code")


def _extend(v: int, s: int) -> int:
    return v - (1 << s) + 1 if s and v < (1 << (s - 1)) else v


def mcu_layout(info: dict):
    comps = info["comps"]
    w, h = info["width"], info["height"]
    hmax = max(c["h"] for c in comps)
    vmax = max(c["v"] for c in comps)
    if len(comps) == 1:
        mcux, mcuy = -(-w // 8), -(-h // 8)
        slots = [(0, 0, 0)]
    else:
        mcux, mcuy = -(-w // (8 * hmax)), -(-h // (8 * vmax))
        slots = [(ci, bv, bh) for ci, c in enumerate(comps)
                 for bv in range(c["v"]) for bh in range(c["h"])]
    return mcux, mcuy, hmax, vmax, slots


def decode_coefficients(data: bytes, info: dict):
    """Per component, a [by, bx, 64] int16 array of dequantization-ready coefficients in
    natural order (DC already predicted), as libjpeg's coefficient buffer holds them."""
    comps = info["comps"]
    mcux, mcuy, hmax, vmax, slots = mcu_layout(info)
    planes = []
    for c in comps:
        bw = mcux * (c["h"] if len(comps) > 1 else 1)
        bh = mcuy * (c["v"] if len(comps) > 1 else 1)
        planes.append(np.zeros((bh, bw, 64), dtype=np.int16))
    dct = {k: _huff_lookup(v) for k, v in info["dc"].items()}
    act = {k: _huff_lookup(v) for k, v in info["ac"].items()}
    segs = unstuff(data, info["scan_start"], info["scan_end"])
    ri = info["dri"] or mcux * mcuy
    n_mcu = mcux * mcuy
    if len(segs) != -(-n_mcu // ri):  # restart markers missing or extra: concealed by libjpeg
        raise Corrupt(f"{len(segs)} restart intervals, {-(-n_mcu // ri)} expected")
    for s_idx, seg in enumerate(segs):
        first = s_idx * ri
        if first >= n_mcu:
            break
        br = _Bits(seg)
        pred = [0] * len(comps)
        for m in range(first, min(n_mcu, first + ri)):
            my, mx = divmod(m, mcux)
            for ci, bv, bh in slots:
                c = comps[ci]
                blk = np.zeros(64, dtype=np.int64)
                t = _decode_sym(br, dct[c["td"]])
                diff = _extend(br.bits(t), t) if t else 0
                pred[ci] += diff
                blk[0] = pred[ci]
                k = 1
                while k < 64:
                    rs = _decode_sym(br, act[c["ta"]])
                    r, s = rs >> 4, rs & 15
                    if s:
                        k += r
                        if k > 63:  # libjpeg writes it to coefficient 63 and goes on
                            raise Corrupt("AC run past coefficient 63")
                        blk[ZIGZAG[k]] = _extend(br.bits(s), s)
                        k += 1
                    elif r == 15:
                        k += 16
                    else:
                        break
                if len(comps) == 1:
                    planes[ci][my, mx] = blk.astype(np.int16)
                else:
                    planes[ci][my * c["v"] + bv, mx * c["h"] + bh] = blk.astype(np.int16)
    return planes


# jidctint.c constants (CONST_BITS = 13)
_F = {"0_298631336": 2446, "0_390180644": 3196, "0_541196100": 4433, "0_765366865": 6270,
      "0_899976223": 7373, "1_175875602": 9633, "1_501321110": 12299, "1_847759065": 15137,
      "1_961570560": 16069, "2_053119869": 16819, "2_562915447": 20995, "3_072711026": 25172}
CONST_BITS, PASS1_BITS = 13, 2


def _descale(x, n):
    return (x + (1 << (n - 1))) >> n


def _idct_1d(d0, d1, d2, d3, d4, d5, d6, d7, shift0):
    """One jidctint.c butterfly over int64 arrays; returns the 8 outputs before the final
    descale (even/odd parts as in the source)."""
    z2, z3 = d2, d6
    z1 = (z2 + z3) * _F["0_541196100"]
    tmp2 = z1 + z3 * -_F["1_847759065"]
    tmp3 = z1 + z2 * _F["0_765366865"]
    tmp0 = (d0 + d4) << CONST_BITS
    tmp1 = (d0 - d4) << CONST_BITS
    tmp10, tmp13, tmp11, tmp12 = tmp0 + tmp3, tmp0 - tmp3, tmp1 + tmp2, tmp1 - tmp2
    t0, t1, t2, t3 = d7, d5, d3, d1
    z1, z2, z3, z4 = t0 + t3, t1 + t2, t0 + t2, t1 + t3
    z5 = (z3 + z4) * _F["1_175875602"]
    t0 = t0 * _F["0_298631336"]
    t1 = t1 * _F["2_053119869"]
    t2 = t2 * _F["3_072711026"]
    t3 = t3 * _F["1_501321110"]
    z1 = z1 * -_F["0_899976223"]
    z2 = z2 * -_F["2_562915447"]
    z3 = z3 * -_F["1_961570560"] + z5
    z4 = z4 * -_F["0_390180644"] + z5
    t0 = t0 + z1 + z3
    t1 = t1 + z2 + z4
    t2 = t2 + z2 + z3
    t3 = t3 + z1 + z4
    return (tmp10 + t3, tmp11 + t2, tmp12 + t1, tmp13 + t0,
            tmp13 - t0, tmp12 - t1, tmp11 - t2, tmp10 - t3)


SIMD_BOUND = 1 << 13  # |dequantized coefficient|, |workspace value| below this: see idct_islow


def range_limit(x: np.ndarray) -> np.ndarray:
    """The sample limit after the IDCT, as Pillow's libjpeg-turbo applies it on x86-64.
    jdmaster.c's table (sample_range_limit[CENTERJSAMPLE + (x & RANGE_MASK)]) clamps x + 128
    to [0, 255] for x in [-512, 511] and wraps beyond; the SIMD ISLOW IDCT that
    jsimd_idct_islow selects (simd/x86_64/jidctint-{sse2,avx2}.asm: packssdw, packsswb,
    + CENTERJSAMPLE) saturates instead.  Inside [-512, 511] the two agree; outside, the
    SIMD saturation is what Pillow returns (pinned by tests/test_jpeg_oracle.py)."""
    return np.clip(x + 128, 0, 255)


class SimdRange(Unsupported):
    """A block whose IDCT leaves the range where libjpeg-turbo's 16-bit SIMD ISLOW IDCT
    equals jidctint.c (only damaged streams get there): decoded by Pillow instead."""


def idct_islow(coefs: np.ndarray, quant: np.ndarray) -> np.ndarray:
    """[..., 64] int16 natural-order coefficients -> [..., 8, 8] uint8 samples.

    The arithmetic is jidctint.c's (64-bit JLONG).  libjpeg-turbo's SIMD version keeps the
    dequantized coefficients and the pass-1 workspace in 16-bit lanes (pmullw, paddw of
    coefficient pairs, packssdw), so it equals jidctint.c only while every dequantized
    coefficient and every workspace value is below 2^13 in magnitude (then no 16-bit sum
    or DC shortcut overflows); beyond that SimdRange is raised."""
    c = (coefs.astype(np.int64) * quant.astype(np.int16).astype(np.int64)).reshape(-1, 8, 8)
    if c.size and np.abs(c).max() >= SIMD_BOUND:
        raise SimdRange("dequantized coefficient outside the SIMD IDCT's exact range")
    # pass 1: columns (index [row, col]; column inputs are rows 0..7)
    cols = _idct_1d(*(c[:, k, :] for k in range(8)), None)
    ws = np.stack([_descale(v, CONST_BITS - PASS1_BITS) for v in cols], axis=1)
    if ws.size and np.abs(ws).max() >= SIMD_BOUND:
        raise SimdRange("IDCT workspace value outside the SIMD IDCT's exact range")
    # (the all-zero-AC column / row shortcuts give the same values as the full butterfly)
    rows = _idct_1d(*(ws[:, :, k] for k in range(8)), None)
    out = np.stack([range_limit(_descale(v, CONST_BITS + PASS1_BITS + 3)) for v in rows],
                   axis=2)
    return out.astype(np.uint8).reshape(coefs.shape[:-1] + (8, 8))


def component_planes(info: dict, planes):
    """IDCT of every block into full component planes (block-padded), uint8."""
    out = []
    for ci, p in enumerate(planes):
        q = info["qt"][info["comps"][ci]["tq"]]
        px = idct_islow(p, q)  # [bh, bw, 8, 8]
        bh, bw = p.shape[:2]
        out.append(px.transpose(0, 2, 1, 3).reshape(bh * 8, bw * 8))
    return out


def _fancy_h2(row: np.ndarray) -> np.ndarray:
    """jdsample.c h2v1_fancy_upsample on one row (int64 in, int64 out of 2n)."""
    n = len(row)
    out = np.empty(2 * n, dtype=np.int64)
    out[0] = row[0]
    out[1] = (row[0] * 3 + row[1] + 2) >> 2
    mid = row[1:n - 1] * 3
    out[2:2 * n - 2:2] = (mid + row[0:n - 2] + 1) >> 2
    out[3:2 * n - 2:2] = (mid + row[2:n] + 2) >> 2
    out[2 * n - 2] = (row[n - 1] * 3 + row[n - 2] + 1) >> 2
    out[2 * n - 1] = row[n - 1]
    return out


def upsample(plane: np.ndarray, ds_w: int, ds_h: int, hx: int, vx: int, out_w: int,
             out_h: int) -> np.ndarray:
    """The jdsample.c method libjpeg picks for expansion (hx, vx), on the real
    downsampled samples (ds_w x ds_h; context rows replicate the edge rows)."""
    p = plane[:ds_h, :ds_w].astype(np.int64)
    if hx == 1 and vx == 1:
        r = p
    elif ds_w <= 2 and hx == 2:  # fancy needs > 2 columns: plain replication
        r = np.repeat(np.repeat(p, hx, axis=1), vx, axis=0)
    elif hx == 2 and vx == 1:
        r = np.stack([_fancy_h2(row) for row in p])
    elif hx == 1 and vx == 2:
        above = np.vstack([p[:1], p[:-1]])
        below = np.vstack([p[1:], p[-1:]])
        r = np.empty((2 * ds_h, ds_w), dtype=np.int64)
        r[0::2] = (p * 3 + above + 1) >> 2
        r[1::2] = (p * 3 + below + 2) >> 2
    else:  # h2v2
        above = np.vstack([p[:1], p[:-1]])
        below = np.vstack([p[1:], p[-1:]])
        r = np.empty((2 * ds_h, 2 * ds_w), dtype=np.int64)
        for dst, other in ((0, above), (1, below)):
            cs = p * 3 + other  # column sums
            o = np.empty((ds_h, 2 * ds_w), dtype=np.int64)
            o[:, 0] = (cs[:, 0] * 4 + 8) >> 4
            o[:, 1] = (cs[:, 0] * 3 + cs[:, 1] + 7) >> 4
            o[:, 2:2 * ds_w - 2:2] = (cs[:, 1:-1] * 3 + cs[:, :-2] + 8) >> 4
            o[:, 3:2 * ds_w - 2:2] = (cs[:, 1:-1] * 3 + cs[:, 2:] + 7) >> 4
            o[:, 2 * ds_w - 2] = (cs[:, -1] * 3 + cs[:, -2] + 8) >> 4
            o[:, 2 * ds_w - 1] = (cs[:, -1] * 4 + 7) >> 4
            r[dst::2] = o
    return r[:out_h, :out_w]


def _fix(x: float) -> int:
    return int(x * 65536 + 0.5)


def ycc_to_rgb(y, cb, cr) -> np.ndarray:
    """jdcolor.c ycc_rgb_convert: SCALEBITS 16 integer tables, range-limited."""
    x_cb, x_cr = cb.astype(np.int64) - 128, cr.astype(np.int64) - 128
    half = 1 << 15
    cr_r = (_fix(1.40200) * x_cr + half) >> 16
    cb_b = (_fix(1.77200) * x_cb + half) >> 16
    cr_g = -_fix(0.71414) * x_cr
    cb_g = -_fix(0.34414) * x_cb + half
    y = y.astype(np.int64)
    r = np.clip(y + cr_r, 0, 255)
    g = np.clip(y + ((cb_g + cr_g) >> 16), 0, 255)
    b = np.clip(y + cb_b, 0, 255)
    return np.stack([r, g, b], axis=-1).astype(np.uint8)


def decode(data: bytes) -> np.ndarray:
    """Baseline JPEG -> (H, W, 3) uint8, as Pillow's decode + convert("RGB")."""
    info = parse(data)
    planes = component_planes(info, decode_coefficients(data, info))
    w, h = info["width"], info["height"]
    comps = info["comps"]
    if len(comps) == 1:
        g = planes[0][:h, :w]
        return np.repeat(g[:, :, None], 3, axis=2)
    hmax = max(c["h"] for c in comps)
    vmax = max(c["v"] for c in comps)
    full = []
    for c, p in zip(comps, planes):
        ds_w = -(-w * c["h"] // hmax)
        ds_h = -(-h * c["v"] // vmax)
        full.append(upsample(p, ds_w, ds_h, hmax // c["h"], vmax // c["v"], w, h))
    return ycc_to_rgb(*full)
