"""The JPEG oracle (oracle/jpeg_oracle.py, a restatement of libjpeg-turbo's baseline
decode) pinned to Pillow -- the reference's decoder (imgproc.py:213-229) -- and the
library's host-side marker parser (tp_jpeg_parse) checked against the oracle's."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from jpeg_cases import corpus_files, encode, fuzzed, pil_rgb, scene, small_cases
from oracle import jpeg_oracle as J
from paper_2603_16987_b200 import jpeg as PJ


@pytest.mark.parametrize("name,data", small_cases(0) + corpus_files()[:6])
def test_oracle_matches_pillow(name, data):
    assert np.array_equal(J.decode(data), pil_rgb(data)), name


def test_oracle_on_damaged_streams():
    """Damaged streams (bit flips, dropped bytes, truncation): the oracle either decodes
    them exactly as Pillow does -- including the saturating sample limit of libjpeg-turbo's
    SIMD IDCT for out-of-range blocks -- or raises Corrupt / Unsupported (the cases the
    device decoder hands to Pillow: bad codes, runs past 63, early data end, stray or
    misnumbered markers, blocks outside the SIMD IDCT's exact range)."""
    from paper_2603_16987_b200._decode import decode_rgb

    decoded = 0
    for t, kind, p in fuzzed(300):
        try:
            got = J.decode(p)
        except (J.Corrupt, J.Unsupported):
            continue
        decoded += 1
        assert np.array_equal(got, decode_rgb(p)), (t, kind)
    assert decoded > 100


def test_oracle_rejects_progressive():
    data = encode(scene(40, 30, 1), progressive=True)
    with pytest.raises(J.Unsupported):
        J.parse(data)


@pytest.mark.parametrize("name,data", small_cases(1) + corpus_files())
def test_host_parse_matches_oracle(name, data):
    info = PJ.parse(data)
    assert info.status == PJ.TP_JPEG_OK, info.message
    o = J.parse(data)
    assert (info.width, info.height, info.ncomp) == (o["width"], o["height"], len(o["comps"]))
    assert info.restart_interval == o["dri"]
    assert info.scan_off == o["scan_start"] and info.scan_off + info.scan_len == o["scan_end"]
    for c, comp in enumerate(o["comps"]):
        assert (info.comp_h[c], info.comp_v[c], info.comp_tq[c]) == (comp["h"], comp["v"], comp["tq"])
        assert (info.comp_td[c], info.comp_ta[c]) == (comp["td"], comp["ta"])
        assert list(info.qt[comp["tq"]]) == o["qt"][comp["tq"]].tolist()


def test_host_parse_statuses():
    px = scene(48, 40, 3)
    assert PJ.parse(encode(px, progressive=True)).status == PJ.TP_JPEG_UNSUPPORTED
    assert PJ.parse(b"\x89PNG\r\n\x1a\n....").status == PJ.TP_JPEG_UNSUPPORTED
    good = encode(px)
    assert PJ.parse(good[:200]).status == PJ.TP_JPEG_CORRUPT  # no SOS / truncated headers
    assert PJ.parse(good[: len(good) - 2]).status == PJ.TP_JPEG_CORRUPT  # no EOI


def test_describe_layout_host_only():
    """tp_jpeg_describe (host): monotone bases, workspace bounds, skipped images."""
    datas = [encode(scene(64, 48, 1)), encode(scene(40, 30, 2), progressive=True),
             encode(scene(100, 75, 3), restart_marker_blocks=2)]
    n = len(datas)
    infos = (PJ.TpJpegInfo * n)()
    for k, d in enumerate(datas):
        PJ.parse(d, infos[k])
    raw_off = np.array([0, 0, 4096], dtype=np.int64)
    out_off = np.array([0, 64 * 48 * 3, 64 * 48 * 3 + 40 * 30 * 3], dtype=np.int64)
    lib = PJ._lib.load()
    desc = (ctypes.c_uint8 * (n * int(lib.tp_jpeg_desc_bytes())))()
    totals = np.zeros(8, dtype=np.int64)
    w = lib.tp_jpeg_describe(ctypes.byref(infos), n, raw_off.ctypes.data, out_off.ctypes.data,
                             2048, ctypes.cast(desc, ctypes.c_void_p), totals.ctypes.data)
    assert w > totals[4] >= totals[3] >= 4096
    mcu = [(64 // 16) * (48 // 16) * 6, 0, 7 * 5 * 6]  # 4:2:0 MCUs x 6 blocks
    assert totals[1] == sum(mcu) and totals[2] == 48 + 75
    assert lib.tp_jpeg_describe(ctypes.byref(infos), n, raw_off.ctypes.data, out_off.ctypes.data,
                                100, ctypes.cast(desc, ctypes.c_void_p), totals.ctypes.data) < 0
