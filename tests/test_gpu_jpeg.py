"""K7 device JPEG decode vs Pillow (the reference's decoder, imgproc.py:213-229):
bit-exact RGB on the reference corpus files, on Pillow-encoded variants (odd sizes,
4:4:4 / 4:2:2 / 4:2:0, qualities, restart markers, grayscale, noise), on 1080p
corpus-like images, and in mixed batches where unsupported payloads (progressive JPEG,
PNG) and corrupt streams go to the host decoder; then decode -> K1/K2 against the oracle."""

from __future__ import annotations

import io

import numpy as np
import pytest
import torch
from PIL import Image

from jpeg_cases import corpus_files, encode, fuzzed, pil_rgb, scene, small_cases
from paper_2603_16987_b200.jpeg import JpegDecoder, decode_images

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _check(payloads, names=None, dec=None, expect_device=None):
    dec = dec or JpegDecoder(DEV)
    pk = dec.decode(payloads)
    host = pk.data.cpu().numpy()
    for k, p in enumerate(payloads):
        w, h = (int(v) for v in pk.wh_host[k])
        o = int(pk.offsets_host[k])
        got = host[o: o + w * h * 3].reshape(h, w, 3)
        want = pil_rgb(p)
        if not np.array_equal(got, want):
            d = np.argwhere(got != want)
            raise AssertionError(f"{names[k] if names else k}: {len(d)} bytes differ, first {d[:3].tolist()}")
    if expect_device is not None:
        assert [k for k in range(len(payloads)) if k not in dec.last_fallback] == expect_device
    return dec


def test_small_cases_one_batch():
    cases = small_cases(3)
    dec = _check([d for _, d in cases], [n for n, _ in cases])
    assert dec.last_fallback == []  # every one of them decoded on the device


def test_reference_corpus_files():
    cases = corpus_files()
    dec = _check([d for _, d in cases], [n for n, _ in cases])
    assert dec.last_fallback == []


@pytest.mark.parametrize("kw", [{}, {"subsampling": 0}, {"subsampling": 1},
                                {"restart_marker_blocks": 7}, {"gray": True},
                                {"quality": 97}, {"quality": 30}])
def test_1080p_variants(kw):
    px = scene(1920, 1080, 11)
    _check([encode(px, **kw)], expect_device=[0])


@pytest.mark.parametrize("ss", [0, 1, 2])
def test_wide_rows(ss):
    # rows wider than one CTA pass (2048 pixels): 16-byte aligned (staged stores), 4-byte
    # aligned and unaligned rows, each with a partial last warp; plus one gray
    payloads = [encode(scene(w, h, w + ss), 85, subsampling=ss)
                for (w, h) in [(2304, 24), (2600, 18), (4097, 9), (2050, 33)]]
    payloads.append(encode(scene(2333, 12, 1), 90, gray=True))
    _check(payloads, expect_device=[0, 1, 2, 3, 4])


@pytest.mark.parametrize("sub_bits", [256, 1024, 2048, 8192])
def test_noise_and_sub_bits(sub_bits):
    rng = np.random.default_rng(sub_bits)
    payloads = [encode(rng.integers(0, 256, (h, w, 3), dtype=np.uint8), q)
                for (w, h, q) in [(640, 480, 85), (333, 517, 95), (1023, 77, 60)]]
    payloads.append(encode(scene(800, 600, 5)))
    _check(payloads, dec=JpegDecoder(DEV, sub_bits=sub_bits), expect_device=[0, 1, 2, 3])


def test_mixed_batch_host_fallbacks():
    px = scene(200, 150, 4)
    png = io.BytesIO()
    Image.fromarray(px).save(png, format="PNG")
    good = encode(px)
    # a corrupt scan: bytes flipped in the middle of the entropy data (Pillow still decodes
    # it, with its own concealment): the device flags it and the host decoder takes over
    bad = bytearray(good)
    mid = len(bad) // 2
    bad[mid: mid + 8] = b"\xff\xd3\x12\x34\x56\x78\x9a\xbc"
    payloads = [good, encode(px, progressive=True), png.getvalue(), bytes(bad), encode(px, 90)]
    try:
        pil_rgb(bytes(bad))
    except Exception:
        payloads.pop(3)
    dec = _check(payloads)
    assert 1 in dec.last_fallback and 2 in dec.last_fallback and 0 not in dec.last_fallback


def test_decode_then_tile_matches_oracle():
    from oracle import tileprep_oracle as O
    from paper_2603_16987_b200.engine import TilePreprocessor
    from paper_2603_16987_b200.imgproc import PreprocessConfig
    from paper_2603_16987_b200.workloads import IMAGENET_MEAN, IMAGENET_STD

    payloads = [d for _, d in corpus_files()[:6]] + [encode(scene(1920, 1080, 2))]
    pk = JpegDecoder(DEV).decode(payloads)
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    out = TilePreprocessor(cfg, DEV)(pk)
    torch.cuda.synchronize()
    off = out.plans.tile_off.cpu().numpy()
    for k, p in enumerate(payloads):
        a = pil_rgb(p)
        plan = O.plan_float(a.shape[1], a.shape[0], 448, 12)
        want = O.normalize(O.tiles_u8(a, plan), IMAGENET_MEAN, IMAGENET_STD, True).transpose(0, 3, 1, 2)
        got = out.pixel_values[off[k]: off[k + 1]].cpu().view(torch.int16).numpy()
        assert np.array_equal(got.view(np.uint16), want.view(np.uint16)), k


def test_decode_images_helper():
    p = encode(scene(50, 40, 9))
    assert np.array_equal(decode_images([p], DEV)[0], pil_rgb(p))


def test_fuzzed_jpegs_match_pillow():
    """Random damage to baseline JPEGs (bit flips and dropped bytes in the entropy-coded
    data, with and without restart markers, truncation): every payload decodes exactly as
    Pillow decodes it -- the same pixels (libjpeg conceals damage; a stream K7 does not find
    clean goes to Pillow on the host) or the same exception -- and nothing faults."""
    from paper_2603_16987_b200._decode import decode_rgb

    dec = JpegDecoder(DEV)
    good = []
    for t, kind, p in fuzzed(240):
        try:
            ref, ref_exc = decode_rgb(p), None
        except Exception as exc:  # noqa: BLE001 -- whatever the reference raises
            ref, ref_exc = None, exc
        try:
            pk = dec.decode([p])
            w, h = (int(v) for v in pk.wh_host[0])
            got, got_exc = pk.data[: w * h * 3].cpu().numpy().reshape(h, w, 3), None
        except Exception as exc:  # noqa: BLE001
            got, got_exc = None, exc
        if ref_exc is not None:
            assert got_exc is not None and type(got_exc) is type(ref_exc), (t, kind, ref_exc, got_exc)
        else:
            assert got_exc is None, (t, kind, got_exc)
            assert np.array_equal(got, ref), (t, kind, dec.last_fallback)
            good.append((p, ref))
    # the decodable ones again as one batch: damage in one image does not leak into another
    pk = dec.decode([p for p, _ in good])
    host = pk.data.cpu().numpy()
    for k, ((p, ref), o, (w, h)) in enumerate(zip(good, pk.offsets_host, pk.wh_host)):
        got = host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
        assert np.array_equal(got, ref), k
