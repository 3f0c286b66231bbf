"""K8 device PNG decode against Pillow (the reference's decoder, imgproc.py:213-229):
identical pixels for every payload the device takes, and for every other payload the
reference's own result (pixels, or the DecodeError / UnsupportedFormatError)."""

import re

import numpy as np
import pytest

from png_cases import bad_cases, custom_cases, pil_cases

pytestmark = pytest.mark.gpu


def _host(payload):
    from paper_2603_16987_b200._decode import decode_rgb

    return decode_rgb(payload)


def _device(payloads):
    import torch

    from paper_2603_16987_b200.png import PngDecoder

    dec = PngDecoder(torch.device("cuda:0"))
    pk = dec.decode(payloads)
    host = pk.data.cpu().numpy()
    imgs = [host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            for o, (w, h) in zip(pk.offsets_host, pk.wh_host)]
    return imgs, dec


def _check(cases, allow_fallback=()):
    names = [c[0] for c in cases]
    imgs, dec = _device([c[1] for c in cases])
    st = dec.last_status()
    bad = []
    for (name, payload), img, s in zip(cases, imgs, st):
        ref = _host(payload)
        if not np.array_equal(img, ref):
            bad.append((name, "pixels"))
        if s != 0 and name not in allow_fallback:
            bad.append((name, f"status {s}"))
    assert not bad, bad
    return names


def test_png_pillow_payloads():
    _check(pil_cases())


def test_png_custom_payloads():
    _check(custom_cases())


def test_png_one_image_batches():
    for name, payload in pil_cases()[:6] + custom_cases()[:3]:
        imgs, dec = _device([payload])
        assert np.array_equal(imgs[0], _host(payload)), name


def test_png_bad_payloads_match_reference():
    from paper_2603_16987_b200.png import PngDecoder
    import torch

    dec = PngDecoder(torch.device("cuda:0"))
    for name, payload in bad_cases():
        try:
            ref = _host(payload)
            ref_exc = None
        except Exception as exc:  # noqa: BLE001 -- compare whatever the reference raises
            ref, ref_exc = None, exc
        try:
            pk = dec.decode([payload])
            got = pk.data[: int(pk.wh_host[0][0]) * int(pk.wh_host[0][1]) * 3].cpu().numpy()
            got_exc = None
        except Exception as exc:  # noqa: BLE001
            got, got_exc = None, exc
        if ref_exc is not None:
            assert got_exc is not None and type(got_exc) is type(ref_exc), name
            # Pillow's message may name the BytesIO object (its address differs per call)
            addr = re.compile(r"0x[0-9a-f]+")
            assert addr.sub("0x", str(got_exc)) == addr.sub("0x", str(ref_exc)), name
            assert getattr(got_exc, "byte_offset", None) == getattr(ref_exc, "byte_offset", None)
        else:
            assert got_exc is None, (name, got_exc)
            assert np.array_equal(got, ref.reshape(-1)), name


def test_png_chunked_batches():
    """A workspace cap smaller than the batch: sub-batches decoded in turn into one output
    (with a host-decoded payload in the middle)."""
    import torch

    from paper_2603_16987_b200.png import PngDecoder
    from png_cases import content, pil_png

    payloads = [pil_png(content("scene", 200 + 7 * i, 120 + 3 * i, i)) for i in range(5)]
    payloads.insert(2, pil_png(content("scene", 50, 40, 9), "RGBA"[:3]))  # plain RGB
    payloads.insert(4, dict(bad_cases())["truncated_tail"])  # Pillow decodes it, device may not
    dec = PngDecoder(torch.device("cuda:0"), max_work_bytes=3 << 20)
    for sync in (True, False):
        res = dec.decode(payloads, sync=sync)
        pk = res if sync else res.images
        if not sync:
            res.finish()
        host = pk.data.cpu().numpy()
        for k, (o, (w, h)) in enumerate(zip(pk.offsets_host, pk.wh_host)):
            got = host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            assert np.array_equal(got, _host(payloads[k])), k


def test_png_fuzzed_payloads_match_reference():
    """Random damage to valid PNGs (bit flips in the IDAT data, dropped bytes, truncation):
    every payload comes out exactly as the reference's decode gives it -- the same pixels
    or the same exception -- and nothing hangs or faults on the device."""
    import re

    import torch

    from paper_2603_16987_b200.png import PngDecoder
    from png_cases import fuzzed

    addr = re.compile(r"0x[0-9a-f]+")
    dec = PngDecoder(torch.device("cuda:0"))
    for t, kind, p in fuzzed(128):
        try:
            ref, ref_exc = _host(p), None
        except Exception as exc:  # noqa: BLE001
            ref, ref_exc = None, exc
        try:
            pk = dec.decode([p])
            w, h = (int(v) for v in pk.wh_host[0])
            got, got_exc = pk.data[: w * h * 3].cpu().numpy().reshape(h, w, 3), None
        except Exception as exc:  # noqa: BLE001
            got, got_exc = None, exc
        if ref_exc is not None:
            assert got_exc is not None and type(got_exc) is type(ref_exc), (t, kind, ref_exc)
            assert addr.sub("0x", str(got_exc)) == addr.sub("0x", str(ref_exc)), t
        else:
            assert got_exc is None, (t, kind, got_exc)
            assert np.array_equal(got, ref), (t, kind)


def test_png_false_finder_starts_are_dropped():
    """Every third unit start moved one bit on (a planted finder false positive): the
    chain check drops them all in one walk, the preceding units decode again, and the
    images still decode on the device, bit-exact."""
    import torch

    from paper_2603_16987_b200.png import PngDecoder
    from png_cases import content, pil_png

    payloads = [pil_png(content("scene", 1280, 720, 21)), pil_png(content("scene", 640, 480, 22)),
                pil_png(content("noise", 700, 500, 23))]
    dec = PngDecoder(torch.device("cuda:0"))
    dec._debug_flags = 1
    pk = dec.decode(payloads)
    assert dec.last_fallback == []
    host = pk.data.cpu().numpy()
    for k, (o, (w, h)) in enumerate(zip(pk.offsets_host, pk.wh_host)):
        got = host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
        assert np.array_equal(got, _host(payloads[k])), k
