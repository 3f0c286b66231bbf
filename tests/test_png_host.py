"""K8 host side (no GPU): tp_png_parse takes exactly the PNGs whose decode the device can
reproduce, and leaves everything Pillow treats specially to Pillow."""

import pytest

from png_cases import bad_cases, content, custom_cases, custom_png, pil_cases, pil_png
from paper_2603_16987_b200 import png as P


@pytest.fixture(scope="module", autouse=True)
def _lib():
    pytest.importorskip("ctypes")
    from paper_2603_16987_b200 import _lib

    try:
        _lib.load()
    except _lib.LibraryMissingError:
        pytest.skip("libtileprep.so not built")


def test_pillow_pngs_are_device_decodable():
    for name, payload in pil_cases():
        info, offs, lens = P.parse(payload)
        assert info.status == P.TP_PNG_OK, (name, info.message)
        assert int(lens.sum()) == info.zlib_len
        assert info.color_type in (0, 2, 3)


def test_custom_pngs_parse():
    for name, payload in custom_cases():
        info, offs, lens = P.parse(payload)
        assert info.status == P.TP_PNG_OK, (name, info.message)
        # the IDAT data back to back is the zlib stream
        z = b"".join(payload[o: o + n] for o, n in zip(offs.tolist(), lens.tolist()))
        import zlib

        zlib.decompress(z)


def test_idat_table_grows():
    a = content("scene", 64, 64, 1)
    payload = custom_png(a, 2, idat=7)  # hundreds of IDAT chunks
    info, offs, lens = P.parse(payload, cap=4)
    assert info.status == P.TP_PNG_OK and len(offs) == info.n_idat > 4


@pytest.mark.parametrize("name", ["ihdr_crc", "rgba", "la"])
def test_left_to_pillow(name):
    payload = dict(bad_cases())[name]
    info, _, _ = P.parse(payload)
    assert info.status == P.TP_PNG_UNSUPPORTED


def test_modes_left_to_pillow():
    import numpy as np

    a = content("scene", 40, 30, 2)
    assert P.parse(pil_png(a, "RGBA"))[0].status == P.TP_PNG_UNSUPPORTED
    g16 = (a[..., 0].astype(np.uint16) * 257)
    from PIL import Image
    import io

    buf = io.BytesIO()
    Image.fromarray(g16).save(buf, format="PNG")
    assert P.parse(buf.getvalue())[0].status == P.TP_PNG_UNSUPPORTED
    assert P.parse(pil_png(a, "1"))[0].status == P.TP_PNG_UNSUPPORTED
    # a chunk with a Pillow handler after the image data: Pillow may raise there
    late = custom_png(a, 2, post_chunks=[(b"tEXt", b"k\0v")])
    assert P.parse(late)[0].status == P.TP_PNG_UNSUPPORTED
