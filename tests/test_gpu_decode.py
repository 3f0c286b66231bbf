"""Mixed JPEG / PNG batches through decode.ImageDecoder: every image equals the
reference's decode (Pillow, imgproc.py:213-229), in the caller's order."""

import io

import numpy as np
import pytest
from PIL import Image

from jpeg_cases import encode, scene
from png_cases import content, pil_png

pytestmark = pytest.mark.gpu


def _pillow(p):
    from paper_2603_16987_b200._decode import decode_rgb

    return decode_rgb(p)


def test_mixed_batch_in_order():
    import torch

    from paper_2603_16987_b200.decode import ImageDecoder

    prog = io.BytesIO()
    Image.fromarray(scene(150, 90, 3)).save(prog, format="JPEG", quality=80, progressive=True)
    payloads = [encode(scene(320, 200, 1)), pil_png(content("scene", 200, 120, 2)),
                prog.getvalue(), pil_png(content("flat", 64, 48, 3), "P"),
                encode(scene(97, 33, 4), quality=95), pil_png(content("noise", 50, 30, 5), "L")]
    dec = ImageDecoder(torch.device("cuda:0"))
    for batch in (payloads, payloads[::-1], [payloads[0], payloads[4]], [payloads[1], payloads[3]]):
        pk = dec.decode(batch)
        host = pk.data.cpu().numpy()
        for k, (o, (w, h)) in enumerate(zip(pk.offsets_host, pk.wh_host)):
            got = host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            assert np.array_equal(got, _pillow(batch[k])), k
    pk = dec.decode(payloads)
    assert dec.last_fallback == [2]  # the progressive JPEG: Pillow on the host
