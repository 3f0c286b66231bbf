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


def test_mixed_batches_of_damaged_payloads():
    """Decodable damaged JPEGs and PNGs (tests' fuzz generators) interleaved with clean
    ones in mixed batches: every image equals Pillow's decode, in the caller's order, and
    a damaged image sent to the host does not disturb its neighbours on the device."""
    import jpeg_cases
    import png_cases
    import torch

    from paper_2603_16987_b200.decode import ImageDecoder

    pool = []
    for _, _, p in jpeg_cases.fuzzed(120, seed=3) + png_cases.fuzzed(240, seed=3):
        try:
            pool.append((p, _pillow(p)))
        except Exception:  # noqa: BLE001 -- Pillow rejects it: not a decodable payload
            pass
    clean = [encode(scene(200, 150, 8)), pil_png(content("scene", 180, 100, 9)),
             pil_png(content("smooth", 90, 60, 10), "P"), encode(scene(64, 64, 11), gray=True)]
    pool += [(p, _pillow(p)) for p in clean]
    rng = np.random.default_rng(4)
    dec = ImageDecoder(torch.device("cuda:0"))
    for _ in range(4):
        pick = rng.permutation(len(pool))[:48]
        batch = [pool[i] for i in pick]
        pk = dec.decode([p for p, _ in batch])
        host = pk.data.cpu().numpy()
        for k, ((_, ref), o, (w, h)) in enumerate(zip(batch, pk.offsets_host, pk.wh_host)):
            got = host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            assert np.array_equal(got, ref), k
