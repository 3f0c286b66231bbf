"""Input regeneration for the golden cases (same generators as make_golden.py)."""

from __future__ import annotations

import math

import numpy as np

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def smooth_image(rng: np.random.Generator, h: int, w: int, c: int) -> np.ndarray:
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    chans = []
    for _ in range(c):
        a, f, p = rng.uniform(0, 2 * math.pi), rng.uniform(1.0, 5.0), rng.uniform(0, 6.28)
        field = 127.5 + 120.0 * np.sin(
            2 * math.pi * f * (xx / max(w, 1) * math.cos(a) + yy / max(h, 1) * math.sin(a)) + p)
        chans.append(field)
    return np.clip(np.rint(np.stack(chans, axis=-1)), 0, 255).astype(np.uint8)


def make_input(h: int, w: int, c: int, kind: str, seed: int) -> np.ndarray:
    if kind == "checker":
        return np.array([[0, 255], [255, 0]], dtype=np.uint8)[:, :, None]
    rng = np.random.default_rng(seed)
    if kind == "random":
        return rng.integers(0, 256, size=(h, w, c), dtype=np.uint8)
    return smooth_image(rng, h, w, c)


def png_payload(arr: np.ndarray) -> bytes:
    import io

    from PIL import Image

    buf = io.BytesIO()
    Image.fromarray(arr).save(buf, format="PNG")
    return buf.getvalue()
