"""JPEG test inputs shared by the CPU and GPU decode tests: the reference corpus files
(tests/golden/jpeg, written by the reference's own make_corpus.py) and payloads encoded
here with Pillow (the encoder the reference corpus uses) over sizes, qualities,
subsampling modes, restart intervals, grayscale and content kinds."""

from __future__ import annotations

import io
import json
from pathlib import Path

import numpy as np
from PIL import Image

GOLDEN_JPEG = Path(__file__).resolve().parent / "golden" / "jpeg"


def corpus_files():
    meta = json.loads((GOLDEN_JPEG / "manifest.json").read_text())
    return [(m["file"], (GOLDEN_JPEG / m["file"]).read_bytes()) for m in meta]


def scene(w: int, h: int, seed: int, noise: float = 10.0) -> np.ndarray:
    """Smooth gradients + a few blocks + Gaussian noise (corpus-like content)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float32)
    a = np.stack([(xx * 0.9 + yy * 0.4) % 256, 128 + 100 * np.sin(xx / 37.0 + yy / 53.0),
                  (yy * 0.7 + 40) % 256], axis=-1)
    for _ in range(3):
        x0, y0 = int(rng.integers(0, max(w // 2, 1))), int(rng.integers(0, max(h // 2, 1)))
        a[y0: y0 + h // 4, x0: x0 + w // 4] = rng.uniform(0, 255, 3)
    a += rng.normal(0.0, noise, a.shape)
    return np.clip(a, 0, 255).astype(np.uint8)


def encode(px: np.ndarray, quality: int = 85, gray: bool = False, **kw) -> bytes:
    im = Image.fromarray(px)
    if gray:
        im = im.convert("L")
    buf = io.BytesIO()
    im.save(buf, format="JPEG", quality=quality, **kw)
    return buf.getvalue()


def pil_rgb(data: bytes) -> np.ndarray:
    """The reference's decode of a payload (Pillow, then RGB)."""
    return np.asarray(Image.open(io.BytesIO(data)).convert("RGB"))


def small_cases(seed: int = 0):
    """(name, payload) over odd sizes x subsampling x quality x content, restart
    markers and grayscale; small enough for the pure-Python oracle."""
    rng = np.random.default_rng(seed)
    out = []
    for w, h in [(64, 48), (37, 29), (100, 75), (17, 9), (3, 5), (2, 2), (1, 1), (130, 66),
                 (33, 200), (8, 8), (16, 16), (15, 17)]:
        for ss in (0, 1, 2):
            q = int(rng.choice([50, 85, 97]))
            px = scene(w, h, int(rng.integers(1 << 30))) if rng.random() < 0.7 else \
                rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
            out.append((f"{w}x{h}_ss{ss}_q{q}", encode(px, q, subsampling=ss)))
    px = scene(90, 70, 7)
    out.append(("rst3_420", encode(px, 85, restart_marker_blocks=3)))
    out.append(("rst1_444", encode(px, 85, subsampling=0, restart_marker_blocks=1)))
    out.append(("gray", encode(px, 85, gray=True)))
    out.append(("gray_rst", encode(px, 85, gray=True, restart_marker_blocks=2)))
    return out


def fuzzed(n: int, seed: int = 20261019):
    """n damaged baseline JPEGs as (t, kind, payload): kind 0 flips bits in the entropy-
    coded data, 1 drops 1-4 bytes from it, 2 truncates the file inside the scan.  The six
    bases cover 4:2:0 / 4:4:4 / 4:2:2-free colour, restart markers, noise and grayscale."""
    rng = np.random.default_rng(seed)
    base = [encode(scene(160, 120, 1)), encode(scene(97, 61, 2), quality=95),
            encode(scene(200, 90, 3), subsampling=0),
            encode(scene(128, 128, 4), restart_marker_blocks=4),
            encode(np.random.default_rng(5).integers(0, 256, (64, 80, 3), dtype=np.uint8)),
            encode(scene(90, 70, 6), gray=True)]
    out = []
    for t in range(n):
        p = bytearray(base[t % len(base)])
        sos = p.find(b"\xff\xda")
        start = sos + 2 + int.from_bytes(p[sos + 2: sos + 4], "big")
        kind = t % 3
        if kind == 0:
            for _ in range(1 + t % 4):
                i = int(rng.integers(start, len(p) - 2))
                p[i] ^= 1 << int(rng.integers(0, 8))
        elif kind == 1:
            i = int(rng.integers(start, len(p) - 2))
            del p[i: i + int(rng.integers(1, 5))]
        else:
            p = p[: int(rng.integers(start, len(p)))]
        out.append((t, kind, bytes(p)))
    return out
