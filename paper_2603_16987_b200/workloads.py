"""The BASELINE.json configurations as synthetic workloads, and the
algorithmic-byte model the roofline is quoted against.

Bytes per image (the definition `roofline.achieved` uses):
    B = R_touched * W * C  +  n_images * C * E^2 * s_out  (+ C * E^2 per tile
        when the uint8 side output is also written)
where R_touched is the number of distinct source rows the 2-tap stencil reads
(tile rows H -> rows*E and thumbnail rows H -> E); columns are not
discounted (horizontal steps stay below the 32 B sector).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)

# (width : height) ratios of the reference corpus (scripts/make_corpus.py:35-48)
ASPECT_RATIOS = [(1, 1), (4, 3), (3, 4), (3, 2), (2, 3), (16, 9), (9, 16), (2, 1), (1, 2),
                 (5, 4), (7, 5), (3, 1)]


@dataclass(frozen=True)
class Workload:
    name: str
    description: str
    wh: np.ndarray  # [n, 2] int32
    tile_edge: int
    max_tiles: int
    mean: tuple
    std: tuple
    bf16: bool
    seed: int


def c2(n: int = 64) -> Workload:
    """configs[1]: InternVL3-2B dynamic tiling, 448 px tiles, max 12 + thumbnail,
    ImageNet mean/std, batch of 64 synthetic 1080p images, bf16 NCHW out."""
    return Workload("C2", "InternVL3-2B tiling: 64 x 1920x1080 RGB, E=448, max 12 + thumb, "
                    "ImageNet mean/std, bf16 NCHW", np.tile([[1920, 1080]], (n, 1)).astype(np.int32),
                    448, 12, IMAGENET_MEAN, IMAGENET_STD, True, 20260817)


def c1() -> Workload:
    """configs[0]: SmolVLM-style, one 1920x1080 image, 512 px tiles, mean=std=0.5, fp32."""
    return Workload("C1", "SmolVLM-style: 1 x 1920x1080, E=512, max 12, mean=std=0.5, fp32",
                    np.array([[1920, 1080]], dtype=np.int32), 512, 12, (0.5,) * 3, (0.5,) * 3,
                    False, 20260817)


def c3() -> Workload:
    """configs[2]: batch-1 latency, one 3840x2160 image, InternVL3-2B tiling."""
    return Workload("C3", "batch-1 latency: 1 x 3840x2160, E=448, ImageNet, bf16 NCHW",
                    np.array([[3840, 2160]], dtype=np.int32), 448, 12, IMAGENET_MEAN,
                    IMAGENET_STD, True, 20260817)


def c4_shapes(n: int = 8192, start: int = 0) -> np.ndarray:
    """configs[3] sizes: image i has aspect ASPECT_RATIOS[i % 12], short edge
    uniform in [480, 2160] (default_rng(20261018 + i)), long edge
    round(short * ratio) capped at 3840."""
    out = np.empty((n, 2), dtype=np.int32)
    for j in range(n):
        i = start + j
        a, b = ASPECT_RATIOS[i % 12]
        short = int(np.random.default_rng(20261018 + i).integers(480, 2161))
        long_ = min(3840, int(round(short * max(a, b) / min(a, b))))
        out[j] = (long_, short) if a >= b else (short, long_)
    return out


def c4(n: int = 8192, start: int = 0) -> Workload:
    return Workload("C4", f"throughput sweep: {n} mixed-aspect images 480p-4K, E=448, ImageNet, "
                    "bf16 NCHW", c4_shapes(n, start), 448, 12, IMAGENET_MEAN, IMAGENET_STD,
                    True, 20261018)


def axis_rows(src: int, out: int) -> np.ndarray:
    """Source indices {i0, i1} the half-pixel 2-tap stencil reads along one axis
    (same formula as imgproc.py:298-306; used only to count bytes)."""
    pos = (np.arange(out, dtype=np.float64) + 0.5) * (src / out) - 0.5
    pos = np.minimum(np.maximum(pos, 0.0), float(src - 1))
    i0 = np.minimum(np.floor(pos).astype(np.int64), src - 1)
    return np.union1d(i0, np.minimum(i0 + 1, src - 1))


def plan_rows_cols(w: int, h: int, tile_edge: int, max_tiles: int) -> tuple[int, int]:
    """Exact integer grid choice (same rule as K1; used only to count bytes)."""
    best = None
    for r in range(1, max_tiles + 1):
        for c in range(1, max_tiles // r + 1):
            a, b = w * r, h * c
            key = (max(a, b), min(a, b))
            if best is None:
                best = (key, r, c)
                continue
            lhs, rhs = key[0] * best[0][1], best[0][0] * key[1]
            if lhs < rhs or (lhs == rhs and (r * c, r) < (best[1] * best[2], best[1])):
                best = (key, r, c)
    return best[1], best[2]


def image_bytes(w: int, h: int, tile_edge: int, max_tiles: int, channels: int = 3,
                s_out: int = 2, with_u8: bool = False) -> dict:
    rows, cols = plan_rows_cols(w, h, tile_edge, max_tiles)
    n_img = rows * cols + (1 if rows * cols > 1 else 0)
    touched = axis_rows(h, rows * tile_edge)
    if n_img > rows * cols:
        touched = np.union1d(touched, axis_rows(h, tile_edge))
    read = int(len(touched)) * w * channels
    per_tile = channels * tile_edge * tile_edge * (s_out + (1 if with_u8 else 0))
    return {"read": read, "write": n_img * per_tile, "n_images": n_img,
            "read_full": w * h * channels}


def workload_bytes(wl: Workload, with_u8: bool = False) -> dict:
    """Algorithmic bytes of a whole workload (cached per distinct shape)."""
    s_out = 2 if wl.bf16 else 4
    cache: dict = {}
    tot = {"read": 0, "write": 0, "n_images": 0, "read_full": 0}
    for w, h in wl.wh:
        key = (int(w), int(h))
        if key not in cache:
            cache[key] = image_bytes(*key, wl.tile_edge, wl.max_tiles, 3, s_out, with_u8)
        for k in tot:
            tot[k] += cache[key][k]
    tot["total"] = tot["read"] + tot["write"]
    return tot


# ---------------------------------------------------------------------------
# compressed inputs: corpus-like content encoded as JPEG (decode-inclusive end to end)

def scene_image(width: int, height: int, seed: int, noise: float = 10.0) -> np.ndarray:
    """Smooth gradients + a few flat blocks + Gaussian noise, the character of the
    reference corpus (make_corpus.py:111-136 draws sinusoid fields, blocks and N(0, 10)
    noise); synthetic, generated here."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float32)
    a = np.stack([(xx * 0.9 + yy * 0.4) % 256, 128 + 100 * np.sin(xx / 37.0 + yy / 53.0),
                  (yy * 0.7 + 40) % 256], axis=-1)
    for _ in range(3):
        x0 = int(rng.integers(0, max(width // 2, 1)))
        y0 = int(rng.integers(0, max(height // 2, 1)))
        a[y0: y0 + height // 4, x0: x0 + width // 4] = rng.uniform(0, 255, 3)
    a += rng.normal(0.0, noise, a.shape).astype(np.float32)
    return np.clip(a, 0, 255).astype(np.uint8)


def jpeg_payloads(n: int, width: int = 1920, height: int = 1080, quality: int = 85,
                  seed: int = 20260817, distinct: int = 8) -> list:
    """n JPEG payloads (Pillow, baseline 4:2:0, the reference corpus encoder settings,
    make_corpus.py:139-142) of `distinct` different scenes, repeated."""
    import io

    from PIL import Image

    base = []
    for k in range(min(n, distinct)):
        buf = io.BytesIO()
        Image.fromarray(scene_image(width, height, seed + k)).save(buf, format="JPEG",
                                                                   quality=quality)
        base.append(buf.getvalue())
    return [base[k % len(base)] for k in range(n)]


def png_payloads(n: int, width: int = 1920, height: int = 1080, seed: int = 20260817,
                 distinct: int = 8) -> list:
    """n PNG payloads of `distinct` different scenes, repeated, written by Pillow with its
    default settings (the encoder of the reference's own PNG path, decode_image's
    re-encode, imgproc.py:252-256)."""
    import io

    from PIL import Image

    base = []
    for k in range(min(n, distinct)):
        buf = io.BytesIO()
        Image.fromarray(scene_image(width, height, seed + k)).save(buf, format="PNG")
        base.append(buf.getvalue())
    return [base[k % len(base)] for k in range(n)]


# ---------------------------------------------------------------------------
# C5 prompts: rendered chat prompts tokenized on the device (K6)

C5_PROMPTS = [
    "describe the image",
    "what is in the picture?",
    "count the objects in the scene",
    "describe every region with a caption",
    "what color is the car on the left?",
    "read the text in the image",
    "is there a person in this photo? answer yes or no",
    "list the objects from left to right",
    "where was this picture taken?",
    "summarize the chart in one sentence",
    "what is unusual about this image?",
    "give a detailed description of the scene, including the background",
]

_C5_WORDS = ["describe", "the", "image", "picture", "what", "count", "objects", "scene",
             "every", "region", "caption", "color", "left", "right", "text", "person",
             "photo", "answer", "where", "chart", "sentence", "unusual", "detailed", " the ",
             " of ", " in ", "ing", "tion"]


def synthetic_vocab_text() -> str:
    """A vocab file in the reference format (JSON header naming the specials, one token
    per line): the specials, all 256 byte-fallback tokens, printable ASCII and a few
    words. Synthetic (the reference vocabulary does not travel to the GPU box)."""
    specials = {"bos": "<|bos|>", "eos": "<|eos|>", "user_header": "<|user|>",
                "assistant_header": "<|assistant|>", "image_marker": "<|image|>",
                "image_context": "<IMG_CONTEXT>", "pad": "<|pad|>"}
    import json as _json

    toks = list(specials.values()) + [f"<0x{b:02X}>" for b in range(256)]
    toks += [chr(c) for c in range(32, 127)] + _C5_WORDS
    return _json.dumps({"specials": specials}) + "\n" + "\n".join(toks) + "\n"


def c5_texts(n: int, seed: int = 20261018) -> list:
    """n rendered prompts: "<|user|><|image|>" + prompt + "<|assistant|>"."""
    rng = np.random.default_rng(seed)
    return ["<|user|><|image|>" + C5_PROMPTS[int(rng.integers(len(C5_PROMPTS)))] + "<|assistant|>"
            for _ in range(n)]
