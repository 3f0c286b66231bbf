#!/usr/bin/env python3
"""Generate the golden vectors the oracle and the CUDA path are pinned to.

Runs the REFERENCE implementation itself (vlmfp, imported read-only from
/root/reference/pkg/src) and writes its outputs to tests/golden/golden_v1.npz
plus golden_v1.json.  Inputs are regenerated from seeds at test time
(np.random.default_rng), so only outputs are stored.  The GPU box has no
/root/reference: tests there read these committed files only.

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import io
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT_NPZ = HERE / "golden_v1.npz"
OUT_JSON = HERE / "golden_v1.json"

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)

# small-image tiling cases: (name, h, w, c, tile_edge, max_tiles, kind, seed)
TILE_CASES = [
    ("wide_1x2", 30, 60, 3, 8, 6, "random", 3),
    ("odd_23x37", 23, 37, 3, 8, 6, "random", 11),
    ("gray_17x9", 17, 9, 1, 4, 4, "random", 5),
    ("tall_75x30", 75, 30, 3, 16, 12, "random", 21),
    ("up_48x64", 48, 64, 3, 16, 12, "random", 7),
    ("smooth_97x131", 97, 131, 3, 32, 12, "smooth", 13),
    ("square_1x1", 40, 40, 3, 16, 12, "random", 17),
    ("tiny_1x1px", 1, 1, 3, 8, 12, "random", 19),
    ("strip_5x200", 5, 200, 3, 16, 12, "random", 23),
    ("mid_333x517", 333, 517, 3, 64, 12, "smooth", 29),
]

# end-to-end preprocess() cases on PNG payloads: (name, h, w, seed, cfg kwargs, defer)
PREPROCESS_CASES = [
    ("pp_f32", 24, 36, 0, dict(tile_edge=8, max_tiles=4), False),
    ("pp_bf16_imagenet", 20, 28, 1, dict(tile_edge=8, max_tiles=4, mean=IMAGENET_MEAN,
                                          std=IMAGENET_STD, reduced_precision_normalize=True),
     False),
    ("pp_defer", 30, 60, 2, dict(tile_edge=8, max_tiles=6), True),
    ("pp_split", 16, 24, 9, dict(tile_edge=8, max_tiles=4, avoid_per_item_split=True,
                                  fused_transform=True, skip_pixel_mask=True), False),
]

PROMPTS = [
    "describe the image",
    "what is in the picture ?",
    "count the objects in the scene",
    "describe every region with a caption",
    "what color is the largest object ?",
    "is there a person in the image ?",
    "summarize the scene in one sentence",
    "list the animals you can see",
    "where is the small red box ?",
    "what is behind the large object ?",
    "read any visible text in the image",
    "describe the background of the photo",
]


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
    """Shared with the tests (tests/golden_data.py re-implements it identically)."""
    rng = np.random.default_rng(seed)
    if kind == "random":
        return rng.integers(0, 256, size=(h, w, c), dtype=np.uint8)
    return smooth_image(rng, h, w, c)


def plan_inputs() -> np.ndarray:
    rng = np.random.default_rng(20260817)
    rows = []
    for _ in range(3000):
        rows.append((int(rng.integers(1, 4097)), int(rng.integers(1, 4097)),
                     int(rng.integers(1, 13))))
    for _ in range(400):  # large edges, inside the 65536 exact domain
        rows.append((int(rng.integers(1, 65537)), int(rng.integers(1, 65537)),
                     int(rng.integers(1, 13))))
    for wh in [(1920, 1080), (3840, 2160), (640, 480), (448, 448), (900, 450), (800, 600),
               (1, 1), (65536, 1), (1, 65536), (65536, 65536), (977, 313), (300, 100)]:
        for mt in (1, 4, 6, 12):
            rows.append((*wh, mt))
    # exact-tie aspect ratios: w/h = sqrt(c1 c2 / (r1 r2)) rational, and ratios of
    # candidate grids themselves (every candidate pair with equal c/r ties too)
    ties = set()
    for mt in range(1, 13):
        cands = [(r, c) for r in range(1, mt + 1) for c in range(1, mt // r + 1)]
        for r1, c1 in cands:
            for r2, c2 in cands:
                num, den = c1 * c2, r1 * r2
                sn, sd = math.isqrt(num), math.isqrt(den)
                if sn * sn == num and sd * sd == den:
                    for s in (1, 2, 3, 7):
                        ties.add((sn * s, sd * s, mt))
                for s in (1, 5):
                    ties.add((c1 * s, r1 * s, mt))
    rows.extend(sorted(ties))
    return np.asarray(rows, dtype=np.int64)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from PIL import Image
    from vlmfp import imgproc as R
    from vlmfp import tokenizer as T
    from vlmfp.tokenred import tokens_per_tile

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": "vlmfp (pkg/src) at /root/reference", "cases": {}}

    # 1. planner ---------------------------------------------------------------
    pin = plan_inputs()
    plans = []
    for w, h, mt in pin:
        p = R.select_tile_plan(int(w), int(h), R.PreprocessConfig(tile_edge=32, max_tiles=int(mt)))
        plans.append((p.rows, p.cols, p.tile_edge, int(p.include_thumbnail), p.resized_width,
                      p.resized_height))
    arrays["plan_in"] = pin
    arrays["plan_out"] = np.asarray(plans, dtype=np.int64)

    # 2. resize ----------------------------------------------------------------
    rng = np.random.default_rng(99)
    rcases = []
    for i in range(160):
        h, w = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        c = int(rng.choice([1, 3]))
        oh, ow = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        rcases.append((h, w, c, oh, ow, 1000 + i, "random"))
    rcases += [(37, 53, 3, 17, 91, 5000, "random"), (64, 48, 3, 480, 640, 5001, "smooth"),
               (101, 203, 1, 50, 33, 5002, "random"), (2, 2, 1, 1, 1, -1, "checker"),
               (5, 9, 3, 5, 9, 7, "random")]
    meta["resize_cases"] = rcases
    for i, (h, w, c, oh, ow, seed, kind) in enumerate(rcases):
        if kind == "checker":
            arr = np.array([[0, 255], [255, 0]], dtype=np.uint8)[:, :, None]
        else:
            arr = make_input(h, w, c, kind, seed)
        out = R.resize_bilinear(R.ImageBuffer.from_array(arr), ow, oh)
        arrays[f"resize_{i}"] = out.data

    # 3. tiling + normalize ------------------------------------------------------
    meta["tile_cases"] = TILE_CASES
    for name, h, w, c, e, mt, kind, seed in TILE_CASES:
        arr = make_input(h, w, c, kind, seed)
        img = R.ImageBuffer.from_array(arr)
        cfg = R.PreprocessConfig(tile_edge=e, max_tiles=mt)
        plan = R.select_tile_plan(w, h, cfg)
        tiles = R.tile_image(img, plan, cfg)
        arrays[f"tile_{name}_plan"] = np.array(
            [plan.rows, plan.cols, plan.tile_edge, int(plan.include_thumbnail),
             plan.resized_width, plan.resized_height], dtype=np.int64)
        arrays[f"tile_{name}_u8"] = np.stack([t.data for t in tiles])
        norm = R.normalize_tiles(tiles, R.PreprocessConfig(tile_edge=e, max_tiles=mt,
                                                           mean=IMAGENET_MEAN, std=IMAGENET_STD))
        arrays[f"tile_{name}_f32_imagenet"] = np.stack([t.data for t in norm])
        normb = R.normalize_tiles(tiles, R.PreprocessConfig(tile_edge=e, max_tiles=mt,
                                                            reduced_precision_normalize=True))
        arrays[f"tile_{name}_bf16_half_bits"] = np.stack([t.data for t in normb]).view(np.uint16)

    # 4. normalize LUTs ---------------------------------------------------------
    allv = np.tile(np.arange(256, dtype=np.uint8)[None, :, None], (1, 1, 3))
    for tag, mean, std in (("half", (0.5,) * 3, (0.5,) * 3), ("imagenet", IMAGENET_MEAN,
                                                               IMAGENET_STD)):
        for prec in ("f32", "bf16"):
            cfg = R.PreprocessConfig(mean=mean, std=std,
                                     reduced_precision_normalize=(prec == "bf16"))
            out = R.normalize(R.ImageBuffer.from_array(allv), cfg).data[0]  # [256, 3]
            out = np.ascontiguousarray(out.T)
            arrays[f"lut_{tag}_{prec}"] = out.view(np.uint16) if prec == "bf16" else out
        gray = R.normalize(R.ImageBuffer.from_array(allv[:, :, :1]),
                           R.PreprocessConfig(mean=mean, std=std)).data[0]
        arrays[f"lut_{tag}_f32_gray"] = np.ascontiguousarray(gray.T)

    # 5. end-to-end preprocess on PNG payloads -----------------------------------
    meta["preprocess_cases"] = [(n, h, w, s, kw, d) for n, h, w, s, kw, d in PREPROCESS_CASES]
    for name, h, w, seed, kw, defer in PREPROCESS_CASES:
        arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        buf = io.BytesIO()
        Image.fromarray(arr).save(buf, format="PNG")
        res = R.preprocess(buf.getvalue(), R.PreprocessConfig(**kw), defer_normalize=defer)
        data = np.stack([t.data for t in res.tiles])
        if data.dtype != np.uint8 and data.dtype != np.float32:
            data = data.view(np.uint16)
        arrays[f"pp_{name}"] = data
        meta["cases"][name] = {
            "plan": [res.plan.rows, res.plan.cols, res.plan.tile_edge,
                     int(res.plan.include_thumbnail), res.plan.resized_width,
                     res.plan.resized_height],
            "keys": sorted(res.stage_timings_ns),
            "elem": res.tiles[0].elem,
        }

    # 6. token expansion ---------------------------------------------------------
    vocab = T.load_vocab(Path(args.ref) / "vlmfp" / "data" / "base_vocab.txt")
    sp = vocab.specials
    meta["specials"] = {k: getattr(sp, k) for k in ("bos", "eos", "user_header",
                                                     "assistant_header", "image_marker",
                                                     "image_context", "pad")}
    prompt_ids = []
    for p in PROMPTS:
        text, counts = T.render_chat([T.ChatMessage("user", (T.ImagePart(1), T.TextPart(p)))],
                                     vocab)
        prompt_ids.append(T.tokenize(text, vocab))
    meta["prompt_ids"] = prompt_ids
    exp_cases = []
    rng = np.random.default_rng(4242)
    words = ["describe", "the", "image", "objects", "left", "right", "red", "car", "a", "count"]
    for i in range(60):
        parts = []
        for _ in range(int(rng.integers(1, 5))):
            if rng.random() < 0.5:
                parts.append(T.TextPart(" ".join(rng.choice(words, size=int(rng.integers(1, 5))))
                                        + " "))
            else:
                parts.append(T.ImagePart(int(rng.integers(1, 14))))
        msgs = [T.ChatMessage("user", tuple(parts))]
        if rng.random() < 0.5:
            msgs.append(T.ChatMessage("assistant", (T.TextPart(
                " ".join(rng.choice(words, size=int(rng.integers(1, 6))))),)))
        tpt = int(rng.choice([1, 4, 64, 256]))
        text, counts = T.render_chat(msgs, vocab)
        ids = T.tokenize(text, vocab)
        seq = T.build_token_sequence(msgs, vocab, tpt)
        plain = T.expand_image_placeholders(ids, counts, tpt, vocab)
        assert plain.ids == seq.ids
        exp_cases.append({"ids": ids, "counts": counts, "tpt": tpt, "out_len": len(seq.ids),
                          "spans": seq.image_spans, "first": seq.first_assistant_index})
        arrays[f"expand_{i}_ids"] = np.asarray(seq.ids, dtype=np.int32)
        arrays[f"expand_{i}_mask"] = np.asarray(seq.supervision_mask, dtype=np.uint8)
    meta["expand_cases"] = exp_cases
    meta["tokens_per_tile"] = {"512_16_4": tokens_per_tile(512, 16, 4),
                               "448_14_2": tokens_per_tile(448, 14, 2)}

    # 7. pixel_unshuffle ------------------------------------------------------------
    from vlmfp.tokenred import PatchGrid, pixel_unshuffle

    ucases = [(4, 6, 3, 2, "float32", 1), (32, 32, 5, 2, "float32", 2), (8, 12, 7, 4, "int32", 3),
              (6, 9, 2, 3, "float64", 4), (5, 5, 4, 1, "float32", 5)]
    meta["unshuffle_cases"] = ucases
    for i, (h, w, d, r, dt, seed) in enumerate(ucases):
        data = np.random.default_rng(seed).standard_normal(h * w * d).astype(dt)
        out = pixel_unshuffle(PatchGrid(h, w, d, data), r)
        arrays[f"unshuffle_{i}"] = out.data
        meta.setdefault("unshuffle_shapes", []).append([out.h, out.w, out.d])

    # 8. greedy tokenizer ------------------------------------------------------------
    # the reference vocabulary file (a data fixture: the GPU box has no /root/reference)
    vocab_path = Path(args.ref) / "vlmfp" / "data" / "base_vocab.txt"
    meta["vocab_file"] = vocab_path.read_text(encoding="utf-8")
    rng = np.random.default_rng(777)
    alphabet = list("abcdefghijklmnopqrstuvwxyz ABCXYZ0123456789.,;:!?'\"()[]{}<>|_-+=/\\\n\t") + [
        "\u00e9", "\u00fc", "\u4e2d", "\u6587", "\u2603", "\U0001F600", "<|user|>", "<|image|>",
        "<IMG_CONTEXT>", "<|assistant|>", "<|bos|>", "<|eos|>", "<|pad|>", "<|", "|>", "describe",
        "image", "the ", " of ", "\x00", "\x7f"]
    texts = ["", "a", " ", "<|user|><|image|>describe the image<|assistant|>", "\u2603" * 5,
             "<<|||>>", "<|assistant|" * 3, "x" * 3000]
    for _ in range(300):
        k = int(rng.integers(0, 60))
        texts.append("".join(str(alphabet[int(j)]) for j in rng.integers(0, len(alphabet), k)))
    meta["tok_texts"] = texts
    meta["tok_ids"] = [T.tokenize(t, vocab) for t in texts]

    np.savez_compressed(OUT_NPZ, **arrays)
    OUT_JSON.write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT_NPZ} ({OUT_NPZ.stat().st_size / 1e6:.2f} MB), {OUT_JSON}")


if __name__ == "__main__":
    main()
