"""Pin the CPU oracle to the reference: golden vectors produced by running the
reference itself (tests/golden/make_golden.py), plus live cross-checks when
/root/reference is present.  CPU only."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from golden_data import IMAGENET_MEAN, IMAGENET_STD, make_input, png_payload
from oracle import tileprep_oracle as O


def test_plan_float_matches_golden(golden):
    data, _ = golden
    pin, want = data["plan_in"], data["plan_out"]
    got = np.array([O.plan_float(int(w), int(h), 32, int(mt)) for w, h, mt in pin])
    assert np.array_equal(got, want)


def test_plan_int_matches_golden_including_ties(golden):
    data, _ = golden
    pin, want = data["plan_in"], data["plan_out"]
    got = np.array([O.plan_int(int(w), int(h), 32, int(mt)) for w, h, mt in pin])
    assert np.array_equal(got, want)


def test_plan_int_equals_float_dense_square():
    # every (w, h) in [1, 96]^2 at the configs' max_tiles, plus max_tiles 1..12 on a coarse grid
    for mt in (6, 12):
        for w in range(1, 97):
            for h in range(1, 97):
                assert O.plan_int(w, h, 8, mt) == O.plan_float(w, h, 8, mt), (w, h, mt)
    for mt in range(1, 13):
        for w in range(1, 400, 13):
            for h in range(1, 400, 7):
                assert O.plan_int(w, h, 8, mt) == O.plan_float(w, h, 8, mt), (w, h, mt)


def test_plan_known_grids():
    assert O.plan_float(448, 448, 448, 12)[:2] == (1, 1)
    assert O.plan_float(900, 450, 448, 12) == (1, 2, 448, 1, 896, 448)
    assert O.plan_float(800, 600, 448, 12)[:2] == (3, 4)
    assert O.plan_float(1920, 1080, 512, 12) == (1, 2, 512, 1, 1024, 512)
    assert O.plan_float(3840, 2160, 448, 12) == (1, 2, 448, 1, 896, 448)
    assert O.plan_float(640, 480, 448, 12) == (3, 4, 448, 1, 1792, 1344)


def test_resize_matches_golden(golden):
    data, meta = golden
    for i, (h, w, c, oh, ow, seed, kind) in enumerate(meta["resize_cases"]):
        arr = make_input(h, w, c, kind, seed)
        want = data[f"resize_{i}"]
        assert np.array_equal(O.resize_u8(arr, ow, oh), want), i
        if h * w * oh * ow <= 4096:
            assert np.array_equal(O.resize_scalar(arr, ow, oh), want), i


def test_tiles_and_normalize_match_golden(golden):
    data, meta = golden
    for name, h, w, c, e, mt, kind, seed in meta["tile_cases"]:
        arr = make_input(h, w, c, kind, seed)
        plan = O.plan_float(w, h, e, mt)
        assert np.array_equal(np.array(plan), data[f"tile_{name}_plan"]), name
        tiles = O.tiles_u8(arr, plan)
        assert np.array_equal(tiles, data[f"tile_{name}_u8"]), name
        f32 = O.normalize(tiles, IMAGENET_MEAN, IMAGENET_STD, bf16=False)
        assert np.array_equal(f32, data[f"tile_{name}_f32_imagenet"]), name
        b16 = O.normalize(tiles, (0.5,) * 3, (0.5,) * 3, bf16=True)
        assert np.array_equal(b16.view(np.uint16), data[f"tile_{name}_bf16_half_bits"]), name


def test_luts_match_golden(golden):
    data, _ = golden
    for tag, mean, std in (("half", (0.5,) * 3, (0.5,) * 3),
                           ("imagenet", IMAGENET_MEAN, IMAGENET_STD)):
        assert np.array_equal(O.lut(mean, std, 3, False), data[f"lut_{tag}_f32"])
        assert np.array_equal(O.lut(mean, std, 3, True).view(np.uint16), data[f"lut_{tag}_bf16"])
        assert np.array_equal(O.lut(mean, std, 1, False), data[f"lut_{tag}_f32_gray"])


def test_preprocess_cases_match_golden(golden):
    data, meta = golden
    from PIL import Image
    import io

    for name, h, w, seed, kw, defer in meta["preprocess_cases"]:
        arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        dec = np.asarray(Image.open(io.BytesIO(png_payload(arr))).convert("RGB"))
        e, mt = kw["tile_edge"], kw["max_tiles"]
        plan = O.plan_float(w, h, e, mt)
        assert list(plan) == meta["cases"][name]["plan"]
        tiles = O.tiles_u8(dec, plan)
        if defer:
            got = tiles
        else:
            bf16 = kw.get("reduced_precision_normalize", False)
            got = O.normalize(tiles, kw.get("mean", (0.5,) * 3), kw.get("std", (0.5,) * 3), bf16)
            if bf16:
                got = got.view(np.uint16)
        assert np.array_equal(got, data[f"pp_{name}"]), name


def test_expand_matches_golden(golden):
    data, meta = golden
    sp = meta["specials"]
    for i, case in enumerate(meta["expand_cases"]):
        ids, spans, first = O.expand(case["ids"], case["counts"], case["tpt"],
                                     sp["image_marker"], sp["image_context"],
                                     sp["assistant_header"])
        assert ids == data[f"expand_{i}_ids"].tolist()
        assert [list(s) for s in spans] == [list(s) for s in case["spans"]]
        assert first == case["first"]
        mask = O.supervision_mask(ids, first, sp["assistant_header"])
        assert np.array_equal(mask.astype(np.uint8), data[f"expand_{i}_mask"])


def test_expand_errors():
    with pytest.raises(ValueError):
        O.expand([2, 4, 3], [1, 2], 64, 4, 5, 3)
    with pytest.raises(ValueError):
        O.expand([2, 4], [1], 64, 4, 5, 3)


def test_synth_twin_is_deterministic_and_distinct():
    a = O.synth_image(7, 0, 33, 17, 3, 0)
    b = O.synth_image(7, 0, 33, 17, 3, 0)
    c = O.synth_image(7, 1, 33, 17, 3, 0)
    assert a.shape == (17, 33, 3) and np.array_equal(a, b) and not np.array_equal(a, c)
    # uniform bytes: all 256 values appear in a 64 KiB sample
    big = O.synth_image(1, 0, 256, 256, 1, 0)
    assert len(np.unique(big)) == 256
    s = O.synth_image(3, 2, 40, 30, 3, 1)
    assert int(np.abs(np.diff(s.astype(int), axis=1)).max()) <= 6


# ---------------------------------------------------------------------------
# live cross-checks against the reference (build box only)

@pytest.mark.reference
@settings(max_examples=150, deadline=None)
@given(h=st.integers(1, 9), w=st.integers(1, 9), c=st.sampled_from([1, 3]),
       oh=st.integers(1, 9), ow=st.integers(1, 9), seed=st.integers(0, 2**31))
def test_resize_vs_live_reference(reference, h, w, c, oh, ow, seed):
    from vlmfp.imgproc import ImageBuffer, resize_bilinear

    arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, c), dtype=np.uint8)
    want = resize_bilinear(ImageBuffer.from_array(arr), ow, oh).data
    assert np.array_equal(O.resize_u8(arr, ow, oh), want)


@pytest.mark.reference
@settings(max_examples=300, deadline=None)
@given(w=st.integers(1, 65536), h=st.integers(1, 65536), mt=st.integers(1, 12))
def test_plan_vs_live_reference(reference, w, h, mt):
    from vlmfp.imgproc import PreprocessConfig, select_tile_plan

    p = select_tile_plan(w, h, PreprocessConfig(tile_edge=16, max_tiles=mt))
    want = (p.rows, p.cols, p.tile_edge, int(p.include_thumbnail), p.resized_width,
            p.resized_height)
    assert O.plan_int(w, h, 16, mt) == want
    assert O.plan_float(w, h, 16, mt) == want


@pytest.mark.reference
@settings(max_examples=40, deadline=None)
@given(h=st.integers(3, 60), w=st.integers(3, 60), seed=st.integers(0, 2**31),
       e=st.sampled_from([4, 8, 16]), mt=st.integers(1, 12))
def test_tiles_vs_live_reference(reference, h, w, seed, e, mt):
    from vlmfp.imgproc import ImageBuffer, PreprocessConfig, select_tile_plan, tile_image

    arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    cfg = PreprocessConfig(tile_edge=e, max_tiles=mt)
    plan = select_tile_plan(w, h, cfg)
    want = np.stack([t.data for t in tile_image(ImageBuffer.from_array(arr), plan, cfg)])
    assert np.array_equal(O.tiles_u8(arr, O.plan_float(w, h, e, mt)), want)


def test_pixel_unshuffle_matches_golden(golden):
    data, meta = golden
    for i, (h, w, d, r, dt, seed) in enumerate(meta["unshuffle_cases"]):
        grid = np.random.default_rng(seed).standard_normal(h * w * d).astype(dt).reshape(h, w, d)
        got = O.pixel_unshuffle(grid, r)
        assert list(got.shape) == meta["unshuffle_shapes"][i]
        assert np.array_equal(got.reshape(-1), data[f"unshuffle_{i}"])


@pytest.mark.reference
@settings(max_examples=400, deadline=None)
@given(text=st.text(max_size=80))
def test_tokenize_vs_live_reference(reference, text):
    from vlmfp import tokenizer as T

    vocab = T.load_vocab(Path("/root/reference/pkg/src/vlmfp/data/base_vocab.txt"))
    want = T.tokenize(text, vocab)
    assert O.tokenize(text, vocab.byte_ids, vocab.match_table, vocab.max_token_bytes) == want


@pytest.mark.reference
@pytest.mark.parametrize("w,h,e", [(1920, 1080, 512), (3840, 2160, 448), (640, 480, 448)])
def test_port_costs_what_vlmfp_costs(reference, w, h, e):
    """The oracle port (bench.py's CPU leg when baseline/_ref is absent) restates vlmfp's
    fused path with the same band sharing and in-place ops, so it also costs what vlmfp
    costs: C1 (1080p, E=512), C3 (4K) and a 13-tile image, best of 5 interleaved rounds on
    one core, within 40% (the restatement was measured within 10%; the margin absorbs
    load on a shared build box)."""
    import time

    from oracle import tileprep_oracle as O

    V = reference
    arr = O.synth_image(5, 0, w, h, 3, 0)
    mean, std = (0.485, 0.456, 0.406), (0.229, 0.224, 0.225)
    cfg = V.PreprocessConfig(tile_edge=e, max_tiles=12, mean=mean, std=std,
                             reduced_precision_normalize=True, fused_transform=True,
                             contiguous_tensor_path=True, avoid_per_item_split=True,
                             skip_pixel_mask=True)

    def ref():
        img = V.ImageBuffer.from_array(arr)
        plan = V.select_tile_plan(img.width, img.height, cfg)
        V.normalize_tiles(V.tile_image(img, plan, cfg), cfg)

    def port():
        O.preprocess_image(arr, e, 12, mean, std, True)

    # interleaved rounds, best of each: a load spike on the shared build box hits both
    ref(), port()
    rs, ps = [], []
    for _ in range(5):
        for fn, ts in ((ref, rs), (port, ps)):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
    r, p = min(rs), min(ps)
    assert 1 / 1.4 <= p / r <= 1.4, (r, p)
