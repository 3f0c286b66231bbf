"""The drop-in API (reference signatures) on the GPU: the reference's own
imgproc / tokenizer / tokenred / backend test cases re-expressed against this
package, plus golden-vector parity.  Runs on the B200 box (`-m gpu`)."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from golden_data import IMAGENET_MEAN, IMAGENET_STD, make_input, png_payload
from oracle import tileprep_oracle as O
import paper_2603_16987_b200 as P
from paper_2603_16987_b200.dtypes import FLOAT16_WIDE, FLOAT32, UINT8

pytestmark = pytest.mark.gpu

FAST = P.PreprocessConfig(tile_edge=16, max_tiles=4, decode_once=True, simd_decode=True,
                          fused_transform=True, contiguous_tensor_path=True,
                          skip_pixel_mask=True, avoid_per_item_split=True)


# ---------------------------------------------------------------------------
# resize (reference tests/test_imgproc.py:92-131)

def test_resize_checkerboard_halving():
    cb = P.ImageBuffer.from_array(np.array([[0, 255], [255, 0]], dtype=np.uint8))
    assert P.resize_bilinear(cb, 1, 1).data.ravel().tolist() == [128]


def test_resize_identity_is_exact():
    arr = np.random.default_rng(7).integers(0, 256, size=(5, 9, 3), dtype=np.uint8)
    assert np.array_equal(P.resize_bilinear(P.ImageBuffer.from_array(arr), 9, 5).data, arr)


def test_resize_constant_image_stays_constant():
    arr = np.full((3, 3, 3), 77, dtype=np.uint8)
    assert np.all(P.resize_bilinear(P.ImageBuffer.from_array(arr), 7, 5).data == 77)


@settings(max_examples=120, deadline=None)
@given(h=st.integers(1, 8), w=st.integers(1, 8), c=st.sampled_from([1, 3]),
       out_h=st.integers(1, 8), out_w=st.integers(1, 8), seed=st.integers(0, 2**31))
def test_resize_matches_scalar_oracle(h, w, c, out_h, out_w, seed):
    arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, c), dtype=np.uint8)
    got = P.resize_bilinear(P.ImageBuffer.from_array(arr), out_w, out_h)
    assert np.array_equal(got.data, O.resize_scalar(arr, out_w, out_h))


def test_resize_rejects_float_input():
    buf = P.ImageBuffer(2, 2, 3, FLOAT32, np.zeros((2, 2, 3), dtype=np.float32))
    with pytest.raises(ValueError):
        P.resize_bilinear(buf, 1, 1)
    with pytest.raises(ValueError):
        P.resize_bilinear(P.ImageBuffer.from_array(np.zeros((2, 2, 3), np.uint8)), 0, 1)


# ---------------------------------------------------------------------------
# planning (reference tests/test_imgproc.py:137-175)

@settings(max_examples=200, deadline=None)
@given(w=st.integers(1, 4096), h=st.integers(1, 4096), max_tiles=st.integers(1, 12))
def test_plan_matches_bruteforce(w, h, max_tiles):
    plan = P.select_tile_plan(w, h, P.PreprocessConfig(tile_edge=32, max_tiles=max_tiles))
    assert (plan.rows, plan.cols) == O.plan_float(w, h, 32, max_tiles)[:2]


def test_plan_known_grids():
    cfg = P.PreprocessConfig(tile_edge=448, max_tiles=12)
    sq = P.select_tile_plan(448, 448, cfg)
    assert (sq.rows, sq.cols) == (1, 1) and not sq.include_thumbnail
    wide = P.select_tile_plan(900, 450, cfg)
    assert (wide.rows, wide.cols) == (1, 2) and wide.include_thumbnail
    assert (wide.resized_width, wide.resized_height) == (896, 448)
    assert (P.select_tile_plan(800, 600, cfg).rows, P.select_tile_plan(800, 600, cfg).cols) == (3, 4)
    assert (P.select_tile_plan(1, 1, cfg).rows, P.select_tile_plan(1, 1, cfg).cols) == (1, 1)


def test_plan_thumbnail_iff_multi_tile():
    cfg = P.PreprocessConfig(tile_edge=64, max_tiles=12)
    for w, h in [(64, 64), (128, 64), (300, 100), (50, 50), (977, 313)]:
        plan = P.select_tile_plan(w, h, cfg)
        assert plan.include_thumbnail == (plan.n_tiles > 1)
        assert plan.n_images == plan.n_tiles + int(plan.include_thumbnail)


def test_plan_rejects_bad_sizes():
    with pytest.raises(ValueError):
        P.select_tile_plan(0, 5, P.PreprocessConfig())
    with pytest.raises(ValueError):
        P.select_tile_plan(70000, 5, P.PreprocessConfig())


# ---------------------------------------------------------------------------
# tiling (reference tests/test_imgproc.py:181-236)

@settings(max_examples=40, deadline=None)
@given(h=st.integers(3, 40), w=st.integers(3, 40), fused=st.booleans(), split=st.booleans(),
       seed=st.integers(0, 2**31))
def test_tiling_matches_oracle_under_toggles(h, w, fused, split, seed):
    arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    cfg = P.PreprocessConfig(tile_edge=8, max_tiles=6, fused_transform=fused,
                             avoid_per_item_split=split)
    plan = P.select_tile_plan(w, h, cfg)
    got = P.tile_image(P.ImageBuffer.from_array(arr), plan, cfg)
    want = O.tiles_u8(arr, O.plan_float(w, h, 8, 6))
    assert len(got) == plan.n_images == len(want)
    for a, b in zip(got, want):
        assert np.array_equal(a.data, b)


def test_tiles_row_major_then_thumbnail():
    arr = np.random.default_rng(3).integers(0, 256, size=(30, 60, 3), dtype=np.uint8)
    img = P.ImageBuffer.from_array(arr)
    cfg = P.PreprocessConfig(tile_edge=8, max_tiles=6)
    plan = P.select_tile_plan(60, 30, cfg)
    assert (plan.rows, plan.cols) == (1, 2)
    tiles = P.tile_image(img, plan, cfg)
    assert len(tiles) == 3
    resized = P.resize_bilinear(img, plan.resized_width, plan.resized_height)
    assert np.array_equal(tiles[0].data, resized.data[:, :8])
    assert np.array_equal(tiles[1].data, resized.data[:, 8:])
    assert np.array_equal(tiles[2].data, P.resize_bilinear(img, 8, 8).data)


def test_shared_backing_views_when_split_avoided():
    arr = np.random.default_rng(4).integers(0, 256, size=(20, 40, 3), dtype=np.uint8)
    img = P.ImageBuffer.from_array(arr)
    plan = P.select_tile_plan(40, 20, P.PreprocessConfig(tile_edge=8, max_tiles=6))
    joined = P.tile_image(img, plan, P.PreprocessConfig(tile_edge=8, max_tiles=6,
                                                        avoid_per_item_split=True))
    assert all(t.data.base is not None for t in joined)
    assert len({id(t.data.base) for t in joined}) == 1
    split = P.tile_image(img, plan, P.PreprocessConfig(tile_edge=8, max_tiles=6))
    assert all(t.data.base is None for t in split)


def test_tile_image_golden(golden):
    data, meta = golden
    for name, h, w, c, e, mt, kind, seed in meta["tile_cases"]:
        arr = make_input(h, w, c, kind, seed)
        cfg = P.PreprocessConfig(tile_edge=e, max_tiles=mt)
        plan = P.select_tile_plan(w, h, cfg)
        tiles = P.tile_image(P.ImageBuffer.from_array(arr), plan, cfg)
        assert np.array_equal(np.stack([t.data for t in tiles]), data[f"tile_{name}_u8"]), name
        norm = P.normalize_tiles(tiles, P.PreprocessConfig(tile_edge=e, max_tiles=mt,
                                                           mean=IMAGENET_MEAN, std=IMAGENET_STD))
        assert np.array_equal(np.stack([t.data for t in norm]),
                              data[f"tile_{name}_f32_imagenet"]), name


# ---------------------------------------------------------------------------
# normalization (reference tests/test_imgproc.py:242-263)

def test_normalize_reference_values():
    arr = np.array([[[0, 128, 255]]], dtype=np.uint8)
    out = P.normalize(P.ImageBuffer.from_array(arr), P.PreprocessConfig())
    assert out.elem == FLOAT32
    want = (arr.astype(np.float32) / np.float32(255.0) - np.float32(0.5)) / np.float32(0.5)
    assert np.array_equal(out.data, want)


@settings(max_examples=40, deadline=None)
@given(seed=st.integers(0, 2**31))
def test_reduced_precision_within_relative_tolerance(seed):
    arr = np.random.default_rng(seed).integers(0, 256, size=(4, 4, 3), dtype=np.uint8)
    img = P.ImageBuffer.from_array(arr)
    full = P.normalize(img, P.PreprocessConfig())
    wide = P.normalize(img, P.PreprocessConfig(reduced_precision_normalize=True))
    assert wide.elem == FLOAT16_WIDE
    a, b = full.data.astype(np.float64), wide.data.astype(np.float64)
    nz = a != 0
    assert np.all(np.abs(b[nz] - a[nz]) <= 2.0**-7 * np.abs(a[nz]))
    assert np.all(b[~nz] == 0)
    assert np.array_equal(wide.data.view(np.uint16),
                          O.normalize(arr, (0.5,) * 3, (0.5,) * 3, True).view(np.uint16))


def test_normalize_rejects_float():
    with pytest.raises(ValueError):
        P.normalize(P.ImageBuffer(1, 1, 3, FLOAT32, np.zeros((1, 1, 3), np.float32)),
                    P.PreprocessConfig())


def test_normalize_tiles_shared_backing():
    arr = np.random.default_rng(2).integers(0, 256, size=(20, 40, 3), dtype=np.uint8)
    cfg = P.PreprocessConfig(tile_edge=8, max_tiles=6, avoid_per_item_split=True)
    tiles = P.tile_image(P.ImageBuffer.from_array(arr), P.select_tile_plan(40, 20, cfg), cfg)
    out = P.normalize_tiles(tiles, cfg)
    assert len({id(t.data.base) for t in out}) == 1
    assert P.normalize_tiles([], cfg) == []


# ---------------------------------------------------------------------------
# end-to-end preprocess (reference tests/test_imgproc.py:365-429)

def test_stage_timing_keys_exact():
    payload = png_payload(np.random.default_rng(0).integers(0, 256, (24, 36, 3), np.uint8))
    r = P.preprocess(payload, P.PreprocessConfig(tile_edge=8, max_tiles=4))
    assert set(r.stage_timings_ns) == {"decode", "plan", "resize", "tile", "normalize", "mask"}
    r2 = P.preprocess(payload, FAST)
    assert set(r2.stage_timings_ns) == {"decode", "plan", "resize", "tile", "normalize"}
    r3 = P.preprocess(payload, FAST, defer_normalize=True)
    assert set(r3.stage_timings_ns) == {"decode", "plan", "resize", "tile", "defer"}
    assert all(t.elem == UINT8 for t in r3.tiles)
    assert not r.deferred and r3.deferred


def test_preprocess_output_matches_plan():
    payload = png_payload(np.random.default_rng(1).integers(0, 256, (30, 60, 3), np.uint8))
    r = P.preprocess(payload, P.PreprocessConfig(tile_edge=8, max_tiles=6))
    assert len(r.tiles) == r.plan.n_images
    for t in r.tiles:
        assert (t.width, t.height) == (8, 8) and t.elem == FLOAT32


def test_preprocess_golden(golden):
    data, meta = golden
    for name, h, w, seed, kw, defer in meta["preprocess_cases"]:
        arr = np.random.default_rng(seed).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        kw = dict(kw)
        for k in ("mean", "std"):
            if k in kw:
                kw[k] = tuple(kw[k])
        r = P.preprocess(png_payload(arr), P.PreprocessConfig(**kw), defer_normalize=defer)
        case = meta["cases"][name]
        assert [r.plan.rows, r.plan.cols, r.plan.tile_edge, int(r.plan.include_thumbnail),
                r.plan.resized_width, r.plan.resized_height] == case["plan"]
        assert sorted(r.stage_timings_ns) == case["keys"]
        assert r.tiles[0].elem == case["elem"]
        got = np.stack([t.data for t in r.tiles])
        if got.dtype not in (np.uint8, np.float32):
            got = got.view(np.uint16)
        assert np.array_equal(got, data[f"pp_{name}"]), name


def test_deferred_tiles_equal_normalized_after_the_fact():
    payload = png_payload(np.random.default_rng(9).integers(0, 256, (16, 24, 3), np.uint8))
    cfg = P.PreprocessConfig(tile_edge=8, max_tiles=4)
    eager = P.preprocess(payload, cfg)
    lazy = P.preprocess(payload, cfg, defer_normalize=True)
    for a, b in zip(eager.tiles, lazy.tiles):
        assert np.array_equal(a.data, P.normalize(b, cfg).data)


@settings(max_examples=12, deadline=None)
@given(seed=st.integers(0, 2**31), toggles=st.tuples(*[st.booleans()] * 7))
def test_recipe_subsets_preserve_output(seed, toggles):
    fused, contig, once, reduced, simd, skipmask, split = toggles
    payload = png_payload(np.random.default_rng(seed).integers(0, 256, (20, 28, 3), np.uint8))
    ref = P.preprocess(payload, P.PreprocessConfig(tile_edge=8, max_tiles=4))
    got = P.preprocess(payload, P.PreprocessConfig(
        tile_edge=8, max_tiles=4, fused_transform=fused, contiguous_tensor_path=contig,
        decode_once=once, reduced_precision_normalize=reduced, simd_decode=simd,
        skip_pixel_mask=skipmask, avoid_per_item_split=split))
    for a, b in zip(ref.tiles, got.tiles):
        if b.elem == FLOAT32:
            assert np.array_equal(a.data, b.data)
        else:
            av, bv = a.data.astype(np.float64), b.data.astype(np.float64)
            nz = av != 0
            assert np.all(np.abs(bv[nz] - av[nz]) <= 2.0**-7 * np.abs(av[nz]))
            assert np.all(bv[~nz] == 0)


# ---------------------------------------------------------------------------
# token expansion (reference tests/test_tokenizer.py:173-283)

@pytest.fixture(scope="module")
def vocab(golden):
    _, meta = golden
    return P.tokenizer.SpecialVocab(P.SpecialIds(**meta["specials"]))


def test_expand_no_markers_is_identity(vocab):
    ids = [2, 50, 60, 3]
    seq = P.expand_image_placeholders(ids, [], 64, vocab)
    assert seq.ids == ids and seq.image_spans == []


def test_expand_counts_and_span(vocab):
    seq = P.expand_image_placeholders([2, 4, 3], [2], 64, vocab)
    assert seq.image_spans == [(1, 128)]
    assert seq.ids[1:129] == [5] * 128 and len(seq.ids) == 3 - 1 + 128
    assert seq.supervision_mask == [False] * len(seq.ids)


def test_expand_marker_count_mismatch(vocab):
    with pytest.raises(P.ExpansionError):
        P.expand_image_placeholders([2, 4, 3], [1, 2], 64, vocab)
    with pytest.raises(P.ExpansionError):
        P.expand_image_placeholders([2, 4, 3], [], 64, vocab)


def test_expand_requires_assistant(vocab):
    with pytest.raises(P.MalformedSequenceError):
        P.expand_image_placeholders([2, 4, 7], [1], 4, vocab)


def test_expand_golden(golden, vocab):
    data, meta = golden
    for i, case in enumerate(meta["expand_cases"]):
        seq = P.expand_image_placeholders(case["ids"], case["counts"], case["tpt"], vocab)
        assert seq.ids == data[f"expand_{i}_ids"].tolist()
        assert [list(s) for s in seq.image_spans] == [list(s) for s in case["spans"]]
        assert seq.first_assistant_index == case["first"]
        full = P.build_supervision_mask(seq, vocab)
        assert np.array_equal(np.asarray(full.supervision_mask, np.uint8),
                              data[f"expand_{i}_mask"])
        both = P.expand_and_mask(case["ids"], case["counts"], case["tpt"], vocab)
        assert both.supervision_mask == full.supervision_mask


def test_mask_bad_index_raises(vocab):
    with pytest.raises(P.MalformedSequenceError):
        P.build_supervision_mask(P.TokenSequence([1, 2, 3], 7, [], [False] * 3), vocab)


def test_validate_rejects_span_over_text(vocab):
    seq = P.TokenSequence([2, 50, 3], 2, [(0, 2)], [False] * 3)
    with pytest.raises(P.MalformedSequenceError):
        seq.validate(vocab)


# ---------------------------------------------------------------------------
# contract (reference tests/test_tokenred.py:182-200, tests/test_backend.py:56-112)

def test_assemble_contract_with_device_plans(vocab):
    cfg = P.PreprocessConfig(tile_edge=448, max_tiles=12)
    tr = P.TokenReductionConfig(patch_edge=14, r=2)
    for w, h in [(1920, 1080), (640, 480), (448, 448), (1000, 3000)]:
        plan = P.select_tile_plan(w, h, cfg)
        seq = P.expand_and_mask([2, 4, 77, 3], [plan.n_images],
                                P.tokens_per_tile(448, 14, 2), vocab)
        assert P.assemble(seq, plan, tr).n_visual == plan.n_images * 256
    plan = P.select_tile_plan(1920, 1080, cfg)
    bad = P.expand_and_mask([2, 4, 3], [plan.n_images + 1], 256, vocab)
    with pytest.raises(P.AssemblyError):
        P.assemble(bad, plan, tr)


# ---------------------------------------------------------------------------
# pixel_unshuffle (reference tests/test_tokenred.py:19-74)

def test_pixel_unshuffle_golden(golden):
    data, meta = golden
    for i, (h, w, d, r, dt, seed) in enumerate(meta["unshuffle_cases"]):
        flat = np.random.default_rng(seed).standard_normal(h * w * d).astype(dt)
        out = P.pixel_unshuffle(P.PatchGrid(h, w, d, flat), r)
        assert [out.h, out.w, out.d] == meta["unshuffle_shapes"][i]
        assert out.data.dtype == flat.dtype
        assert np.array_equal(out.data, data[f"unshuffle_{i}"])


@settings(max_examples=30, deadline=None)
@given(oh=st.integers(1, 9), ow=st.integers(1, 9), d=st.integers(1, 40), r=st.integers(1, 4),
       dt=st.sampled_from(["float32", "float16", "int8", "float64"]), seed=st.integers(0, 2**31))
def test_pixel_unshuffle_is_the_oracle_permutation(oh, ow, d, r, dt, seed):
    h, w = oh * r, ow * r
    flat = (np.random.default_rng(seed).standard_normal(h * w * d) * 50).astype(dt)
    out = P.pixel_unshuffle(P.PatchGrid(h, w, d, flat), r)
    want = O.pixel_unshuffle(flat.reshape(h, w, d), r)
    assert np.array_equal(out.as_array(), want)
    assert np.array_equal(np.sort(out.data.view(np.uint8)), np.sort(flat.view(np.uint8)))


def test_pixel_unshuffle_errors_and_identity():
    g = P.PatchGrid(4, 6, 2, np.arange(48, dtype=np.float32))
    assert P.pixel_unshuffle(g, 1).data is g.data
    with pytest.raises(P.DomainError):
        P.pixel_unshuffle(g, 0)
    with pytest.raises(P.ShapeError):
        P.pixel_unshuffle(g, 4)
    with pytest.raises(P.ShapeError):
        P.PatchGrid(2, 2, 2, np.zeros(7, np.float32))


def test_pixel_unshuffle_device_tensor():
    import torch

    t = torch.randn(32, 32, 1024, dtype=torch.bfloat16, device="cuda")
    out = P.pixel_unshuffle_tensor(t, 2)
    want = t.reshape(16, 2, 16, 2, 1024).permute(0, 2, 1, 3, 4).reshape(16, 16, 4096)
    assert torch.equal(out, want)
