"""Parity of the CUDA path (through the C-ABI) with the oracle and the
reference's golden vectors.  Runs on the B200 box (`-m gpu`)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_data import IMAGENET_MEAN, IMAGENET_STD, make_input
from oracle import tileprep_oracle as O
from paper_2603_16987_b200 import _lib
from paper_2603_16987_b200.engine import (
    TilePreprocessor,
    empty_packed,
    pack_images,
    synth_packed,
)
from paper_2603_16987_b200.imgproc import PreprocessConfig

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _plans_on_gpu(wh: np.ndarray, tile_edge: int, max_tiles: int):
    n = len(wh)
    d_wh = torch.from_numpy(np.ascontiguousarray(wh, dtype=np.int32)).to(DEV)
    plan = torch.empty((n, 6), dtype=torch.int32, device=DEV)
    n_img = torch.empty((n,), dtype=torch.int32, device=DEV)
    off = torch.empty((n + 1,), dtype=torch.int32, device=DEV)
    _lib.call("tp_plan", _lib.ptr(d_wh), n, tile_edge, max_tiles, _lib.ptr(plan),
              _lib.ptr(n_img), _lib.ptr(off), torch.cuda.current_stream().cuda_stream)
    return plan.cpu().numpy(), n_img.cpu().numpy(), off.cpu().numpy()


# ---------------------------------------------------------------------------
# K1 planner

def test_plan_matches_golden(golden):
    data, _ = golden
    pin, want = data["plan_in"], data["plan_out"]
    for mt in np.unique(pin[:, 2]):
        sel = pin[:, 2] == mt
        plan, n_img, off = _plans_on_gpu(pin[sel, :2], 32, int(mt))
        assert np.array_equal(plan, want[sel]), int(mt)
        assert np.array_equal(n_img, want[sel, 0] * want[sel, 1] + want[sel, 3])
        assert off[0] == 0 and np.array_equal(np.diff(off), n_img)


def test_plan_dense_square_vs_oracle():
    w, h = np.meshgrid(np.arange(1, 301), np.arange(1, 301))
    wh = np.stack([w.ravel(), h.ravel()], axis=1)
    for mt in (1, 2, 6, 12, 40):
        plan, _, _ = _plans_on_gpu(wh, 448, mt)
        for i in range(0, len(wh), 97):
            assert tuple(plan[i]) == O.plan_float(int(wh[i, 0]), int(wh[i, 1]), 448, mt)
        if mt == 12:  # full check of the config value
            want = np.array([O.plan_int(int(a), int(b), 448, 12) for a, b in wh[::7]])
            assert np.array_equal(plan[::7], want)


def test_plan_invalid_size_flags_batch():
    plan, n_img, off = _plans_on_gpu(np.array([[10, 10], [0, 5], [20, 10]]), 16, 12)
    assert off[-1] == -1
    assert n_img[1] == 0


def test_plan_large_batch_offsets():
    rng = np.random.default_rng(1)
    wh = rng.integers(1, 4097, size=(5000, 2))
    plan, n_img, off = _plans_on_gpu(wh, 448, 12)
    assert off[-1] == n_img.sum() and np.array_equal(np.cumsum(n_img), off[1:])
    for i in range(0, 5000, 250):
        assert tuple(plan[i]) == O.plan_int(int(wh[i, 0]), int(wh[i, 1]), 448, 12)


# ---------------------------------------------------------------------------
# K2 fused tiling (+ normalize through the LUT)

def _run_engine(arrs, cfg, layout="NCHW", emit_uint8=True, normalize=True):
    packed = pack_images(arrs).to(DEV)
    prep = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=emit_uint8, normalize=normalize)
    out = prep(packed)
    torch.cuda.synchronize()
    T = out.num_tiles()
    pv = out.pixel_values[:T].cpu() if out.pixel_values is not None else None
    u8 = out.pixel_u8[:T].cpu().numpy() if out.pixel_u8 is not None else None
    return out, pv, u8


def test_tiles_match_golden_all_layouts(golden):
    data, meta = golden
    for name, h, w, c, e, mt, kind, seed in meta["tile_cases"]:
        arr = make_input(h, w, c, kind, seed)
        want_u8 = data[f"tile_{name}_u8"]
        cfg = PreprocessConfig(tile_edge=e, max_tiles=mt, mean=IMAGENET_MEAN, std=IMAGENET_STD)
        out, pv, u8 = _run_engine([arr], cfg, layout="NHWC")
        assert np.array_equal(out.plans.plan.cpu().numpy()[0], data[f"tile_{name}_plan"]), name
        assert np.array_equal(u8, want_u8), name
        assert np.array_equal(pv.numpy(), data[f"tile_{name}_f32_imagenet"]), name
        cfgb = PreprocessConfig(tile_edge=e, max_tiles=mt, reduced_precision_normalize=True)
        _, pvb, _ = _run_engine([arr], cfgb, layout="NCHW", emit_uint8=False)
        want_b = data[f"tile_{name}_bf16_half_bits"].transpose(0, 3, 1, 2)
        assert np.array_equal(pvb.view(torch.int16).numpy().view(np.uint16), want_b), name


def test_tiles_batch_mixed_sizes_vs_oracle():
    rng = np.random.default_rng(5)
    arrs = []
    for i in range(12):
        h, w = int(rng.integers(1, 120)), int(rng.integers(1, 120))
        arrs.append(make_input(h, w, 3, "random" if i % 2 else "smooth", 100 + i))
    cfg = PreprocessConfig(tile_edge=24, max_tiles=9)
    out, pv, u8 = _run_engine(arrs, cfg)
    off = out.plans.tile_off.cpu().numpy()
    lut = O.lut((0.5,) * 3, (0.5,) * 3, 3, False)
    for k, a in enumerate(arrs):
        plan = O.plan_float(a.shape[1], a.shape[0], 24, 9)
        want = O.tiles_u8(a, plan)
        assert np.array_equal(u8[off[k]: off[k + 1]], want), k
        norm = pv[off[k]: off[k + 1]].numpy()  # NCHW
        assert np.array_equal(norm, O.normalize(want, (0.5,) * 3, (0.5,) * 3, False)
                              .transpose(0, 3, 1, 2)), k
    assert np.array_equal(lut[:, u8[..., 0].ravel()][0], pv[:, 0].numpy().ravel())


def test_tiles_grayscale_channel():
    arr = make_input(40, 70, 1, "random", 3)
    cfg = PreprocessConfig(tile_edge=16, max_tiles=6, mean=IMAGENET_MEAN, std=IMAGENET_STD)
    _, pv, u8 = _run_engine([arr], cfg, layout="NHWC")
    plan = O.plan_float(70, 40, 16, 6)
    want = O.tiles_u8(arr, plan)
    assert np.array_equal(u8, want)
    assert np.array_equal(pv.numpy(), O.normalize(want, IMAGENET_MEAN, IMAGENET_STD, False))


@pytest.mark.parametrize("w,h,e,kind", [(1920, 1080, 448, "random"), (1920, 1080, 512, "smooth"),
                                        (3840, 2160, 448, "random"), (640, 480, 448, "smooth"),
                                        (333, 517, 448, "random")])
def test_full_size_bit_exact(w, h, e, kind):
    arr = make_input(h, w, 3, kind, w * 7 + h)
    cfg = PreprocessConfig(tile_edge=e, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    _, pv, u8 = _run_engine([arr], cfg)
    plan = O.plan_float(w, h, e, 12)
    want = O.tiles_u8(arr, plan)
    assert np.array_equal(u8, want)
    wb = O.normalize(want, IMAGENET_MEAN, IMAGENET_STD, True).transpose(0, 3, 1, 2)
    assert np.array_equal(pv.view(torch.int16).numpy().view(np.uint16), wb.view(np.uint16))


def test_capacity_guard_never_writes_past_buffer():
    arrs = [make_input(100, 200, 3, "random", 1)]  # 1x2 + thumb = 3 tiles
    cfg = PreprocessConfig(tile_edge=16, max_tiles=12)
    packed = pack_images(arrs).to(DEV)
    prep = TilePreprocessor(cfg, DEV, emit_uint8=True)
    plans = prep.plan(packed)
    guard = torch.full((3, 16, 16, 3), 7, dtype=torch.uint8, device=DEV)
    pv = torch.zeros((2, 3, 16, 16), dtype=torch.float32, device=DEV)
    prep.tile(packed, plans, pv, guard[:2])
    torch.cuda.synchronize()
    assert int(guard[2].min()) == 7 and int(guard[2].max()) == 7


def test_resize_matches_golden(golden):
    data, meta = golden
    stream = torch.cuda.current_stream().cuda_stream
    for i, (h, w, c, oh, ow, seed, kind) in enumerate(meta["resize_cases"]):
        arr = make_input(h, w, c, kind, seed)
        src = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(DEV)
        dst = torch.empty((oh, ow, arr.shape[2]), dtype=torch.uint8, device=DEV)
        _lib.call("tp_resize", _lib.ptr(src), arr.shape[1], arr.shape[0], arr.shape[2], ow, oh,
                  _lib.ptr(dst), stream)
        assert np.array_equal(dst.cpu().numpy(), data[f"resize_{i}"]), i


def test_lut_matches_golden(golden):
    data, _ = golden
    from paper_2603_16987_b200.runtime import normalize_lut

    d = torch.device(DEV)
    for tag, mean, std in (("half", (0.5,) * 3, (0.5,) * 3),
                           ("imagenet", IMAGENET_MEAN, IMAGENET_STD)):
        f = normalize_lut(mean, std, 3, _lib.TP_DTYPE_F32, d).cpu().numpy()
        assert np.array_equal(f, data[f"lut_{tag}_f32"])
        b = normalize_lut(mean, std, 3, _lib.TP_DTYPE_BF16, d).cpu().view(torch.int16).numpy()
        assert np.array_equal(b.view(np.uint16), data[f"lut_{tag}_bf16"])
        g = normalize_lut(mean, std, 1, _lib.TP_DTYPE_F32, d).cpu().numpy()
        assert np.array_equal(g, data[f"lut_{tag}_f32_gray"])


def test_normalize_kernel_layouts():
    from paper_2603_16987_b200.runtime import normalize_lut

    d = torch.device(DEV)
    rng = np.random.default_rng(9)
    u8 = rng.integers(0, 256, size=(5, 7, 11, 3), dtype=np.uint8)
    lut = normalize_lut(IMAGENET_MEAN, IMAGENET_STD, 3, _lib.TP_DTYPE_F32, d)
    src = torch.from_numpy(u8.reshape(-1)).to(DEV)
    want = O.normalize(u8, IMAGENET_MEAN, IMAGENET_STD, False)
    for layout, shape, ref in ((_lib.TP_LAYOUT_NHWC, u8.shape, want),
                               (_lib.TP_LAYOUT_NCHW, (5, 3, 7, 11), want.transpose(0, 3, 1, 2))):
        out = torch.empty(shape, dtype=torch.float32, device=DEV)
        _lib.call("tp_normalize", _lib.ptr(src), 5, 77, 3, _lib.ptr(lut), _lib.TP_DTYPE_F32,
                  layout, _lib.ptr(out), torch.cuda.current_stream().cuda_stream)
        assert np.array_equal(out.cpu().numpy(), ref)


# ---------------------------------------------------------------------------
# synthetic inputs: device generator == CPU twin

@pytest.mark.parametrize("kind", [0, 1])
def test_synth_matches_cpu_twin(kind):
    wh = np.array([[37, 11], [64, 48], [5, 3], [1920, 2]], dtype=np.int32)
    packed = synth_packed(wh, 3, DEV, seed=20260817, kind=kind)
    buf = packed.data.cpu().numpy()
    for k, (w, h) in enumerate(wh):
        off = packed.offsets_host[k]
        got = buf[off: off + w * h * 3].reshape(h, w, 3)
        assert np.array_equal(got, O.synth_image(20260817, k, int(w), int(h), 3, kind)), k


def test_c4_style_batch_sample_bit_exact():
    """A slice of the 8192-image mixed-aspect sweep (C4) checked image by image."""
    from paper_2603_16987_b200.workloads import c4_shapes

    wh = c4_shapes(48, start=0)
    packed = synth_packed(wh, 3, DEV, seed=20261018, kind=0)
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    prep = TilePreprocessor(cfg, DEV, emit_uint8=True)
    out = prep(packed)
    torch.cuda.synchronize()
    off = out.plans.tile_off.cpu().numpy()
    for k in range(0, 48, 5):
        w, h = (int(v) for v in wh[k])
        arr = O.synth_image(20261018, k, w, h, 3, 0)
        want = O.tiles_u8(arr, O.plan_float(w, h, 448, 12))
        got = out.pixel_u8[off[k]: off[k + 1]].cpu().numpy()
        assert np.array_equal(got, want), k
    # normalized output is the LUT image of the uint8 tiles for the whole batch
    T = out.num_tiles()
    lut = torch.from_numpy(O.lut(IMAGENET_MEAN, IMAGENET_STD, 3, True).view(np.int16)).to(DEV)
    u8 = out.pixel_u8[:T].long()
    for c in range(3):
        want_c = lut[c][u8[..., c]]
        got_c = out.pixel_values[:T, c].view(torch.int16)
        assert torch.equal(want_c, got_c)


# ---------------------------------------------------------------------------
# fast kernel (fp32 + exactness window) == exact fp64 kernel, at full size

def _fast_vs_exact(wh, seed, kind, cfg, layout="NCHW"):
    packed = synth_packed(wh, 3, DEV, seed=seed, kind=kind)
    outs = []
    for algo in ("fast", "exact"):
        prep = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=True, algo=algo)
        outs.append(prep(packed))
    torch.cuda.synchronize()
    T = outs[0].num_tiles()
    assert T == outs[1].num_tiles()
    assert torch.equal(outs[0].pixel_u8[:T], outs[1].pixel_u8[:T])
    assert torch.equal(outs[0].pixel_values[:T].view(torch.uint8),
                       outs[1].pixel_values[:T].view(torch.uint8))
    return T


@pytest.mark.parametrize("kind", [0, 1])
def test_fast_equals_exact_c4_slice(kind):
    from paper_2603_16987_b200.workloads import c4_shapes

    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    assert _fast_vs_exact(c4_shapes(256, start=512 * kind), 20261018 + kind, kind, cfg) > 256


@pytest.mark.parametrize("e,layout", [(512, "NCHW"), (448, "NHWC"), (7, "NCHW"), (33, "NHWC")])
def test_fast_equals_exact_edges(e, layout):
    rng = np.random.default_rng(e)
    wh = np.stack([rng.integers(1, 3000, 40), rng.integers(1, 3000, 40)], axis=1)
    cfg = PreprocessConfig(tile_edge=e, max_tiles=12)
    _fast_vs_exact(wh, 99, 0, cfg, layout)
    _fast_vs_exact(wh, 98, 1, cfg, layout)


def test_fast_integer_scale_ties():
    # integer down/up-scales put many values exactly on k + 0.5: all go through the fallback
    cfg = PreprocessConfig(tile_edge=64, max_tiles=4)
    wh = np.array([[128, 128], [256, 128], [32, 32], [64, 128], [96, 96]])
    for kind in (0, 1):
        _fast_vs_exact(wh, 5, kind, cfg)
        packed = synth_packed(wh, 3, DEV, seed=5, kind=kind)
        prep = TilePreprocessor(cfg, DEV, emit_uint8=True)
        out = prep(packed)
        torch.cuda.synchronize()
        off = out.plans.tile_off.cpu().numpy()
        for k, (w, h) in enumerate(wh):
            arr = O.synth_image(5, k, int(w), int(h), 3, kind)
            want = O.tiles_u8(arr, O.plan_float(int(w), int(h), 64, 4))
            assert np.array_equal(out.pixel_u8[off[k]: off[k + 1]].cpu().numpy(), want)


# ---------------------------------------------------------------------------
# affine normalize (TP_TILE_NORM_AFFINE): one fma per value instead of the table,
# taken when no uint8 tiles are requested; must give the table's exact bits

CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)


def _bf16_rne(x: np.ndarray) -> np.ndarray:
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


@pytest.mark.parametrize("mean,std", [(IMAGENET_MEAN, IMAGENET_STD), ((0.5,) * 3, (0.5,) * 3),
                                      (CLIP_MEAN, CLIP_STD)])
def test_affine_block_reproduces_table(mean, std):
    from paper_2603_16987_b200.runtime import normalize_tables

    table, ok = normalize_tables(mean, std, 3, _lib.TP_DTYPE_BF16, torch.device(DEV))
    assert ok
    want = O.lut(mean, std, 3, True).view(np.uint16)
    assert np.array_equal(table.cpu().view(torch.int16).numpy().view(np.uint16), want)
    # the constants after the table: fma(v, a, b) (exact in float64, rounded once to fp32)
    # must round to the table entry for every v
    lib = _lib.load()
    off = lib.tp_lut_table_bytes(3, _lib.TP_DTYPE_BF16)
    full = torch.empty(0, dtype=torch.uint8, device=DEV).set_(table.untyped_storage())
    assert full.numel() == lib.tp_lut_bytes(3, _lib.TP_DTYPE_BF16)
    block = full[off: off + 32].clone()
    ab = block.cpu().numpy().view(np.float32)
    v = np.arange(256, dtype=np.float64)
    for c in range(3):
        y = (v * np.float64(ab[c]) + np.float64(ab[4 + c])).astype(np.float32)
        assert np.array_equal(_bf16_rne(y), want[c]), c


def _pixels(cfg, packed, layout, emit_uint8):
    prep = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=emit_uint8)
    out = prep(packed)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("layout", ["NCHW", "NHWC"])
@pytest.mark.parametrize("kind", [0, 1])
def test_affine_normalize_equals_table_c4_slice(layout, kind):
    from paper_2603_16987_b200.workloads import c4_shapes

    wh = c4_shapes(192, start=2048 + 192 * kind)
    packed = synth_packed(wh, 3, DEV, seed=7 + kind, kind=kind)
    for mean, std in ((IMAGENET_MEAN, IMAGENET_STD), (CLIP_MEAN, CLIP_STD)):
        cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=mean, std=std,
                               reduced_precision_normalize=True)
        lut_path = _pixels(cfg, packed, layout, True)     # uint8 tiles: table lookups
        aff_path = _pixels(cfg, packed, layout, False)    # affine fma
        T = lut_path.num_tiles()
        assert T == aff_path.num_tiles() > 192
        assert torch.equal(lut_path.pixel_values[:T].view(torch.int16),
                           aff_path.pixel_values[:T].view(torch.int16))


@pytest.mark.parametrize("w,h,c", [(1920, 1080, 3), (333, 517, 3), (700, 300, 1)])
def test_affine_normalize_vs_oracle(w, h, c):
    arr = make_input(h, w, c, "random", w + h)
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    _, pv, _ = _run_engine([arr], cfg, layout="NCHW", emit_uint8=False)
    want = O.tiles_u8(arr, O.plan_float(w, h, 448, 12))
    wb = O.normalize(want, IMAGENET_MEAN, IMAGENET_STD, True).transpose(0, 3, 1, 2)
    assert np.array_equal(pv.view(torch.int16).numpy().view(np.uint16), wb.view(np.uint16))


# ---------------------------------------------------------------------------
# K3 at C5 scale: 1024 ragged prompts, counts straight from K1's n_images

def test_c5_expansion_batch_bit_exact(golden):
    from paper_2603_16987_b200.tokenizer import PlaceholderExpander, SpecialIds, SpecialVocab
    from paper_2603_16987_b200.workloads import c4_shapes

    _, meta = golden
    sp = meta["specials"]
    vocab = SpecialVocab(SpecialIds(**sp))
    prompts = meta["prompt_ids"]  # tokenized by the reference: <|user|><|image|>prompt<|assistant|>
    n = 1024
    wh = c4_shapes(n, start=4096)
    d_wh = torch.from_numpy(wh).to(DEV)
    plan = torch.empty((n, 6), dtype=torch.int32, device=DEV)
    n_img = torch.empty((n,), dtype=torch.int32, device=DEV)
    off = torch.empty((n + 1,), dtype=torch.int32, device=DEV)
    _lib.call("tp_plan", _lib.ptr(d_wh), n, 448, 12, _lib.ptr(plan), _lib.ptr(n_img),
              _lib.ptr(off), torch.cuda.current_stream().cuda_stream)
    seqs = [prompts[i % len(prompts)] for i in range(n)]
    flat = np.concatenate([np.asarray(s, np.int32) for s in seqs])
    seq_off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])]).astype(np.int32)
    cap = int(len(flat) + n * 13 * 256)
    exp = PlaceholderExpander(vocab, 256, DEV)
    res = exp(torch.from_numpy(flat).to(DEV), torch.from_numpy(seq_off).to(DEV), n_img,
              torch.arange(n + 1, dtype=torch.int32, device=DEV), cap)
    torch.cuda.synchronize()
    counts = n_img.cpu().numpy()
    assert int(res.err.cpu().numpy().max()) == 0
    oo = res.out_off.cpu().numpy()
    ids = res.ids.cpu().numpy()
    mask = res.mask.cpu().numpy()
    spans = res.spans.cpu().numpy()
    first = res.first_assistant.cpu().numpy()
    for s in range(n):
        want, wspans, t = O.expand(seqs[s], [int(counts[s])], 256, sp["image_marker"],
                                   sp["image_context"], sp["assistant_header"])
        assert ids[oo[s]: oo[s + 1]].tolist() == want, s
        assert [tuple(spans[s])] == [tuple(x) for x in wspans]
        assert first[s] == t
        assert np.array_equal(mask[oo[s]: oo[s + 1]].astype(bool),
                              O.supervision_mask(want, t, sp["assistant_header"]))
    # the contract the consumer checks (backend.assemble): spans carry the plan's tokens
    assert int(spans[:, 1].sum()) == int(counts.sum()) * 256


def test_expand_errors_and_capacity_flags():
    from paper_2603_16987_b200.tokenizer import PlaceholderExpander, SpecialIds, SpecialVocab

    vocab = SpecialVocab(SpecialIds(0, 1, 2, 3, 4, 5, 6))
    exp = PlaceholderExpander(vocab, 4, DEV)
    ids = torch.tensor([2, 4, 3, 2, 4, 4, 3, 2, 9, 9], dtype=torch.int32, device=DEV)
    seq_off = torch.tensor([0, 3, 7, 10], dtype=torch.int32, device=DEV)
    counts = torch.tensor([2, 1, 1], dtype=torch.int32, device=DEV)
    count_off = torch.tensor([0, 1, 2, 3], dtype=torch.int32, device=DEV)  # seq 1 short a count
    res = exp(ids, seq_off, counts, count_off, capacity=100)
    torch.cuda.synchronize()
    err = res.err.cpu().tolist()
    assert err[0] == 0
    assert err[1] & _lib.TP_EXPAND_ERR_MARKER_COUNT
    assert err[2] & _lib.TP_EXPAND_ERR_NO_ASSISTANT
    oo = res.out_off.cpu().tolist()
    assert oo[1] - oo[0] == 3 - 1 + 8 and oo[3] == oo[1]  # errored sequences take no space
    small = exp(ids[:3], seq_off[:2], counts[:1], count_off[:2], capacity=5)
    torch.cuda.synchronize()
    assert int(small.out_off[-1]) == -1  # capacity overflow is flagged, nothing written


# ---------------------------------------------------------------------------
# geometry extremes: rows wider than a shared-memory stage (column chunks), very tall
# images, more tiles per image than the per-image tile cache, large tile edges

@pytest.mark.parametrize("w,h,e,mt", [(30000, 40, 448, 12), (40, 30000, 448, 12),
                                      (9000, 700, 256, 40), (1500, 1500, 1024, 4),
                                      (2000, 1200, 96, 64)])
def test_fast_equals_exact_geometry_extremes(w, h, e, mt):
    cfg = PreprocessConfig(tile_edge=e, max_tiles=mt, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    wh = np.array([[w, h], [h, w]])
    T = _fast_vs_exact(wh, 31, 0, cfg)
    assert T >= 2
    T = _fast_vs_exact(wh, 32, 1, cfg, layout="NHWC")


def test_many_tiles_per_image_vs_oracle():
    # 17+ tiles per image exceeds the producer's per-image tile cache (16)
    arr = make_input(300, 1700, 3, "random", 77)
    cfg = PreprocessConfig(tile_edge=64, max_tiles=40)
    _, pv, u8 = _run_engine([arr], cfg)
    plan = O.plan_float(1700, 300, 64, 40)
    assert plan[0] * plan[1] + plan[3] > 16
    assert np.array_equal(u8, O.tiles_u8(arr, plan))


# ---------------------------------------------------------------------------
# randomized configurations: every dtype/layout/side-output/normalize-form combination
# on random sizes and tile edges, checked image by image against the oracle

def test_randomized_configs_vs_oracle():
    rng = np.random.default_rng(2026)
    means = [((0.5,) * 3, (0.5,) * 3), (IMAGENET_MEAN, IMAGENET_STD),
             ((0.48145466, 0.4578275, 0.40821073), (0.26862954, 0.26130258, 0.27577711))]
    for case in range(40):
        c = 3 if case % 5 else 1
        n = int(rng.integers(1, 6))
        e = int(rng.choice([7, 16, 33, 64, 100, 448]))
        mt = int(rng.integers(1, 14))
        arrs = [make_input(int(rng.integers(1, 300)), int(rng.integers(1, 300)), c,
                           "random" if rng.random() < 0.5 else "smooth", 1000 * case + i)
                for i in range(n)]
        mean, std = means[case % 3]
        bf16 = bool(case % 2)
        cfg = PreprocessConfig(tile_edge=e, max_tiles=mt, mean=mean[:c], std=std[:c],
                               reduced_precision_normalize=bf16)
        layout = "NCHW" if case % 4 < 2 else "NHWC"
        emit = bool((case // 2) % 2)
        out, pv, u8 = _run_engine(arrs, cfg, layout=layout, emit_uint8=emit)
        off = out.plans.tile_off.cpu().numpy()
        for k, a in enumerate(arrs):
            plan = O.plan_float(a.shape[1], a.shape[0], e, mt)
            want = O.tiles_u8(a, plan)
            if emit:
                assert np.array_equal(u8[off[k]: off[k + 1]], want), (case, k)
            wn = O.normalize(want, mean[:c], std[:c], bf16)
            got = pv[off[k]: off[k + 1]]
            if layout == "NCHW":
                wn = wn.transpose(0, 3, 1, 2)
            if bf16:
                assert np.array_equal(got.view(torch.int16).numpy().view(np.uint16),
                                      wn.view(np.uint16)), (case, k)
            else:
                assert np.array_equal(got.numpy(), wn), (case, k)


def test_plan_after_kernel_steady_state():
    # the bench loop: plan (programmatic dependent of the previous tile) -> tile -> ...
    from paper_2603_16987_b200.workloads import c4_shapes

    wh = c4_shapes(64, start=300)
    packed = synth_packed(wh, 3, DEV, seed=9, kind=0)
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    prep = TilePreprocessor(cfg, DEV)
    ref = prep(packed)
    torch.cuda.synchronize()
    want_plan = ref.plans.plan.clone()
    want_pv = ref.pixel_values.clone()
    T = ref.num_tiles()
    s = torch.cuda.Stream(DEV)
    with torch.cuda.stream(s):
        for _ in range(20):
            prep.plan(packed, ref.plans, s, after_kernel=True)
            prep.tile(packed, ref.plans, ref.pixel_values, None, s, after_plan=True)
    torch.cuda.synchronize()
    assert torch.equal(ref.plans.plan, want_plan)
    assert torch.equal(ref.pixel_values[:T].view(torch.int16), want_pv[:T].view(torch.int16))
