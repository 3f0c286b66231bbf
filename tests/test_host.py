"""Host-side logic that needs no GPU: the C-ABI library's exports and argument
checks, the drop-in types' validation, decode error reporting, contract
arithmetic, workload byte model and batch packing."""

from __future__ import annotations

import io
import re
import subprocess

import numpy as np
import pytest
import torch
from PIL import Image

import paper_2603_16987_b200 as P
from paper_2603_16987_b200 import _lib
from paper_2603_16987_b200.dtypes import FLOAT16_WIDE, FLOAT32, UINT8
from paper_2603_16987_b200.engine import layout_offsets, pack_images
from paper_2603_16987_b200.workloads import c1, c2, c3, c4_shapes, plan_rows_cols, workload_bytes

HEADER = _lib.LIB_PATH.parent.parent / "include" / "tileprep.h"


# ---------------------------------------------------------------------------
# C-ABI library

def _declared_symbols() -> list[str]:
    return re.findall(r"^TP_API\s+[\w\s\*]+?\b(tp_\w+)\(", HEADER.read_text(), flags=re.M)


def test_every_declared_symbol_is_exported_and_typed():
    names = _declared_symbols()
    assert len(names) >= 12
    lib = _lib.load()
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert set(_lib.SIGNATURES) == set(names)


def test_header_constants_match_binding():
    defs = dict(re.findall(r"#define\s+(TP_\w+)\s+(-?\d+)", HEADER.read_text()))
    for k, v in defs.items():
        if hasattr(_lib, k):
            assert getattr(_lib, k) == int(v), k
    assert _lib.load().tp_abi_version() == int(defs["TP_ABI_VERSION"])


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_argument_errors_return_codes_without_touching_the_gpu():
    lib = _lib.load()
    assert lib.tp_plan(None, 1, 448, 0, None, None, None, None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert "max_tiles" in _lib.last_error()
    assert lib.tp_plan(None, 1, 448, 5000, None, None, None, None) == _lib.TP_ERR_UNSUPPORTED
    assert lib.tp_tile(None, None, None, 1, 2, None, None, 448, None, 1, 0, None, None, 1,
                       None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert "channels" in _lib.last_error()
    assert lib.tp_tile_ex(None, None, None, 1, 3, None, None, 448, None, 1, 0, None, None, 1, 9,
                          None) == _lib.TP_ERR_INVALID_ARGUMENT
    zero = _lib.f32_array([0.5, 0.5, 0.5])
    bad = _lib.f32_array([0.5, 0.0, 0.5])
    assert lib.tp_build_lut(3, zero, bad, 1, None, None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert lib.tp_expand(None, None, -1, None, None, 4, 1, 2, 3, 1, None, 0, None, None, None,
                         None, None, None, None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert lib.tp_supervision_mask(None, 3, 9, 3, None, None) == _lib.TP_ERR_INVALID_ARGUMENT
    # unknown algo flag bits, tokenizer and norm-table argument checks
    assert lib.tp_tile_ex(None, None, None, 1, 3, None, None, 448, None, 1, 0, None, None, 1,
                          1 << 12, None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert lib.tp_tokenize(None, None, None, 1, 10, None, None, None, None, 0,
                           None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert lib.tp_tokenize_workspace_bytes(-1, 1) == -1
    assert lib.tp_vocab_table_bytes(-1) == -1
    assert lib.tp_build_norm(3, zero, bad, 2, None, None, None) == _lib.TP_ERR_INVALID_ARGUMENT
    assert lib.tp_lut_bytes(3, _lib.TP_DTYPE_BF16) == lib.tp_lut_table_bytes(3, 2) + 32
    assert lib.tp_lut_table_bytes(3, _lib.TP_DTYPE_F32) == 3 * 256 * 4
    with pytest.raises(ValueError):
        _lib.check(_lib.TP_ERR_INVALID_ARGUMENT, "x")
    with pytest.raises(P.DeviceError):
        _lib.check(_lib.TP_ERR_CUDA, "x")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_compute_entry_points_fail_loudly_without_gpu():
    with pytest.raises(P.DeviceError):
        P.select_tile_plan(10, 10, P.PreprocessConfig())
    with pytest.raises(P.DeviceError):
        P.resize_bilinear(P.ImageBuffer.from_array(np.zeros((2, 2, 3), np.uint8)), 1, 1)
    with pytest.raises(P.DeviceError):
        P.TilePreprocessor(P.PreprocessConfig())


# ---------------------------------------------------------------------------
# drop-in types (imgproc.py:29-128)

def test_image_buffer_validation():
    ok = P.ImageBuffer.from_array(np.zeros((4, 5), np.uint8))
    assert (ok.width, ok.height, ok.channels, ok.elem) == (5, 4, 1, UINT8)
    with pytest.raises(ValueError):
        P.ImageBuffer(0, 1, 3, UINT8, np.zeros((1, 0, 3), np.uint8))
    with pytest.raises(ValueError):
        P.ImageBuffer(2, 2, 2, UINT8, np.zeros((2, 2, 2), np.uint8))
    with pytest.raises(ValueError):
        P.ImageBuffer(2, 2, 3, UINT8, np.zeros((2, 3, 3), np.uint8))
    with pytest.raises(ValueError):
        P.ImageBuffer(2, 2, 3, FLOAT32, np.zeros((2, 2, 3), np.uint8))
    with pytest.raises(ValueError):
        P.ImageBuffer(2, 2, 3, UINT8, np.zeros((2, 2, 6), np.uint8)[:, :, ::2])
    bf = P.ImageBuffer.from_array(np.zeros((2, 2, 3), np.float32), FLOAT16_WIDE)
    assert bf.data.dtype.name == "bfloat16"


def test_preprocess_config_validation():
    with pytest.raises(ValueError):
        P.PreprocessConfig(tile_edge=0)
    with pytest.raises(ValueError):
        P.PreprocessConfig(max_tiles=0)
    with pytest.raises(ValueError):
        P.PreprocessConfig(std=(0.5, 0.0, 0.5))
    with pytest.raises(ValueError):
        P.PreprocessConfig(normalize_precision="float64")
    assert P.PreprocessConfig().effective_precision == FLOAT32
    assert P.PreprocessConfig(reduced_precision_normalize=True).effective_precision == FLOAT16_WIDE


def test_tile_plan_properties_and_records():
    p = P.TilePlan(3, 4, 448, True, 1792, 1344)
    assert p.n_tiles == 12 and p.n_images == 13
    assert P.TilePlan.from_record(p.as_record()) == p
    assert P.TilePlan(1, 1, 448, False, 448, 448).n_images == 1


# ---------------------------------------------------------------------------
# decode (host; imgproc.py:131-260 behaviour, reference tests/test_imgproc.py:269-341)

def _encode(arr, fmt="PNG", **kw):
    buf = io.BytesIO()
    Image.fromarray(arr).save(buf, format=fmt, **kw)
    return buf.getvalue()


def test_png_roundtrip_lossless():
    arr = np.random.default_rng(11).integers(0, 256, size=(13, 17, 3), dtype=np.uint8)
    img = P.decode_image(_encode(arr), P.PreprocessConfig())
    assert (img.width, img.height, img.channels, img.elem) == (17, 13, 3, UINT8)
    assert np.array_equal(img.data, arr)


def test_grayscale_and_palette_promoted_to_rgb():
    gray = np.arange(16, dtype=np.uint8).reshape(4, 4) * 16
    out = P.decode_image(_encode(gray), P.PreprocessConfig())
    assert out.channels == 3 and np.array_equal(out.data[:, :, 0], gray)
    pal = Image.fromarray(np.stack([gray] * 3, axis=-1)).convert("P",
                                                                palette=Image.Palette.ADAPTIVE)
    buf = io.BytesIO()
    pal.save(buf, format="PNG")
    assert P.decode_image(buf.getvalue(), P.PreprocessConfig()).channels == 3


def test_alpha_modes_rejected():
    with pytest.raises(P.UnsupportedFormatError):
        P.decode_image(_encode(np.zeros((4, 4, 4), np.uint8)), P.PreprocessConfig())


def test_decode_fault_offsets():
    with pytest.raises(P.DecodeError) as exc:
        P.decode_image(b"definitely not an image", P.PreprocessConfig())
    assert exc.value.byte_offset == 0
    arr = np.random.default_rng(13).integers(0, 256, size=(32, 32, 3), dtype=np.uint8)
    payload = _encode(arr)
    cut = payload[: len(payload) // 2]
    with pytest.raises(P.DecodeError) as exc:
        P.decode_image(cut, P.PreprocessConfig())
    assert exc.value.byte_offset == len(cut)
    bad = bytearray(payload)
    idat = bytes(bad).index(b"IDAT")
    for k in range(6, 30):
        bad[idat + 4 + k] ^= 0xFF
    with pytest.raises(P.DecodeError) as exc:
        P.decode_image(bytes(bad), P.PreprocessConfig())
    assert exc.value.byte_offset == idat + 4
    jpg = _encode(arr, fmt="JPEG", quality=85)
    cutj = jpg[: len(jpg) - 40]
    with pytest.raises(P.DecodeError) as exc:
        P.decode_image(cutj, P.PreprocessConfig())
    assert exc.value.byte_offset == len(cutj)


@pytest.mark.reference
def test_fault_locator_matches_live_reference(reference):
    from paper_2603_16987_b200._decode import fault_offset
    from vlmfp.imgproc import _locate_fault

    rng = np.random.default_rng(0)
    for trial in range(600):
        arr = rng.integers(0, 256, size=(int(rng.integers(1, 30)), int(rng.integers(1, 30)), 3),
                           dtype=np.uint8)
        p = bytearray(_encode(arr, fmt=["PNG", "JPEG"][trial % 2]))
        mode = trial % 4
        if mode == 0:
            p = p[: int(rng.integers(0, len(p)))]
        elif mode == 1:
            for _ in range(int(rng.integers(1, 6))):
                p[int(rng.integers(0, len(p)))] ^= 0xFF
        elif mode == 2:
            p = bytes(rng.integers(0, 256, size=int(rng.integers(0, 30)), dtype=np.uint8))
        assert fault_offset(bytes(p)) == _locate_fault(bytes(p))


# ---------------------------------------------------------------------------
# contract arithmetic (tokenred.py:106-127, backend.py:92-109)

def test_tokens_per_tile_and_count():
    assert P.tokens_per_tile(512, 16, 4) == 64
    assert P.tokens_per_tile(448, 14, 2) == 256
    with pytest.raises(P.ShapeError):
        P.tokens_per_tile(448, 15, 2)
    with pytest.raises(P.ShapeError):
        P.tokens_per_tile(448, 14, 3)
    with pytest.raises(P.ShapeError):
        P.TokenReductionConfig(patch_edge=0)
    plan = P.TilePlan(2, 1, 448, True, 448, 896)
    assert P.visual_token_count(plan, 14, 2) == 768


def test_assemble_contract():
    plan = P.TilePlan(1, 1, 512, False, 512, 512)
    tr = P.TokenReductionConfig(patch_edge=16, r=4)
    seq = P.TokenSequence([1] + [5] * 64 + [3], 65, [(1, 64)], [False] * 66)
    out = P.assemble(seq, plan, tr)
    assert out.n_visual == 64 and out.n_text == 2 and out.ids == seq.ids
    assert P.assemble(P.TokenSequence([1, 3], 1, [], [False] * 2), None, tr).n_visual == 0
    bad = P.TokenSequence([1] + [5] * 60 + [3], 61, [(1, 60)], [False] * 62)
    with pytest.raises(P.AssemblyError) as exc:
        P.assemble(bad, plan, tr)
    assert (exc.value.expected, exc.value.got) == (64, 60)


def test_token_sequence_validate():
    v = P.tokenizer.SpecialVocab(P.SpecialIds(0, 1, 2, 3, 4, 5, 6))
    P.TokenSequence([2, 5, 5, 3], 3, [(1, 2)], [False] * 4).validate(v)
    with pytest.raises(P.MalformedSequenceError):
        P.TokenSequence([2, 5, 5, 3], 9, [], [False] * 4).validate(v)
    with pytest.raises(P.MalformedSequenceError):
        P.TokenSequence([2, 5, 5, 3], 3, [(0, 2)], [False] * 4).validate(v)
    with pytest.raises(P.MalformedSequenceError):
        P.TokenSequence([2, 5, 5, 3], 3, [], [False] * 3).validate(v)


def test_load_specials(tmp_path):
    import json

    specials = {"bos": "<b>", "eos": "<e>", "user_header": "<u>", "assistant_header": "<a>",
                "image_marker": "<i>", "image_context": "<c>", "pad": "<p>"}
    body = ["<b>", "<e>", "<u>", "<a>", "<i>", "<c>", "<p>", "x"]
    f = tmp_path / "v.txt"
    f.write_text(json.dumps({"specials": specials}) + "\n" + "\n".join(body) + "\n")
    sp = P.load_specials(f).specials
    assert (sp.image_marker, sp.image_context, sp.assistant_header) == (4, 5, 3)
    f.write_text("not json\n<b>\n")
    with pytest.raises(P.DataError):
        P.load_specials(f)


def test_expand_error_mapping():
    from paper_2603_16987_b200.tokenizer import _raise_for

    with pytest.raises(P.ExpansionError):
        _raise_for(_lib.TP_EXPAND_ERR_MARKER_COUNT | _lib.TP_EXPAND_ERR_NO_ASSISTANT, 1, 2)
    with pytest.raises(P.MalformedSequenceError):
        _raise_for(_lib.TP_EXPAND_ERR_NO_ASSISTANT, 1, 1)
    _raise_for(0, 1, 1)


# ---------------------------------------------------------------------------
# workloads, byte model, packing

def test_workload_byte_model_matches_survey():
    b = workload_bytes(c2())
    assert b["n_images"] == 192
    assert abs(b["total"] / 1e6 - 561.5) < 0.1
    assert abs(workload_bytes(c1())["total"] / 1e6 - 15.3) < 0.1
    assert abs(workload_bytes(c3())["total"] / 1e6 - 13.9) < 0.1


def test_c4_plan_mix_matches_survey():
    from collections import Counter

    mix = Counter(plan_rows_cols(int(w), int(h), 448, 12) for w, h in c4_shapes(1200))
    assert mix[(3, 4)] == 300 and mix[(1, 2)] == 228 and mix[(2, 1)] == 200
    assert mix[(1, 3)] == 49 and mix[(2, 5)] == 23


def test_layout_offsets_alignment():
    wh = np.array([[3, 5], [1920, 1080], [7, 1]])
    off, total = layout_offsets(wh, 3)
    assert off[0] == 0 and all(o % 256 == 0 for o in off)
    assert off[1] >= 45 and off[2] >= off[1] + 1920 * 1080 * 3
    assert total >= off[2] + 21


def test_pack_images_roundtrip():
    rng = np.random.default_rng(0)
    arrs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for h, w in [(3, 4), (10, 1), (5, 5)]]
    packed = pack_images(arrs, pin=False)
    buf = packed.data.numpy()
    for a, off in zip(arrs, packed.offsets_host):
        assert np.array_equal(buf[off: off + a.size].reshape(a.shape), a)
    assert packed.wh_host.tolist() == [[4, 3], [1, 10], [5, 5]]
    with pytest.raises(ValueError):
        pack_images([np.zeros((2, 2, 3), np.uint8), np.zeros((2, 2, 1), np.uint8)], pin=False)


def test_host_planner_matches_reference_rule():
    """tp_plan_host (host C, used for touched-row staging) is K1's exact rule: equal to
    the reference's float-log planner (oracle restatement, imgproc.py:266-292)."""
    from oracle import tileprep_oracle as O

    lib = _lib.load()
    rng = np.random.default_rng(17)
    plan = np.zeros(_lib.TP_PLAN_FIELDS, dtype=np.int32)
    cases = [(1, 1, 448, 12), (900, 450, 448, 12), (800, 600, 448, 12), (65536, 1, 448, 12)]
    cases += [(int(w), int(h), int(e), int(m)) for w, h, e, m in zip(
        rng.integers(1, 8192, 400), rng.integers(1, 8192, 400),
        rng.choice([224, 336, 448, 512], 400), rng.integers(1, 13, 400))]
    for w, h, e, m in cases:
        assert lib.tp_plan_host(w, h, e, m, plan.ctypes.data) == _lib.TP_OK
        assert tuple(plan.tolist()) == O.plan_float(w, h, e, m), (w, h, e, m)
    assert lib.tp_plan_host(0, 5, 448, 12, plan.ctypes.data) == _lib.TP_ERR_INVALID_ARGUMENT
    assert lib.tp_plan_host(5, 5, 448, 0, plan.ctypes.data) == _lib.TP_ERR_INVALID_ARGUMENT


# ---------------------------------------------------------------------------
# layout guards of the batch engine (touched-row vs whole-image batches)

def _cpu_packed(touched: bool, tiling=(448, 12), map_len=8):
    from paper_2603_16987_b200.engine import PackedImages

    wh = np.array([[4, 3]], dtype=np.int32)
    p = PackedImages(torch.zeros(256, dtype=torch.uint8), torch.zeros(1, dtype=torch.int64),
                     torch.from_numpy(wh.copy()), 3, wh, np.zeros(1, dtype=np.int64))
    if touched:
        p.row_map = torch.arange(map_len, dtype=torch.int32)
        p.row_map_off = torch.zeros(1, dtype=torch.int64)
        p.touched_for = tiling
    return p


def test_copy_from_carries_row_maps_and_rejects_layout_mismatch():
    a, b = _cpu_packed(True), _cpu_packed(True)
    b.row_map += 100
    b.data += 7
    a.copy_from_(b, non_blocking=False)
    assert torch.equal(a.row_map, b.row_map) and torch.equal(a.data, b.data)
    with pytest.raises(ValueError, match="touched-row"):
        _cpu_packed(False).copy_from_(_cpu_packed(True))
    with pytest.raises(ValueError, match="touched-row"):
        _cpu_packed(True).copy_from_(_cpu_packed(False))
    with pytest.raises(ValueError, match="tilings"):
        _cpu_packed(True).copy_from_(_cpu_packed(True, tiling=(512, 12)))
    with pytest.raises(ValueError, match="differ in size"):
        _cpu_packed(True).copy_from_(_cpu_packed(True, map_len=9))


def test_plan_tile_rejects_touched_row_batches():
    from paper_2603_16987_b200.engine import TilePreprocessor

    prep = object.__new__(TilePreprocessor)  # no device needed: the guard comes first
    with pytest.raises(ValueError, match="whole-image"):
        prep.plan_tile(_cpu_packed(True), out=None)
