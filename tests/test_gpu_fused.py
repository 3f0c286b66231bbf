"""tp_plan_tile (K1 inside K2 for batches of <= TP_PLAN_TILE_MAX_IMAGES images) against
the two-launch path tp_plan + tp_tile_ex: identical plans, counts, offsets and tile bytes;
and against the oracle's plans (select_tile_plan, imgproc.py:266-292)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import tileprep_oracle as O
from paper_2603_16987_b200 import _lib
from paper_2603_16987_b200.engine import TileBatch, TilePreprocessor, synth_packed
from paper_2603_16987_b200.imgproc import PreprocessConfig

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
IMAGENET = ((0.485, 0.456, 0.406), (0.229, 0.224, 0.225))


def _both(wh, cfg, channels=3, kind=0, seed=5, **kw):
    packed = synth_packed(np.asarray(wh, dtype=np.int32), channels, DEV, seed=seed, kind=kind)
    outs = []
    for fuse in (True, False):
        prep = TilePreprocessor(cfg, DEV, fuse_small=fuse, **kw)
        outs.append(prep(packed))
    torch.cuda.synchronize()
    return outs


def _assert_same(a, b):
    assert torch.equal(a.plans.plan, b.plans.plan)
    assert torch.equal(a.plans.n_images, b.plans.n_images)
    assert torch.equal(a.plans.tile_off, b.plans.tile_off)
    T = int(a.plans.tile_off[-1])
    assert T >= 0
    for x, y in ((a.pixel_values, b.pixel_values), (a.pixel_u8, b.pixel_u8)):
        assert (x is None) == (y is None)
        if x is not None:
            assert torch.equal(x[:T].view(torch.uint8), y[:T].view(torch.uint8))
    return T


@pytest.mark.parametrize("wh", [
    [[1920, 1080]],
    [[3840, 2160]],
    [[640, 480], [1080, 1920]],
    [[517, 333], [1, 1], [448, 448], [8000, 90]],
])
@pytest.mark.parametrize("bf16,layout,emit_uint8", [(True, "NCHW", False), (False, "NCHW", True),
                                                    (True, "NHWC", True)])
def test_fused_equals_two_launches(wh, bf16, layout, emit_uint8):
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET[0], std=IMAGENET[1],
                           reduced_precision_normalize=bf16)
    a, b = _both(wh, cfg, layout=layout, emit_uint8=emit_uint8)
    _assert_same(a, b)
    plans = a.plans.plan.cpu().numpy()
    for k, (w, h) in enumerate(wh):
        assert tuple(plans[k]) == O.plan_float(w, h, 448, 12)


@pytest.mark.parametrize("e,mt,channels,kind", [(512, 12, 3, 1), (33, 6, 1, 0), (448, 1, 3, 0),
                                                (224, 40, 3, 1)])
def test_fused_other_geometries(e, mt, channels, kind):
    cfg = PreprocessConfig(tile_edge=e, max_tiles=mt, mean=(0.5,) * 3, std=(0.5,) * 3)
    wh = [[1920, 1080], [300, 1200], [77, 5]][: 1 + (e % 3)]
    a, b = _both(wh, cfg, channels=channels, kind=kind, emit_uint8=True)
    _assert_same(a, b)


def test_fused_uint8_only_and_invalid_size():
    cfg = PreprocessConfig(tile_edge=448, max_tiles=12)
    a, b = _both([[1920, 1080]], cfg, normalize=False, emit_uint8=True)
    _assert_same(a, b)
    # an out-of-range size flags the batch exactly as tp_plan does (tile_off[n] = -1)
    wh = torch.tensor([[1920, 1080], [70000, 10]], dtype=torch.int32, device=DEV)
    packed = synth_packed(np.array([[1920, 1080], [1, 1]], np.int32), 3, DEV, seed=1)
    packed.wh.copy_(wh)
    outs = []
    for fuse in (True, False):
        prep = TilePreprocessor(cfg, DEV, fuse_small=fuse)
        plans = prep.alloc_plans(2)
        pv, u8 = prep.alloc_outputs(3, 26)
        out = TileBatch(plans, pv, u8)
        prep(packed, out=out)
        outs.append(out)
    torch.cuda.synchronize()
    for o in outs:
        assert int(o.plans.tile_off[-1]) == -1
    assert torch.equal(outs[0].plans.plan, outs[1].plans.plan)
    assert torch.equal(outs[0].plans.n_images, outs[1].plans.n_images)


def test_plan_tile_abi_limits():
    n = _lib.TP_PLAN_TILE_MAX_IMAGES + 1
    lib = _lib.load()
    rc = lib.tp_plan_tile(None, None, None, n, 3, 448, 12, None, None, None, None,
                          _lib.TP_DTYPE_BF16, _lib.TP_LAYOUT_NCHW, None, None, 1, 0, None)
    assert rc == _lib.TP_ERR_UNSUPPORTED
    rc = lib.tp_plan_tile(None, None, None, 1, 3, 448, 12, None, None, None, None,
                          _lib.TP_DTYPE_BF16, _lib.TP_LAYOUT_NCHW, None, None, 1,
                          _lib.TP_TILE_ALGO_EXACT, None)
    assert rc == _lib.TP_ERR_INVALID_ARGUMENT
