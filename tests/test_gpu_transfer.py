"""Pinned staging + one-copy H2D + pipelined K1/K2 on the device (`-m gpu`)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_data import IMAGENET_MEAN, IMAGENET_STD, make_input
from paper_2603_16987_b200.engine import TilePreprocessor, pack_images
from paper_2603_16987_b200.imgproc import PreprocessConfig
from paper_2603_16987_b200.transfer import (
    CostModel,
    HostArena,
    PipelinedPreprocessor,
    pack,
    stage_images,
    staged_bytes,
    transfer,
    unpack,
    upload_images,
)

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
CFG = PreprocessConfig(tile_edge=448, max_tiles=12, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                       reduced_precision_normalize=True)


def _batch(seed: int, n: int):
    rng = np.random.default_rng(seed)
    sizes = [(1080, 1920), (480, 640), (517, 333), (2160, 3840), (300, 700), (64, 64)]
    return [make_input(*sizes[int(rng.integers(len(sizes)))], 3,
                       "random" if i % 2 else "smooth", seed * 100 + i) for i in range(n)]


def test_arena_is_pinned_and_device_transfer_round_trips():
    arena = HostArena(capacity=1 << 16, alignment=64)
    assert arena.pinned and arena.tensor.is_pinned()
    rng = np.random.default_rng(1)
    bufs = [rng.integers(0, 256, n, dtype=np.uint8) for n in (1, 100, 4097)]
    batch = pack(bufs, arena)
    dest = torch.empty(len(batch.payload), dtype=torch.uint8, device=DEV)
    res = transfer(batch, CostModel(1e-5, 1e9), dest=dest)
    res.done.synchronize()
    for got, want in zip(unpack(batch, source=dest), bufs):
        assert np.array_equal(got, want)


def test_staged_upload_feeds_k2_bit_exact():
    imgs = _batch(3, 6)
    arena = HostArena(capacity=staged_bytes(imgs), alignment=256)
    staged = stage_images(imgs, arena)
    dest = torch.empty(staged_bytes(imgs), dtype=torch.uint8, device=DEV)
    packed, done = upload_images(staged, dest)
    prep = TilePreprocessor(CFG, DEV)
    out = prep(packed)
    ref = prep(pack_images(imgs).to(DEV))
    torch.cuda.synchronize()
    T = ref.num_tiles()
    assert out.num_tiles() == T
    assert torch.equal(out.plans.plan, ref.plans.plan)
    assert torch.equal(out.pixel_values[:T].view(torch.int16), ref.pixel_values[:T].view(torch.int16))


@pytest.mark.parametrize("seed,n,e,mt,emit_uint8", [(4, 6, 448, 12, False), (5, 3, 448, 12, True),
                                                    (6, 9, 512, 6, True), (7, 2, 224, 1, True)])
def test_touched_row_upload_equals_full(seed, n, e, mt, emit_uint8):
    """Only the rows K2 reads go over the link (tp_tile_rows): same plans and tile bytes."""
    imgs = _batch(seed, n)
    cfg = PreprocessConfig(tile_edge=e, max_tiles=mt, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    nbytes = staged_bytes(imgs, touched=(e, mt))
    staged = stage_images(imgs, HostArena(capacity=nbytes, alignment=256), touched=(e, mt))
    assert len(staged.batch.payload) == nbytes <= staged_bytes(imgs)
    dest = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    packed, done = upload_images(staged, dest)
    assert packed.row_map is not None
    prep = TilePreprocessor(cfg, DEV, emit_uint8=emit_uint8)
    out = prep(packed)
    ref = prep(pack_images(imgs).to(DEV))
    torch.cuda.synchronize()
    T = ref.num_tiles()
    assert out.num_tiles() == T
    assert torch.equal(out.plans.plan, ref.plans.plan)
    assert torch.equal(out.pixel_values[:T].view(torch.int16), ref.pixel_values[:T].view(torch.int16))
    if emit_uint8:
        assert torch.equal(out.pixel_u8[:T], ref.pixel_u8[:T])
    other = TilePreprocessor(PreprocessConfig(tile_edge=e + 16, max_tiles=mt), DEV)
    with pytest.raises(ValueError):
        other(packed)  # rows staged for another tiling


@pytest.mark.parametrize("touched", [False, True])
def test_pipeline_matches_direct_calls(touched):
    batches = [_batch(10 + i, 4 + i % 3) for i in range(5)]
    slab = max(staged_bytes(b) for b in batches)
    prep = TilePreprocessor(CFG, DEV)
    pipe = PipelinedPreprocessor(prep, slab, depth=2, touched=touched)
    outs = pipe.run(batches)
    pipe.synchronize()
    for b, out in zip(batches, outs):
        ref = prep(pack_images(b).to(DEV))
        torch.cuda.synchronize()
        T = ref.num_tiles()
        assert out.num_tiles() == T
        assert torch.equal(out.pixel_values[:T].view(torch.int16),
                           ref.pixel_values[:T].view(torch.int16))


@pytest.mark.parametrize("layout,bf16", [("NHWC", False), ("NCHW", True)])
def test_touched_rows_grayscale_and_extremes(layout, bf16):
    sizes = [(1, 1), (2, 4000), (4000, 3), (333, 517), (1080, 1920), (64, 64)]
    imgs = [make_input(h, w, 1, "random", 40 + i) for i, (h, w) in enumerate(sizes)]
    cfg = PreprocessConfig(tile_edge=336, max_tiles=9, mean=(0.5,), std=(0.25,),
                           reduced_precision_normalize=bf16)
    nbytes = staged_bytes(imgs, touched=(336, 9))
    staged = stage_images(imgs, HostArena(capacity=nbytes, alignment=256), touched=(336, 9))
    dest = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    packed, _ = upload_images(staged, dest)
    prep = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=True)
    out = prep(packed)
    ref = prep(pack_images(imgs).to(DEV))
    torch.cuda.synchronize()
    T = ref.num_tiles()
    assert out.num_tiles() == T
    assert torch.equal(out.pixel_u8[:T], ref.pixel_u8[:T])
    assert torch.equal(out.pixel_values[:T].view(torch.uint8), ref.pixel_values[:T].view(torch.uint8))
