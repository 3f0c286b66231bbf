"""Parity of the exact instances bench.py times, against the oracle (bit for bit).

* C2: the bench's 64 x 1080p batch (same generator and seed), run through the bench's
  own steady-state loop -- plan(after_kernel=True) then tile(after_plan=True), the
  programmatic-dependent two-launch chain with the affine EK=448 bf16 NCHW instance --
  for several iterations; then every image's tiles compared with the oracle.
* C2 e2e: the same batch from numpy arrays through PipelinedPreprocessor.submit (native
  touched-row packing, one H2D, tp_tile_rows), as bench.run_e2e drives it.
* C1 / C3: the batch-1 configs through the fused launch (tp_plan_tile) captured in a
  CUDA graph and replayed, as bench.batch1_latency times them.
"""

from __future__ import annotations

import multiprocessing as mp

import numpy as np
import pytest
import torch

from oracle import tileprep_oracle as O
from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed
from paper_2603_16987_b200.imgproc import PreprocessConfig
from paper_2603_16987_b200.workloads import c1, c2, c3

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _oracle_job(job):
    seed, k, w, h, e, mt, mean, std, bf16 = job
    arr = O.synth_image(seed, k, w, h, 3, 0)
    plan = O.plan_float(w, h, e, mt)
    return plan, O.normalize(O.tiles_u8(arr, plan), mean, std, bf16).transpose(0, 3, 1, 2)


def _oracle_batch(wl, seed):
    jobs = [(seed, k, int(w), int(h), wl.tile_edge, wl.max_tiles, tuple(wl.mean),
             tuple(wl.std), wl.bf16) for k, (w, h) in enumerate(wl.wh)]
    if len(jobs) == 1:
        return [_oracle_job(jobs[0])]
    with mp.get_context("fork").Pool(min(16, len(jobs))) as pool:
        return pool.map(_oracle_job, jobs, chunksize=1)


def _cfg(wl):
    return PreprocessConfig(tile_edge=wl.tile_edge, max_tiles=wl.max_tiles, mean=wl.mean,
                            std=wl.std, reduced_precision_normalize=wl.bf16)


def _bits(t: torch.Tensor) -> np.ndarray:
    t = t.cpu()
    return (t.view(torch.int16) if t.dtype == torch.bfloat16 else t.view(torch.int32)).numpy()


def _want_bits(a: np.ndarray) -> np.ndarray:
    return a.view(np.int16) if a.dtype.itemsize == 2 else a.view(np.int32)


def _compare(pv, tile_off, want, plans=None):
    for k, (plan, w) in enumerate(want):
        if plans is not None:
            assert tuple(int(v) for v in plans[k]) == tuple(plan), k
        got = pv[int(tile_off[k]): int(tile_off[k + 1])]
        assert got.shape == w.shape, (k, got.shape, w.shape)
        assert np.array_equal(_bits(got), _want_bits(w)), f"image {k} differs"


@pytest.fixture(scope="module")
def c2_batch():
    wl = c2(64)
    return wl, _oracle_batch(wl, wl.seed)  # bench.run_c2 uses wl.seed at rank 0


def test_c2_bench_steady_state_loop_matches_oracle(c2_batch):
    wl, want = c2_batch
    images = synth_packed(wl.wh, 3, DEV, seed=wl.seed, kind=0)
    prep = TilePreprocessor(_cfg(wl), DEV)
    out = prep(images)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(DEV)
    with torch.cuda.stream(s):
        for _ in range(8):  # the bench's step, back to back on one stream
            prep.plan(images, out.plans, s, after_kernel=True)
            prep.tile(images, out.plans, out.pixel_values, None, s, after_plan=True)
    torch.cuda.synchronize()
    assert out.pixel_values.dtype == torch.bfloat16 and out.pixel_values.shape[1] == 3
    _compare(out.pixel_values, out.plans.tile_off.cpu().numpy(), want,
             out.plans.plan.cpu().numpy())


def test_c2_e2e_pipeline_from_numpy_matches_oracle(c2_batch):
    from paper_2603_16987_b200.transfer import PipelinedPreprocessor, staged_bytes

    wl, want = c2_batch
    images = synth_packed(wl.wh, 3, DEV, seed=wl.seed, kind=0)
    host = [images.data[int(o): int(o) + int(w) * int(h) * 3].cpu().numpy().reshape(int(h), int(w), 3)
            for o, (w, h) in zip(images.offsets_host, images.wh_host)]
    cfg = _cfg(wl)
    prep = TilePreprocessor(cfg, DEV)
    pipe = PipelinedPreprocessor(prep, staged_bytes(host, touched=(448, 12)), depth=2,
                                 touched=True)
    outs = [None, None]
    for i in range(5):  # as bench.run_e2e: two rotating slabs and output buffers
        outs[i % 2] = pipe.submit(host, out=outs[i % 2])
    pipe.synchronize()
    for out in outs:
        _compare(out.pixel_values, out.plans.tile_off.cpu().numpy(), want,
                 out.plans.plan.cpu().numpy())


@pytest.mark.parametrize("which", ["c1", "c3"])
def test_batch1_graph_replay_matches_oracle(which):
    wl = c1() if which == "c1" else c3()
    want = _oracle_batch(wl, 7)  # bench.batch1_latency: synth seed 7
    img = synth_packed(wl.wh, 3, DEV, seed=7, kind=0)
    prep = TilePreprocessor(_cfg(wl), DEV)
    out = prep(img)
    s = torch.cuda.Stream(DEV)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prep(img, out=out, stream=torch.cuda.current_stream(DEV))
    out.pixel_values.zero_()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    if which == "c1":  # SmolVLM-style: fp32 out, E=512, mean = std = 0.5
        assert out.pixel_values.dtype == torch.float32 and out.pixel_values.shape[-1] == 512
    _compare(out.pixel_values, out.plans.tile_off.cpu().numpy(), want,
             out.plans.plan.cpu().numpy())
