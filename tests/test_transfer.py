"""Host staging arena, pack/unpack and the transfer model (CPU).

Re-expresses the reference's transfer tests (vlmfp tests/test_transfer.py:49-336) on
paper_2603_16987_b200.transfer: same layouts (checked against an independent integer
layout oracle), same errors, bit-exact unpack round trips, modeled durations.
"""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_2603_16987_b200.dtypes import FLOAT16_WIDE, FLOAT32, INT32, UINT8, to_numpy
from paper_2603_16987_b200.errors import ArenaFullError, DataError, DomainError, ShapeError
from paper_2603_16987_b200.transfer import (
    CostModel,
    HostArena,
    TransferBatch,
    pack,
    payload_bytes,
    stage_images,
    stage_individually,
    staged_bytes,
    transfer,
    unpack,
)


def oracle_layout(sizes, alignment):
    """Sequential aligned placement: (offsets, padded total)."""
    offsets, mark = [], 0
    for size in sizes:
        offsets.append(mark)
        mark = ((mark + size + alignment - 1) // alignment) * alignment
    return offsets, mark


def rand_buffers(rng, sizes):
    return [rng.integers(0, 256, size=size, dtype=np.uint8) for size in sizes]


def test_fresh_alloc_at_offset_zero():
    region = HostArena(capacity=4096, alignment=64).alloc(64)
    assert region.offset == 0 and region.size == 64


def test_alignment_padding_between_allocations():
    arena = HostArena(capacity=4096, alignment=64)
    assert arena.alloc(1).offset == 0
    assert arena.alloc(1).offset == 64
    assert arena.alloc(65).offset == 128
    assert arena.alloc(1).offset == 256


def test_exhaustion_reports_requested_and_remaining():
    arena = HostArena(capacity=100, alignment=64)
    with pytest.raises(ArenaFullError) as e:
        arena.alloc(101)
    assert e.value.requested == 101 and e.value.remaining == 100


def test_exhaustion_after_partial_use():
    arena = HostArena(capacity=128, alignment=64)
    arena.alloc(10)
    with pytest.raises(ArenaFullError) as e:
        arena.alloc(65)
    assert e.value.remaining == 64


def test_allocation_count_capacity_and_reset():
    arena = HostArena(capacity=1024, alignment=64)
    offs = [arena.alloc(10).offset for _ in range(3)]
    assert arena.allocation_count == 3 and arena.capacity == 1024
    arena.reset()
    assert arena.mark == 0
    assert [arena.alloc(10).offset for _ in range(3)] == offs


def test_region_view_is_writable_window():
    arena = HostArena(capacity=256, alignment=64)
    arena.alloc(3)
    r = arena.alloc(5)
    r.view[:] = 7
    assert np.all(arena.tensor.numpy()[64:69] == 7)


def test_bad_parameters_rejected():
    with pytest.raises(DomainError):
        HostArena(capacity=0)
    with pytest.raises(DomainError):
        HostArena(capacity=64, alignment=0)
    with pytest.raises(DomainError):
        HostArena(capacity=64).alloc(0)


@given(sizes=st.lists(st.integers(1, 300), min_size=1, max_size=10),
       alignment=st.sampled_from([1, 8, 64, 256]))
@settings(max_examples=100, deadline=None)
def test_arena_matches_layout_oracle(sizes, alignment):
    arena = HostArena(capacity=1 << 16, alignment=alignment)
    want, _ = oracle_layout(sizes, alignment)
    assert [arena.alloc(s).offset for s in sizes] == want


def test_payload_bytes():
    assert payload_bytes((448, 448, 3), UINT8) == 448 * 448 * 3
    assert payload_bytes((448, 448, 3), FLOAT32) == 4 * 448 * 448 * 3
    assert payload_bytes((1,), FLOAT16_WIDE) == 2
    with pytest.raises(ShapeError):
        payload_bytes((0, 3), UINT8)
    with pytest.raises(DataError):
        payload_bytes((2,), "complex")


def test_pack_layout_and_entries():
    bufs = [np.zeros(10, np.uint8), np.zeros((2, 3), np.float32), np.zeros(5, np.int32)]
    batch = pack(bufs, HostArena(capacity=4096, alignment=64))
    offs, total = oracle_layout([b.nbytes for b in bufs], 64)
    assert [e.offset for e in batch.entries] == offs
    assert [e.dtype for e in batch.entries] == [UINT8, FLOAT32, INT32]
    assert batch.entries[1].shape == (2, 3)
    assert batch.copies == ((0, total),) and batch.n_copies == 1


def test_pack_empty_and_full():
    arena = HostArena(capacity=128, alignment=64)
    empty = pack([], arena)
    assert empty.entries == () and empty.n_copies == 0 and arena.allocation_count == 0
    with pytest.raises(ArenaFullError):
        pack([np.zeros(100, np.uint8), np.zeros(100, np.uint8)], arena)


def test_stage_individually_layout_matches_pack():
    bufs = [np.zeros(n, dtype=np.uint8) for n in (10, 20, 30)]
    packed = pack(bufs, HostArena(capacity=4096, alignment=64))
    arena = HostArena(capacity=4096, alignment=64)
    staged = stage_individually(bufs, arena)
    assert [e.offset for e in staged.entries] == [e.offset for e in packed.entries]
    assert staged.n_copies == 3 and arena.allocation_count == 3


@given(seed=st.integers(0, 2**32 - 1),
       sizes=st.lists(st.integers(1, 64), min_size=0, max_size=8))
@settings(max_examples=120, deadline=None)
def test_unpack_round_trip_bit_exact(seed, sizes):
    rng = np.random.default_rng(seed)
    bufs = []
    for n in sizes:
        tag = rng.choice([UINT8, FLOAT32, INT32, FLOAT16_WIDE])
        dt = to_numpy(tag)
        raw = rng.integers(0, 256, size=n * 4, dtype=np.uint8)
        count = (n * 4) // dt.itemsize
        bufs.append(np.frombuffer(raw.tobytes()[: count * dt.itemsize], dtype=dt).copy())
    for make in (pack, stage_individually):
        out = unpack(make(bufs, HostArena(capacity=1 << 16, alignment=64)))
        assert len(out) == len(bufs)
        for got, want in zip(out, bufs):
            assert got.dtype == want.dtype and got.shape == want.shape
            assert got.tobytes() == want.tobytes()


def test_transfer_model_durations():
    model = CostModel(latency_per_copy=10e-6, bytes_per_second=1e12)
    bufs = [np.zeros(1, dtype=np.uint8) for _ in range(8)]
    packed = transfer(pack(bufs, HostArena(4096, 64)), model)
    staged = transfer(stage_individually(bufs, HostArena(4096, 64)), model)
    assert staged.duration_s == pytest.approx(80e-6 + 8 / 1e12, rel=1e-12)
    assert packed.duration_s == pytest.approx(10e-6 + 8 / 1e12, rel=1e-12)
    assert transfer(pack([], HostArena(64, 64)), model).duration_s == 0.0
    with pytest.raises(DomainError):
        CostModel(latency_per_copy=0.0, bytes_per_second=1e9)
    with pytest.raises(DomainError):
        CostModel(latency_per_copy=1e-5, bytes_per_second=0.0)


def test_transfer_copies_content_and_leaves_source_intact():
    rng = np.random.default_rng(7)
    bufs = rand_buffers(rng, [33, 190, 5])
    batch = pack(bufs, HostArena(capacity=4096, alignment=64))
    before = batch.payload.tobytes()
    result = transfer(batch, CostModel(latency_per_copy=1e-5, bytes_per_second=1e9))
    assert batch.payload.tobytes() == before
    for got, want in zip(unpack(batch, source=result.dest), bufs):
        np.testing.assert_array_equal(got, want)


def test_batch_is_immutable():
    batch = pack([np.zeros(4, dtype=np.uint8)], HostArena(capacity=4096, alignment=64))
    assert isinstance(batch, TransferBatch)
    with pytest.raises(AttributeError):
        batch.entries = ()


def test_stage_images_layout_and_round_trip():
    rng = np.random.default_rng(3)
    imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for h, w in ((5, 7), (1, 1), (33, 2))]
    arena = HostArena(capacity=staged_bytes(imgs), alignment=256)
    st_ = stage_images(imgs, arena)
    assert st_.batch.n_copies == 1 and st_.n == 3
    assert all(o % 256 == 0 for o in st_.offsets)
    out = unpack(st_.batch)
    assert np.array_equal(out[0], [[7, 5], [1, 1], [2, 33]])  # (width, height)
    assert np.array_equal(out[1], st_.offsets)
    for got, want in zip(out[2:], imgs):
        assert np.array_equal(got, want)
    with pytest.raises(DataError):
        stage_images([np.zeros((2, 2, 3), np.uint8), np.zeros((2, 2, 1), np.uint8)], arena)


@pytest.mark.parametrize("seed", range(6))
def test_touched_row_maps_match_oracle_taps(seed):
    """tp_plan_host + tp_touched_rows / _cols (host C) mark exactly the rows and columns
    of the oracle's axis taps for the oracle's plan: tiles H -> rows*E, W -> cols*E and
    the thumbnail H -> E, W -> E."""
    from oracle import tileprep_oracle as O
    from paper_2603_16987_b200.transfer import touched_row_maps

    rng = np.random.default_rng(seed)
    wh = np.stack([rng.integers(1, 5000, 40), rng.integers(1, 5000, 40)], axis=1).astype(np.int32)
    e, mt = [(448, 12), (512, 6), (224, 1), (33, 40), (448, 12), (336, 9)][seed]
    maps = touched_row_maps(wh, e, mt)
    for (w, h), m in zip(wh, maps):
        rows, cols, _, thumb, rw, rh = O.plan_float(int(w), int(h), e, mt)
        for src, outs, part in ((int(h), [rh, e] if thumb else [rh], m[: h + 1]),
                                (int(w), [rw, e] if thumb else [rw], m[h + 1:])):
            want = set()
            for out in outs:
                i0, i1, _ = O.axis_weights(src, out)
                want |= set(i0.tolist()) | set(i1.tolist())
            got = np.nonzero(part[1:] >= 0)[0]
            assert part[0] == len(want) and set(got.tolist()) == want
            assert np.array_equal(part[1:][got], np.arange(len(got)))



@pytest.mark.parametrize("threads", [1, 0])
def test_native_pack_strided_views_whole_and_touched(threads):
    """tp_stage_pack on non-contiguous caller views (row stride > row bytes): whole
    images round-trip; touched staging holds exactly the mapped rows, in order."""
    from paper_2603_16987_b200.transfer import staging_map

    rng = np.random.default_rng(4)
    big = [rng.integers(0, 256, (300, 420, 3), dtype=np.uint8) for _ in range(3)]
    imgs = [b[7:290, 11:400] for b in big]
    st_ = stage_images(imgs, HostArena(staged_bytes(imgs), 256), threads=threads)
    for got, want in zip(unpack(st_.batch)[2:], imgs):
        assert np.array_equal(got, want)
    tt = (64, 6)
    st2 = stage_images(imgs, HostArena(staged_bytes(imgs, touched=tt), 256), touched=tt,
                       threads=threads)
    blocks = unpack(st2.batch)[4:]
    for a, blk in zip(imgs, blocks):
        m = staging_map(a.shape[1], a.shape[0], *tt)
        rows = np.nonzero(m[1: a.shape[0] + 1] >= 0)[0]
        assert np.array_equal(blk, a[rows])
