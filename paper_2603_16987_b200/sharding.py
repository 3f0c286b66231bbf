"""Multi-GPU sharding of independent images.

Images are independent, so a batch is partitioned across ranks with no
data-path collective: each rank plans, tiles and expands its own images on its
own GPU and stream.  Ranks are balanced by longest-processing-time-first (LPT)
greedy assignment on the algorithmic byte cost of each image (a 13-tile image
costs ~4x a 3-tile one).  The only cross-rank operations are the barrier and
the max-over-ranks timing reduction of the benchmark.
"""

from __future__ import annotations

import heapq
from typing import Sequence

import numpy as np

from .workloads import image_bytes


def lpt_assign(costs: Sequence[float], n_ranks: int) -> list[np.ndarray]:
    """Greedy LPT: heaviest image first onto the currently lightest rank
    (ties: lower rank).  Returns per-rank ascending index arrays."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    costs = np.asarray(costs, dtype=np.float64)
    order = np.lexsort((np.arange(len(costs)), -costs))  # cost desc, index asc
    heap = [(0.0, r) for r in range(n_ranks)]
    buckets: list[list[int]] = [[] for _ in range(n_ranks)]
    for i in order:
        load, r = heapq.heappop(heap)
        buckets[r].append(int(i))
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [np.array(sorted(b), dtype=np.int64) for b in buckets]


def image_costs(wh: np.ndarray, tile_edge: int, max_tiles: int, s_out: int = 2) -> np.ndarray:
    cache: dict = {}
    out = np.empty(len(wh), dtype=np.float64)
    for k, (w, h) in enumerate(np.asarray(wh)):
        key = (int(w), int(h))
        if key not in cache:
            b = image_bytes(*key, tile_edge, max_tiles, 3, s_out)
            cache[key] = b["read"] + b["write"]
        out[k] = cache[key]
    return out


def shard(wh: np.ndarray, tile_edge: int, max_tiles: int, rank: int, world: int,
          s_out: int = 2) -> np.ndarray:
    """Indices of the images rank `rank` of `world` processes."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return lpt_assign(image_costs(wh, tile_edge, max_tiles, s_out), world)[rank]


def imbalance(wh: np.ndarray, tile_edge: int, max_tiles: int, world: int) -> float:
    """max rank load / mean rank load under LPT (1.0 = perfect)."""
    costs = image_costs(wh, tile_edge, max_tiles)
    loads = [costs[idx].sum() for idx in lpt_assign(costs, world)]
    return float(max(loads) / (sum(loads) / world))
