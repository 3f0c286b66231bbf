// K1's per-image planner core (exact integer rule, one warp per image), shared by
// the K1 kernel (plan.cu) and K2's fused small-batch mode (tile_tma.cu).
// See plan.cu for the derivation; replaces select_tile_plan (imgproc.py:266-292).
#pragma once

#include "tp_common.cuh"

namespace tp {
namespace {

struct Cand {
  uint32_t big, small;  // ratio = big / small >= 1
  int32_t rows, cols;
};

__device__ __forceinline__ Cand make_cand(uint32_t w, uint32_t h, int r, int c) {
  const uint32_t a = w * static_cast<uint32_t>(r);
  const uint32_t b = h * static_cast<uint32_t>(c);
  Cand k;
  k.big = a > b ? a : b;
  k.small = a > b ? b : a;
  k.rows = r;
  k.cols = c;
  return k;
}

// strict "a precedes b" in the reference key order (ratio, tiles, rows)
__device__ __forceinline__ bool precedes(const Cand& a, const Cand& b) {
  if (b.rows == 0) return a.rows != 0;  // empty slot loses to anything
  if (a.rows == 0) return false;
  const uint64_t lhs = static_cast<uint64_t>(a.big) * b.small;
  const uint64_t rhs = static_cast<uint64_t>(b.big) * a.small;
  if (lhs != rhs) return lhs < rhs;
  const int ta = a.rows * a.cols, tb = b.rows * b.cols;
  if (ta != tb) return ta < tb;
  return a.rows < b.rows;
}

// Whole warp plans one image; returns the winning (rows, cols) on every lane.
__device__ __noinline__ Cand warp_plan(uint32_t w, uint32_t h, int max_tiles) {
  const int lane = threadIdx.x & 31;
  Cand best;
  best.rows = 0;
  best.cols = 0;
  best.big = 1;
  best.small = 1;
  for (int r = lane + 1; r <= max_tiles; r += 32) {
    const int cmax = max_tiles / r;
    // c* = floor(w r / h), candidates c*, c*+1 clamped to [1, cmax]
    int c0 = static_cast<int>((w * static_cast<uint32_t>(r)) / h);  // w r <= 2^26
    c0 = max(1, min(c0, cmax));
    const int c1 = min(c0 + 1, cmax);
    Cand k0 = make_cand(w, h, r, c0);
    if (precedes(k0, best)) best = k0;
    if (c1 != c0) {
      Cand k1 = make_cand(w, h, r, c1);
      if (precedes(k1, best)) best = k1;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    Cand o;
    o.big = __shfl_xor_sync(0xffffffffu, best.big, d);
    o.small = __shfl_xor_sync(0xffffffffu, best.small, d);
    o.rows = __shfl_xor_sync(0xffffffffu, best.rows, d);
    o.cols = __shfl_xor_sync(0xffffffffu, best.cols, d);
    if (precedes(o, best)) best = o;
  }
  return best;
}

}  // namespace
}  // namespace tp
