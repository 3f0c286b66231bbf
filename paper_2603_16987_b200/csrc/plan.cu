// K1 — tile-grid planner (replaces select_tile_plan, imgproc.py:266-292).
//
// The reference minimises the key (|log(w/h) - log(c/r)|, r*c, r) over every
// grid with r*c <= max_tiles, in float64 `math.log`.  Here the first key
// component is compared exactly: |log(w r / (h c))| = log(M/m) with
// M = max(w r, h c), m = min(w r, h c), so key1 < key2  <=>  M1 m2 < M2 m1
// (64-bit products; w, h <= 2^16 and r, c <= 1024 keep them below 2^53).
// DESIGN.md §K1 proves this equals the float ordering on that domain; the
// golden/oracle tests pin it, including every exact tie.
//
// One warp per image: lane L owns rows r = L+1, L+33, ...; for a fixed r the
// key is unimodal in c with its minimum at c ~ w r / h, so only
// c = floor(w r / h) and c + 1 (clamped to [1, max_tiles / r]) can win.  The
// per-lane winners are reduced across the warp with the exact comparator.
// One CTA (one warp per image, up to 1024 threads) walks the batch in chunks of
// blockDim images and block-scans n_images into the output tile offsets.

#include "tp_common.cuh"
#include "plan_core.cuh"

// K1 is a plain launch: a programmatic (PDL) launch may start before a preceding
// non-kernel stream operation (an H2D copy of d_wh, an event wait) has completed,
// which griddepcontrol.wait does not cover.  K1 still releases its dependent early
// (pdl_trigger) so an engine-launched K2 overlaps K1's tail.
#ifndef TP_K1_PDL
#define TP_K1_PDL 0
#endif

namespace tp {
namespace {

constexpr int kPlanThreads = 1024;

__global__ void __launch_bounds__(kPlanThreads)
    k_plan(const int32_t* __restrict__ wh, int32_t n, int32_t tile_edge, int32_t max_tiles,
           int32_t* __restrict__ plan, int32_t* __restrict__ n_img,
           int32_t* __restrict__ tile_off) {
  // per-image counts, blockDim.x entries of dynamic shared memory: a batch-1 plan takes
  // ~0.4 KB, so it shares an SM with two K2 CTAs (the SM K1 runs on would otherwise
  // start its second K2 CTA only after K1 exits: +1 us on batch-1 latency)
  extern __shared__ int32_t s_cnt[];
  __shared__ int64_t s_scan[33];
  __shared__ int s_bad;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  pdl_wait();  // no-op unless launched as a programmatic dependent (TP_K1_PDL)
  if (threadIdx.x == 0) s_bad = 0;
  int64_t carry = 0;
  const int nthr = blockDim.x;  // sized to the batch (<= 1024): small batches, short syncs
  for (int base = 0; base < n; base += nthr) {
    const int chunk = min(nthr, n - base);
    s_cnt[threadIdx.x] = 0;
    __syncthreads();
    // one warp per image (a block of 32 * n threads for n < 32 images)
    for (int j = warp; j < chunk; j += nthr / 32) {
      const int k = base + j;
      const int w = wh[2 * k], h = wh[2 * k + 1];
      const bool ok = w >= 1 && h >= 1 && w <= TP_MAX_EDGE && h <= TP_MAX_EDGE;
      Cand best;
      best.rows = 0;
      best.cols = 0;
      if (ok) best = warp_plan(static_cast<uint32_t>(w), static_cast<uint32_t>(h), max_tiles);
      if (lane == 0) {
        const int tiles = best.rows * best.cols;
        const int thumb = tiles > 1 ? 1 : 0;
        int32_t* p = plan + static_cast<int64_t>(k) * TP_PLAN_FIELDS;
        p[TP_PLAN_ROWS] = best.rows;
        p[TP_PLAN_COLS] = best.cols;
        p[TP_PLAN_TILE_EDGE] = tile_edge;
        p[TP_PLAN_THUMB] = thumb;
        p[TP_PLAN_RESIZED_W] = best.cols * tile_edge;
        p[TP_PLAN_RESIZED_H] = best.rows * tile_edge;
        const int cnt = tiles + thumb;
        n_img[k] = cnt;
        s_cnt[j] = cnt;
        if (!ok) s_bad = 1;
      }
    }
    __syncthreads();
    int64_t total;
    const int64_t ex = block_exclusive_scan<int64_t>(s_cnt[threadIdx.x], s_scan, &total);
    if (threadIdx.x < chunk) tile_off[base + threadIdx.x] = static_cast<int32_t>(carry + ex);
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const bool overflow = carry > INT32_MAX;
    tile_off[n] = (s_bad || overflow) ? -1 : static_cast<int32_t>(carry);
  }
}

}  // namespace
}  // namespace tp

extern "C" int tp_plan(const int32_t* d_wh, int32_t n, int32_t tile_edge, int32_t max_tiles,
                       int32_t* d_plan, int32_t* d_n_img, int32_t* d_tile_off, void* stream) {
  return tp_plan_ex(d_wh, n, tile_edge, max_tiles, d_plan, d_n_img, d_tile_off, 0, stream);
}

extern "C" int tp_plan_ex(const int32_t* d_wh, int32_t n, int32_t tile_edge, int32_t max_tiles,
                          int32_t* d_plan, int32_t* d_n_img, int32_t* d_tile_off, int32_t flags,
                          void* stream) {
  if (n < 0) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_plan: n must be >= 0");
  if (tile_edge < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tile_edge must be positive");
  if (max_tiles < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "max_tiles must be >= 1");
  if (max_tiles > TP_MAX_TILES_LIMIT)
    return tp::set_error(TP_ERR_UNSUPPORTED, "max_tiles %d above the exact-planner limit %d",
                         max_tiles, TP_MAX_TILES_LIMIT);
  if (static_cast<int64_t>(tile_edge) * max_tiles > INT32_MAX)
    return tp::set_error(TP_ERR_UNSUPPORTED, "tile_edge * max_tiles overflows int32");
  if (flags & ~TP_PLAN_AFTER_KERNEL)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_plan_ex: bad flags %d", flags);
  if (!d_tile_off || (n > 0 && (!d_wh || !d_plan || !d_n_img)))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_plan: null buffer");
  // one warp per image up to a full 1024-thread block (small batches: short block syncs)
  const int threads = static_cast<int>(std::min<int64_t>(tp::kPlanThreads, 32LL * std::max(1, n)));
  const size_t smem = sizeof(int32_t) * threads;
  cudaError_t err = cudaSuccess;
  if (TP_K1_PDL || (flags & TP_PLAN_AFTER_KERNEL)) {
    // programmatic dependent of the kernel before it (the previous batch's K2): K1's
    // launch overlaps that kernel's tail; k_plan waits for it before writing anything
    err = tp::launch_pdl(tp::k_plan, dim3(1), dim3(threads), smem, tp::as_stream(stream), d_wh, n,
                         tile_edge, max_tiles, d_plan, d_n_img, d_tile_off);
  } else {
    tp::k_plan<<<1, threads, smem, tp::as_stream(stream)>>>(d_wh, n, tile_edge, max_tiles, d_plan,
                                                         d_n_img, d_tile_off);
  }
  if (err != cudaSuccess) return tp::set_error(TP_ERR_CUDA, "tp_plan: %s", cudaGetErrorString(err));
  return tp::check_launch("tp_plan");
}
