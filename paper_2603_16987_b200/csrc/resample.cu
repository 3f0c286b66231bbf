// K2 — fused resample + crop + thumbnail + normalize + layout/cast.
//
// Replaces tile_image/_tile_fused (imgproc.py:373-412, :449-465) followed by
// normalize_tiles (imgproc.py:496-513), and resize_bilinear (:352-367).
//
// Work decomposition: the batch's output tiles (tile_off[n] of them, image-
// major, row-major tiles then the thumbnail, imgproc.py:388-398) are cut into
// items of kRowsPerItem output rows.  A persistent grid (a multiple of the SM
// count) strides over items; each item finds its image by binary search in
// tile_off and derives the sampling window from the plan:
//   tile (r, c):  virtual resize H -> rows*E, W -> cols*E, window (r*E, c*E)
//   thumbnail:    virtual resize H -> E,      W -> E,      window (0, 0)
// so no host round trip is needed between the planner and this kernel.
//
// Exact path (this file): every output channel value is computed in fp64 in
// the reference order (tp_common.cuh: blend_exact), bit-exact by construction.

#include "tp_common.cuh"

namespace tp {
namespace {

constexpr int kThreads = 256;
constexpr int kRowsPerItem = 8;

struct TileGeom {
  const uint8_t* img;
  int W, H;
  int RW, RH;  // virtual resized size
  int oy0, ox0;
  int64_t out_tile;  // global tile index
};

__device__ __forceinline__ int find_image(const int32_t* __restrict__ tile_off, int n, int g) {
  int lo = 0, hi = n;  // tile_off[lo] <= g < tile_off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(tile_off + mid) <= g) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ TileGeom tile_geom(const uint8_t* __restrict__ src,
                                              const int64_t* __restrict__ src_off,
                                              const int32_t* __restrict__ wh,
                                              const int32_t* __restrict__ plan,
                                              const int32_t* __restrict__ tile_off, int n,
                                              int E, int g) {
  const int k = find_image(tile_off, n, g);
  const int t = g - __ldg(tile_off + k);
  const int32_t* p = plan + static_cast<int64_t>(k) * TP_PLAN_FIELDS;
  const int rows = __ldg(p + TP_PLAN_ROWS), cols = __ldg(p + TP_PLAN_COLS);
  TileGeom q;
  q.img = src + __ldg(src_off + k);
  q.W = __ldg(wh + 2 * k);
  q.H = __ldg(wh + 2 * k + 1);
  q.out_tile = g;
  if (t < rows * cols) {  // plan's resized size, as _tile_fused samples it (imgproc.py:383-384)
    q.RW = __ldg(p + TP_PLAN_RESIZED_W);
    q.RH = __ldg(p + TP_PLAN_RESIZED_H);
    q.oy0 = (t / cols) * E;
    q.ox0 = (t % cols) * E;
  } else {  // thumbnail: whole-source resize to E x E, last (imgproc.py:395-398)
    q.RW = E;
    q.RH = E;
    q.oy0 = 0;
    q.ox0 = 0;
  }
  return q;
}

template <typename OutT>
__device__ __forceinline__ void store_norm(OutT* out, int64_t idx, const OutT* lut, int c,
                                           uint32_t u) {
  out[idx] = lut[c * 256 + u];
}

// One output row segment [0, OW) of row `oy` of the window, exact fp64.
template <int C, typename OutT, int LAYOUT, bool WRITE_OUT>
__device__ __forceinline__ void exact_row(const TileGeom& q, int j, int E, double sy,
                                          double sx, const OutT* s_lut, OutT* __restrict__ out,
                                          uint8_t* __restrict__ out_u8) {
  const AxisTap ty = axis_tap(q.oy0 + j, q.H, sy);
  const int64_t stride = static_cast<int64_t>(q.W) * C;
  const uint8_t* r0 = q.img + ty.i0 * stride;
  const uint8_t* r1 = q.img + ty.i1 * stride;
  const int64_t EE = static_cast<int64_t>(E) * E;
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const AxisTap tx = axis_tap(q.ox0 + i, q.W, sx);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const uint32_t s00 = __ldg(r0 + tx.i0 * C + c), s01 = __ldg(r0 + tx.i1 * C + c);
      const uint32_t s10 = __ldg(r1 + tx.i0 * C + c), s11 = __ldg(r1 + tx.i1 * C + c);
      const uint32_t u = blend_exact(s00, s01, s10, s11, ty, tx);
      const int64_t pix = q.out_tile * EE + static_cast<int64_t>(j) * E + i;
      if (out_u8) out_u8[pix * C + c] = static_cast<uint8_t>(u);
      if (WRITE_OUT) {
        const int64_t idx = LAYOUT == TP_LAYOUT_NCHW
                                ? (q.out_tile * C + c) * EE + static_cast<int64_t>(j) * E + i
                                : pix * C + c;
        store_norm(out, idx, s_lut, c, u);
      }
    }
  }
}

template <int C, typename OutT, int LAYOUT, bool WRITE_OUT>
__global__ void __launch_bounds__(kThreads)
    k_tile_exact(const uint8_t* __restrict__ src, const int64_t* __restrict__ src_off,
                 const int32_t* __restrict__ wh, int n, const int32_t* __restrict__ plan,
                 const int32_t* __restrict__ tile_off, int E, const OutT* __restrict__ lut,
                 OutT* __restrict__ out, uint8_t* __restrict__ out_u8, int64_t cap) {
  __shared__ OutT s_lut[WRITE_OUT ? C * 256 : 1];
  if (WRITE_OUT)
    for (int i = threadIdx.x; i < C * 256; i += blockDim.x) s_lut[i] = lut[i];
  __syncthreads();
  const int total = static_cast<int>(min(static_cast<int64_t>(__ldg(tile_off + n)), cap));
  if (total <= 0) return;
  const int chunks = (E + kRowsPerItem - 1) / kRowsPerItem;
  const int64_t items = static_cast<int64_t>(total) * chunks;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int g = static_cast<int>(item / chunks);
    const int ch = static_cast<int>(item - static_cast<int64_t>(g) * chunks);
    const TileGeom q = tile_geom(src, src_off, wh, plan, tile_off, n, E, g);
    const double sy = axis_scale(q.H, q.RH), sx = axis_scale(q.W, q.RW);
    const int j_end = min(E, (ch + 1) * kRowsPerItem);
    for (int j = ch * kRowsPerItem; j < j_end; ++j)
      exact_row<C, OutT, LAYOUT, WRITE_OUT>(q, j, E, sy, sx, s_lut, out, out_u8);
  }
}

// Full-frame resize (resize_bilinear): one "tile" whose window is the whole
// virtual image of out_w x out_h; rows are strided over the grid.
template <int C>
__global__ void __launch_bounds__(kThreads)
    k_resize_exact(const uint8_t* __restrict__ src, int W, int H, int OW, int OH,
                   uint8_t* __restrict__ dst) {
  const double sy = axis_scale(H, OH), sx = axis_scale(W, OW);
  const int64_t stride = static_cast<int64_t>(W) * C;
  for (int oy = blockIdx.x; oy < OH; oy += gridDim.x) {
    const AxisTap ty = axis_tap(oy, H, sy);
    const uint8_t* r0 = src + ty.i0 * stride;
    const uint8_t* r1 = src + ty.i1 * stride;
    for (int ox = threadIdx.x; ox < OW; ox += blockDim.x) {
      const AxisTap tx = axis_tap(ox, W, sx);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t u = blend_exact(__ldg(r0 + tx.i0 * C + c), __ldg(r0 + tx.i1 * C + c),
                                       __ldg(r1 + tx.i0 * C + c), __ldg(r1 + tx.i1 * C + c),
                                       ty, tx);
        dst[(static_cast<int64_t>(oy) * OW + ox) * C + c] = static_cast<uint8_t>(u);
      }
    }
  }
}


template <int C, typename OutT, int LAYOUT, bool WRITE_OUT>
int launch_tile(const uint8_t* src, const int64_t* src_off, const int32_t* wh, int n,
                const int32_t* plan, const int32_t* tile_off, int E, const void* lut, void* out,
                uint8_t* out_u8, int64_t cap, int algo, cudaStream_t stream,
                K2Options fuse = K2Options{}) {
  const int sms = max(1, device_sm_count());
  int per_sm = 0;
  if ((algo & 0xFF) == TP_TILE_ALGO_EXACT) {
    auto kern = k_tile_exact<C, OutT, LAYOUT, WRITE_OUT>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
    kern<<<max(1, per_sm) * sms, kThreads, 0, stream>>>(
        src, src_off, wh, n, plan, tile_off, E, static_cast<const OutT*>(lut),
        static_cast<OutT*>(out), out_u8, cap);
    return check_launch("tp_tile(exact)");
  }
  return launch_tile_tma<C, OutT, LAYOUT, WRITE_OUT>(src, src_off, wh, n, plan, tile_off, E, lut,
                                                     out, out_u8, cap,
                                                     (algo & TP_TILE_NORM_AFFINE) != 0,
                                                     (algo & TP_TILE_AFTER_PLAN) != 0, stream,
                                                     fuse);
}

template <int C>
int dispatch_tile(const uint8_t* src, const int64_t* src_off, const int32_t* wh, int n,
                  const int32_t* plan, const int32_t* tile_off, int E, const void* lut,
                  int dtype, int layout, void* out, uint8_t* out_u8, int64_t cap, int algo,
                  cudaStream_t s, K2Options fuse = K2Options{}) {
  if (dtype == TP_DTYPE_NONE)
    return launch_tile<C, float, TP_LAYOUT_NHWC, false>(src, src_off, wh, n, plan, tile_off, E,
                                                        lut, out, out_u8, cap, algo, s, fuse);
  if (dtype == TP_DTYPE_F32) {
    if (layout == TP_LAYOUT_NCHW)
      return launch_tile<C, float, TP_LAYOUT_NCHW, true>(src, src_off, wh, n, plan, tile_off,
                                                         E, lut, out, out_u8, cap, algo, s, fuse);
    return launch_tile<C, float, TP_LAYOUT_NHWC, true>(src, src_off, wh, n, plan, tile_off, E,
                                                       lut, out, out_u8, cap, algo, s, fuse);
  }
  if (layout == TP_LAYOUT_NCHW)
    return launch_tile<C, __nv_bfloat16, TP_LAYOUT_NCHW, true>(src, src_off, wh, n, plan,
                                                               tile_off, E, lut, out, out_u8, cap, algo, s, fuse);
  return launch_tile<C, __nv_bfloat16, TP_LAYOUT_NHWC, true>(src, src_off, wh, n, plan,
                                                             tile_off, E, lut, out, out_u8, cap, algo, s, fuse);
}

// argument checks shared by tp_tile_ex and tp_plan_tile (plans and offsets apart)
int check_tile_args(const uint8_t* src, const int64_t* src_off, const int32_t* wh, int n,
                    int channels, int tile_edge, const void* lut, int dtype, int layout,
                    const void* out, const uint8_t* out_u8, int64_t cap, int algo) {
  const int base_algo = algo & 0xFF;
  if ((base_algo != TP_TILE_ALGO_AUTO && base_algo != TP_TILE_ALGO_FAST &&
       base_algo != TP_TILE_ALGO_EXACT) ||
      (algo & ~(0xFF | TP_TILE_NORM_AFFINE | TP_TILE_AFTER_PLAN)) != 0)
    return set_error(TP_ERR_INVALID_ARGUMENT, "bad algo %d", algo);
  if (n < 0) return set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile: n must be >= 0");
  if (channels != 1 && channels != 3)
    return set_error(TP_ERR_INVALID_ARGUMENT, "channels must be 1 or 3, got %d", channels);
  if (tile_edge < 1) return set_error(TP_ERR_INVALID_ARGUMENT, "tile_edge must be positive");
  if (dtype != TP_DTYPE_NONE && dtype != TP_DTYPE_F32 && dtype != TP_DTYPE_BF16)
    return set_error(TP_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  if (layout != TP_LAYOUT_NCHW && layout != TP_LAYOUT_NHWC)
    return set_error(TP_ERR_INVALID_ARGUMENT, "bad layout %d", layout);
  if (dtype != TP_DTYPE_NONE && (!out || !lut))
    return set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile: normalized output needs out and lut");
  if (dtype == TP_DTYPE_NONE && !out_u8)
    return set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile: nothing to write");
  if (cap < 0) return set_error(TP_ERR_INVALID_ARGUMENT, "bad out_capacity");
  if (n > 0 && cap > 0 && (!src || !src_off || !wh))
    return set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile: null buffer");
  return TP_OK;
}

}  // namespace
}  // namespace tp

extern "C" int tp_tile(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                       int32_t n, int32_t channels, const int32_t* d_plan,
                       const int32_t* d_tile_off, int32_t tile_edge, const void* d_lut,
                       int32_t dtype, int32_t layout, void* d_out, uint8_t* d_out_u8,
                       int64_t out_capacity, void* stream) {
  return tp_tile_ex(d_src, d_src_off, d_wh, n, channels, d_plan, d_tile_off, tile_edge, d_lut,
                    dtype, layout, d_out, d_out_u8, out_capacity, TP_TILE_ALGO_AUTO, stream);
}

extern "C" int tp_plan_tile(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                            int32_t n, int32_t channels, int32_t tile_edge, int32_t max_tiles,
                            int32_t* d_plan, int32_t* d_n_img, int32_t* d_tile_off,
                            const void* d_lut, int32_t dtype, int32_t layout, void* d_out,
                            uint8_t* d_out_u8, int64_t out_capacity, int32_t algo,
                            void* stream) {
  if (n < 0 || n > TP_PLAN_TILE_MAX_IMAGES)
    return tp::set_error(TP_ERR_UNSUPPORTED, "tp_plan_tile: n = %d outside [0, %d] (use tp_plan + tp_tile_ex)",
                         n, TP_PLAN_TILE_MAX_IMAGES);
  if ((algo & 0xFF) == TP_TILE_ALGO_EXACT || (algo & TP_TILE_AFTER_PLAN))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_plan_tile: fast algorithm only, no AFTER_PLAN");
  if (max_tiles < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "max_tiles must be >= 1");
  if (max_tiles > TP_MAX_TILES_LIMIT)
    return tp::set_error(TP_ERR_UNSUPPORTED, "max_tiles %d above the exact-planner limit %d",
                         max_tiles, TP_MAX_TILES_LIMIT);
  if (tile_edge >= 1 && static_cast<int64_t>(tile_edge) * max_tiles > INT32_MAX)
    return tp::set_error(TP_ERR_UNSUPPORTED, "tile_edge * max_tiles overflows int32");
  if (!d_tile_off || (n > 0 && (!d_wh || !d_plan || !d_n_img)))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_plan_tile: null plan buffer");
  int rc = tp::check_tile_args(d_src, d_src_off, d_wh, n, channels, tile_edge, d_lut, dtype,
                               layout, d_out, d_out_u8, out_capacity, algo);
  if (rc != TP_OK) return rc;
  cudaStream_t s = tp::as_stream(stream);
  if (n == 0 || out_capacity == 0)  // nothing to tile: the plans alone (K1)
    return tp_plan(d_wh, n, tile_edge, max_tiles, d_plan, d_n_img, d_tile_off, stream);
  tp::K2Options fuse;
  fuse.max_tiles = max_tiles;
  fuse.n_img = d_n_img;
  if (channels == 3)
    return tp::dispatch_tile<3>(d_src, d_src_off, d_wh, n, d_plan, d_tile_off, tile_edge, d_lut,
                                dtype, layout, d_out, d_out_u8, out_capacity, algo, s, fuse);
  return tp::dispatch_tile<1>(d_src, d_src_off, d_wh, n, d_plan, d_tile_off, tile_edge, d_lut,
                              dtype, layout, d_out, d_out_u8, out_capacity, algo, s, fuse);
}

extern "C" int tp_tile_rows(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                            int32_t n, int32_t channels, const int32_t* d_plan,
                            const int32_t* d_tile_off, int32_t tile_edge, const void* d_lut,
                            int32_t dtype, int32_t layout, void* d_out, uint8_t* d_out_u8,
                            int64_t out_capacity, int32_t algo, const int32_t* d_row_map,
                            const int64_t* d_row_map_off, void* stream) {
  if ((algo & 0xFF) == TP_TILE_ALGO_EXACT)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile_rows: fast algorithm only");
  const int rc = tp::check_tile_args(d_src, d_src_off, d_wh, n, channels, tile_edge, d_lut, dtype,
                                     layout, d_out, d_out_u8, out_capacity, algo);
  if (rc != TP_OK) return rc;
  if (n == 0 || out_capacity == 0) return TP_OK;
  if (!d_plan || !d_tile_off || !d_row_map || !d_row_map_off)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile_rows: null buffer");
  tp::K2Options opt;
  opt.row_map = d_row_map;
  opt.row_map_off = d_row_map_off;
  cudaStream_t s = tp::as_stream(stream);
  if (channels == 3)
    return tp::dispatch_tile<3>(d_src, d_src_off, d_wh, n, d_plan, d_tile_off, tile_edge, d_lut,
                                dtype, layout, d_out, d_out_u8, out_capacity, algo, s, opt);
  return tp::dispatch_tile<1>(d_src, d_src_off, d_wh, n, d_plan, d_tile_off, tile_edge, d_lut,
                              dtype, layout, d_out, d_out_u8, out_capacity, algo, s, opt);
}

extern "C" int tp_tile_ex(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                          int32_t n, int32_t channels, const int32_t* d_plan,
                          const int32_t* d_tile_off, int32_t tile_edge, const void* d_lut,
                          int32_t dtype, int32_t layout, void* d_out, uint8_t* d_out_u8,
                          int64_t out_capacity, int32_t algo, void* stream) {
  const int rc = tp::check_tile_args(d_src, d_src_off, d_wh, n, channels, tile_edge, d_lut, dtype,
                                     layout, d_out, d_out_u8, out_capacity, algo);
  if (rc != TP_OK) return rc;
  if (n == 0 || out_capacity == 0) return TP_OK;
  if (!d_plan || !d_tile_off) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tile: null buffer");
  cudaStream_t s = tp::as_stream(stream);
  if (channels == 3)
    return tp::dispatch_tile<3>(d_src, d_src_off, d_wh, n, d_plan, d_tile_off, tile_edge, d_lut,
                                dtype, layout, d_out, d_out_u8, out_capacity, algo, s);
  return tp::dispatch_tile<1>(d_src, d_src_off, d_wh, n, d_plan, d_tile_off, tile_edge, d_lut,
                              dtype, layout, d_out, d_out_u8, out_capacity, algo, s);
}

extern "C" int tp_resize(const uint8_t* d_src, int32_t width, int32_t height, int32_t channels,
                         int32_t out_w, int32_t out_h, uint8_t* d_dst, void* stream) {
  if (width < 1 || height < 1)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "image dimensions must be >= 1");
  if (out_w < 1 || out_h < 1)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "output dimensions must be >= 1");
  if (channels != 1 && channels != 3)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "channels must be 1 or 3, got %d", channels);
  if (!d_src || !d_dst) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_resize: null buffer");
  const int grid = min(out_h, 8 * max(1, tp::device_sm_count()));
  cudaStream_t s = tp::as_stream(stream);
  if (channels == 3)
    tp::k_resize_exact<3><<<grid, tp::kThreads, 0, s>>>(d_src, width, height, out_w, out_h, d_dst);
  else
    tp::k_resize_exact<1><<<grid, tp::kThreads, 0, s>>>(d_src, width, height, out_w, out_h, d_dst);
  return tp::check_launch("tp_resize");
}
