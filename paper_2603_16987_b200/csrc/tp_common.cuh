// Shared helpers for the tileprep kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <algorithm>

#include "tileprep.h"

namespace tp {

// ---------------------------------------------------------------------------
// error plumbing: thread-local message, int return codes (include/tileprep.h)

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
int device_sm_count();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (K1 -> K2 -> next K1): the kernel may be scheduled
// while its stream predecessor is still running; it must call pdl_wait() before it
// reads anything a predecessor wrote or writes anything a predecessor reads.
// pdl_trigger() lets the stream successor be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------------------
// exact half-pixel axis sampling, restating _axis_weights (imgproc.py:298-306):
//   pos = (i + 0.5) * (src / out) - 0.5, clipped to [0, src-1]
//   i0  = min(floor(pos), src-1);  frac = pos - i0;  i1 = min(i0+1, src-1)
// Every operation is an explicitly rounded fp64 intrinsic so nvcc can never
// contract it into an FMA (the reference relies on the uncontracted order).

struct AxisTap {
  int i0, i1;
  double f;    // frac
  double omf;  // 1.0 - frac, rounded (the reference computes `1.0 - fyc` in fp64)
};

__device__ __forceinline__ double axis_scale(int src, int out) {
  return __ddiv_rn(static_cast<double>(src), static_cast<double>(out));
}

__device__ __forceinline__ AxisTap axis_tap(int i, int src, double scale) {
  double pos = __dadd_rn(__dmul_rn(static_cast<double>(i) + 0.5, scale), -0.5);
  pos = fmin(fmax(pos, 0.0), static_cast<double>(src - 1));
  // floor(pos) for 0 <= pos < 2^52 without the slow F2I/I2F conversions:
  // pos + 2^52 rounded toward -inf is exactly 2^52 + floor(pos)
  const double big = __dadd_rd(pos, 4503599627370496.0);
  const int i0 = min(__double2loint(big), src - 1);  // clip already keeps floor <= src-1
  const double fl = __dsub_rn(big, 4503599627370496.0);
  AxisTap t;
  t.i0 = i0;
  t.i1 = min(i0 + 1, src - 1);
  t.f = __dsub_rn(pos, fl);  // pos - i0, exact (the reference's frac)
  t.omf = __dsub_rn(1.0, t.f);
  return t;
}

// Bilinear sample of one channel in the reference order (imgproc.py:309-335):
// vertical blend first, each product and sum rounded separately, then
// _to_uint8 rounding floor(v + 0.5) clipped to [0, 255] (imgproc.py:338-349).
__device__ __forceinline__ uint32_t blend_exact(uint32_t s00, uint32_t s01, uint32_t s10,
                                                uint32_t s11, const AxisTap& ty,
                                                const AxisTap& tx) {
  const double l = __dadd_rn(__dmul_rn(static_cast<double>(s00), ty.omf),
                             __dmul_rn(static_cast<double>(s10), ty.f));
  const double r = __dadd_rn(__dmul_rn(static_cast<double>(s01), ty.omf),
                             __dmul_rn(static_cast<double>(s11), ty.f));
  const double v = __dadd_rn(__dmul_rn(l, tx.omf), __dmul_rn(r, tx.f));
  double q = floor(__dadd_rn(v, 0.5));
  q = fmin(fmax(q, 0.0), 255.0);
  return static_cast<uint32_t>(q);
}

// ---------------------------------------------------------------------------
// output element types

template <typename T>
struct OutTraits;
template <>
struct OutTraits<float> {
  static constexpr int kDtype = TP_DTYPE_F32;
};
template <>
struct OutTraits<__nv_bfloat16> {
  static constexpr int kDtype = TP_DTYPE_BF16;
};

// ---------------------------------------------------------------------------
// block-wide exclusive scan (blockDim.x a multiple of 32, <= 1024)

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// returns the exclusive prefix of v; *total receives the block sum.
// `scratch` must hold 33 elements of T.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* scratch, T* total) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nwarps ? scratch[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < nwarps) scratch[lane] = wi - w;  // exclusive warp offsets
    if (lane == nwarps - 1) scratch[32] = wi;   // block total (nwarps <= 32)
  }
  __syncthreads();
  T res = scratch[warp] + inc - v;
  if (total) *total = scratch[32];
  __syncthreads();
  return res;
}

// K2 launch options beyond tp_tile_ex's arguments.
//  * fused small-batch mode (tp_plan_tile): max_tiles > 0 makes every CTA plan the
//    batch itself (K1's rule, plan_core.cuh) instead of reading K1's output; CTA 0
//    writes the plans, per-image counts (n_img) and tile offsets for the caller;
//  * touched-row input (tp_tile_rows): row_map != nullptr means image k's pixel block
//    holds only its touched rows; row y is at compact index
//    row_map[row_map_off[k] + 1 + y] (tp_touched_rows).
constexpr int kFuseMaxImages = TP_PLAN_TILE_MAX_IMAGES;
struct K2Options {
  int max_tiles = 0;  // 0: plans come from a preceding tp_plan
  int32_t* n_img = nullptr;
  const int32_t* row_map = nullptr;
  const int64_t* row_map_off = nullptr;
};

// K2 fast path (tile_tma.cu): TMA-staged fp32 kernel with exact fallback
template <int C, typename OutT, int LAYOUT, bool WRITE_OUT>
int launch_tile_tma(const uint8_t* src, const int64_t* src_off, const int32_t* wh, int n,
                    const int32_t* plan, const int32_t* tile_off, int E, const void* lut,
                    void* out, uint8_t* out_u8, int64_t cap, bool affine, bool after_plan,
                    cudaStream_t stream, K2Options fuse = K2Options{});

}  // namespace tp
