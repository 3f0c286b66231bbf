// pixel_unshuffle (tokenred.py:80-103): fold every r x r neighbourhood of patch
// feature vectors into the channel dimension.  Output cell (i, j) is the
// concatenation of input cells (i*r + a, j*r + b), a outer, b inner, so the op
// moves whole d-element vectors: out vector ((i*(w/r) + j)*r + a)*r + b <- in
// vector (i*r + a)*w + j*r + b.  Pure data movement, HBM-bound: one warp copies
// one vector with the widest aligned accesses the element size and d allow.

#include "tp_common.cuh"

namespace tp {
namespace {

template <typename V>
__global__ void __launch_bounds__(256)
    k_unshuffle(const V* __restrict__ in, V* __restrict__ out, int h, int w, int r,
                int64_t vec_words) {
  const int ow = w / r;
  const int64_t n_vec = static_cast<int64_t>(h) * w;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t o = warp; o < n_vec; o += nwarps) {
    // o = ((i*ow + j)*r + a)*r + b
    const int64_t b = o % r;
    const int64_t t1 = o / r;
    const int64_t a = t1 % r;
    const int64_t cell = t1 / r;
    const int64_t i = cell / ow, j = cell - i * ow;
    const int64_t src = (i * r + a) * w + j * r + b;
    const V* s = in + src * vec_words;
    V* d = out + o * vec_words;
    for (int64_t k = lane; k < vec_words; k += 32) d[k] = s[k];
  }
}

template <typename V>
int launch_unshuffle(const void* in, void* out, int h, int w, int r, int64_t words,
                     cudaStream_t s) {
  const int64_t n_vec = static_cast<int64_t>(h) * w;
  const int64_t want = (n_vec * 32 + 255) / 256;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
      want, 16LL * std::max(1, device_sm_count()))));
  k_unshuffle<V><<<grid, 256, 0, s>>>(static_cast<const V*>(in), static_cast<V*>(out), h, w, r,
                                      words);
  return check_launch("tp_pixel_unshuffle");
}

}  // namespace
}  // namespace tp

extern "C" int tp_pixel_unshuffle(const void* d_in, int32_t h, int32_t w, int64_t d,
                                  int32_t elem_bytes, int32_t r, void* d_out, void* stream) {
  if (r < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "reduction factor must be >= 1, got %d", r);
  if (h < 1 || w < 1 || d < 1 || elem_bytes < 1)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "grid dimensions must be positive");
  if (h % r || w % r)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "reduction factor %d does not divide grid (%d, %d)",
                         r, h, w);
  if (!d_in || !d_out) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "null buffer");
  const int64_t vec_bytes = d * elem_bytes;
  const uintptr_t align = reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out);
  cudaStream_t s = tp::as_stream(stream);
  if (vec_bytes % 16 == 0 && align % 16 == 0)
    return tp::launch_unshuffle<uint4>(d_in, d_out, h, w, r, vec_bytes / 16, s);
  if (vec_bytes % 8 == 0 && align % 8 == 0)
    return tp::launch_unshuffle<uint2>(d_in, d_out, h, w, r, vec_bytes / 8, s);
  if (vec_bytes % 4 == 0 && align % 4 == 0)
    return tp::launch_unshuffle<uint32_t>(d_in, d_out, h, w, r, vec_bytes / 4, s);
  return tp::launch_unshuffle<uint8_t>(d_in, d_out, h, w, r, vec_bytes, s);
}
