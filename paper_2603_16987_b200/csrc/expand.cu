// K3 — image-placeholder expansion + supervision mask for batched prompts.
//
// Replaces expand_image_placeholders (tokenizer.py:294-315), _first_assistant
// (:318-322) and build_supervision_mask (:410-418):
//   each marker id becomes counts[k] * tokens_per_tile context ids; spans are
//   (start, length) in the sequence's output coordinates; the first assistant
//   header index t is found in the output; mask[i] = i >= t && ids[i] != asst.
//
// Three launches (all graph-capturable, no host round trip):
//   k_expand_stats: one warp per sequence, 32 ids per step: ballots count the markers,
//                   a warp scan of the per-id length deltas places the first assistant
//                   header in output coordinates, the marker/count contract is checked;
//                   the sequence's output length goes to the workspace (int64)
//   k_expand_size : one CTA block-scans the lengths into out_off (int64 carry,
//                   capacity-checked)
//   k_expand_fill : CTA per sequence; block scans of (is_marker, length) give
//                   each input token its output position; text ids are
//                   scattered, marker runs are filled cooperatively by the
//                   whole block (coalesced), spans and mask written alongside.

#include "tp_common.cuh"

namespace tp {
namespace {

constexpr int kSizeThreads = 1024;
constexpr int kFillThreads = 256;

constexpr int kStatsThreads = 256;

__global__ void __launch_bounds__(kStatsThreads)
    k_expand_stats(const int32_t* __restrict__ ids, const int32_t* __restrict__ seq_off,
                   int n_seq, const int32_t* __restrict__ counts,
                   const int32_t* __restrict__ count_off, int tpt, int marker, int asst,
                   int64_t* __restrict__ out_len, int32_t* __restrict__ first_asst,
                   int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < n_seq; s += warps) {
    const int b = seq_off[s], e = seq_off[s + 1];
    const int cb = count_off[s], nc = count_off[s + 1] - cb;
    int m = 0, e_flags = 0;           // markers seen before this step
    int64_t delta = 0, first = -1;    // output length minus input length so far
    for (int i0 = b; i0 < e; i0 += 32) {
      const int i = i0 + lane;
      const int tok = i < e ? __ldg(ids + i) : -1;
      const bool is_m = i < e && tok == marker;
      const unsigned mk = __ballot_sync(0xffffffffu, is_m);
      const int my_m = m + __popc(mk & ((1u << lane) - 1u));  // this marker's index
      int64_t d = 0;
      if (is_m && my_m < nc) {
        const int cnt = __ldg(counts + cb + my_m);
        if (cnt < 0) e_flags |= TP_EXPAND_ERR_OVERFLOW;
        d = static_cast<int64_t>(cnt) * tpt - 1;
      }
      int64_t x = d;  // inclusive warp scan of the deltas
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (first < 0) {
        const unsigned am = __ballot_sync(0xffffffffu, i < e && tok == asst);
        if (am) {
          const int l = __ffs(am) - 1;  // the first assistant header of the sequence
          const int64_t before = __shfl_sync(0xffffffffu, x - d, l);  // deltas before it
          first = (static_cast<int64_t>(i0 + l) - b) + delta + before;
        }
      }
      delta += __shfl_sync(0xffffffffu, x, 31);
      m += __popc(mk);
    }
    e_flags = __reduce_or_sync(0xffffffffu, e_flags);
    if (lane == 0) {
      if (m != nc) e_flags |= TP_EXPAND_ERR_MARKER_COUNT;
      if (first < 0) e_flags |= TP_EXPAND_ERR_NO_ASSISTANT;
      const int64_t len = (e - b) + delta;
      if (len > INT32_MAX) e_flags |= TP_EXPAND_ERR_OVERFLOW;
      err[s] = e_flags;
      first_asst[s] = first < 0 || first > INT32_MAX ? -1 : static_cast<int32_t>(first);
      out_len[s] = e_flags ? 0 : len;
    }
  }
}

__global__ void __launch_bounds__(kSizeThreads)
    k_expand_size(const int64_t* __restrict__ out_len, int n_seq, int64_t capacity,
                  int32_t* __restrict__ out_off) {
  __shared__ int64_t s_scan[33];
  int64_t carry = 0;
  bool overflow = false;
  for (int base = 0; base < n_seq; base += kSizeThreads) {
    const int s = base + threadIdx.x;
    const int64_t len = s < n_seq ? out_len[s] : 0;
    int64_t total;
    const int64_t ex = block_exclusive_scan<int64_t>(len, s_scan, &total);
    if (s < n_seq) {
      const int64_t off = carry + ex;
      if (off > INT32_MAX) overflow = true;
      out_off[s] = static_cast<int32_t>(off);
    }
    carry += total;
  }
  overflow = __syncthreads_or(overflow);
  if (threadIdx.x == 0)
    out_off[n_seq] = (overflow || carry > capacity || carry > INT32_MAX)
                         ? -1 : static_cast<int32_t>(carry);
}

__global__ void __launch_bounds__(kFillThreads)
    k_expand_fill(const int32_t* __restrict__ ids, const int32_t* __restrict__ seq_off,
                  int n_seq, const int32_t* __restrict__ counts,
                  const int32_t* __restrict__ count_off, int tpt, int marker, int ctx, int asst,
                  int with_mask, const int32_t* __restrict__ out_off,
                  const int32_t* __restrict__ first_asst, const int32_t* __restrict__ err,
                  int32_t* __restrict__ out_ids, int32_t* __restrict__ spans,
                  uint8_t* __restrict__ mask) {
  __shared__ int32_t s_scan[33];
  __shared__ int32_t s_run_pos[kFillThreads];
  __shared__ int32_t s_run_len[kFillThreads];
  if (__ldg(out_off + n_seq) < 0) return;  // capacity/overflow: nothing is written
  const uint8_t ctx_mask_ok = (ctx != asst) ? 1 : 0;
  for (int s = blockIdx.x; s < n_seq; s += gridDim.x) {
    if (__ldg(err + s) != 0) continue;  // block-uniform
    const int b = seq_off[s], e = seq_off[s + 1];
    const int cb = count_off[s];
    const int t = first_asst[s];
    const int64_t obase = out_off[s];
    int carry_pos = 0, carry_m = 0;
    for (int base = b; base < e; base += kFillThreads) {
      const int i = base + threadIdx.x;
      const bool valid = i < e;
      const int tok = valid ? __ldg(ids + i) : 0;
      const int is_m = (valid && tok == marker) ? 1 : 0;
      int n_runs;
      const int m_idx = block_exclusive_scan<int32_t>(is_m, s_scan, &n_runs);
      const int len = is_m ? __ldg(counts + cb + carry_m + m_idx) * tpt : (valid ? 1 : 0);
      int chunk_len;
      const int pos = carry_pos + block_exclusive_scan<int32_t>(len, s_scan, &chunk_len);
      if (valid && !is_m) {
        out_ids[obase + pos] = tok;
        mask[obase + pos] = (with_mask && pos >= t && tok != asst) ? 1 : 0;
      }
      if (is_m) {
        const int k = cb + carry_m + m_idx;
        spans[2 * static_cast<int64_t>(k)] = pos;
        spans[2 * static_cast<int64_t>(k) + 1] = len;
        s_run_pos[m_idx] = pos;
        s_run_len[m_idx] = len;
      }
      __syncthreads();
      for (int r = 0; r < n_runs; ++r) {
        const int p0 = s_run_pos[r], L = s_run_len[r];
        for (int p = threadIdx.x; p < L; p += kFillThreads) {
          out_ids[obase + p0 + p] = ctx;
          mask[obase + p0 + p] = (with_mask && p0 + p >= t && ctx_mask_ok) ? 1 : 0;
        }
      }
      __syncthreads();
      carry_pos += chunk_len;
      carry_m += n_runs;
    }
  }
}

}  // namespace
}  // namespace tp

extern "C" int64_t tp_expand_workspace_bytes(int32_t n_seq) {
  return n_seq > 0 ? 8 * static_cast<int64_t>(n_seq) : 0;  // per-sequence output lengths
}

extern "C" int tp_expand(const int32_t* d_ids, const int32_t* d_seq_off, int32_t n_seq,
                         const int32_t* d_counts, const int32_t* d_count_off,
                         int32_t tokens_per_tile, int32_t marker_id, int32_t ctx_id,
                         int32_t asst_id, int32_t with_mask, int32_t* d_out_ids,
                         int64_t out_capacity, int32_t* d_out_off, int32_t* d_spans,
                         int32_t* d_first_asst, uint8_t* d_mask, int32_t* d_err, void* d_work,
                         void* stream) {
  if (n_seq < 0) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "n_seq must be >= 0");
  if (tokens_per_tile < 0)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tokens_per_tile must be >= 0");
  if (out_capacity < 0) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "bad out_capacity");
  if (!d_out_off) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_expand: null out_off");
  if (n_seq > 0 && (!d_ids || !d_seq_off || !d_count_off || !d_first_asst || !d_err))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_expand: null buffer");
  if (out_capacity > 0 && (!d_out_ids || !d_mask))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_expand: null output buffer");
  if (n_seq > 0 && !d_work)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT,
                         "tp_expand: null workspace (tp_expand_workspace_bytes(n_seq) bytes)");
  cudaStream_t s = tp::as_stream(stream);
  int64_t* lens = static_cast<int64_t*>(d_work);
  if (n_seq > 0) {
    const int grid = std::min<int>((n_seq + 7) / 8, 16 * std::max(1, tp::device_sm_count()));
    tp::k_expand_stats<<<grid, tp::kStatsThreads, 0, s>>>(
        d_ids, d_seq_off, n_seq, d_counts, d_count_off, tokens_per_tile, marker_id, asst_id,
        lens, d_first_asst, d_err);
  }
  tp::k_expand_size<<<1, tp::kSizeThreads, 0, s>>>(lens, n_seq, out_capacity, d_out_off);
  int rc = tp::check_launch("tp_expand(size)");
  if (rc != TP_OK || n_seq == 0) return rc;
  const int grid = std::min<int>(n_seq, 16 * std::max(1, tp::device_sm_count()));
  tp::k_expand_fill<<<grid, tp::kFillThreads, 0, s>>>(
      d_ids, d_seq_off, n_seq, d_counts, d_count_off, tokens_per_tile, marker_id, ctx_id,
      asst_id, with_mask, d_out_off, d_first_asst, d_err, d_out_ids, d_spans, d_mask);
  return tp::check_launch("tp_expand(fill)");
}

namespace tp {
namespace {
// build_supervision_mask law for an already-expanded sequence with a given t
// (tokenizer.py:410-418): mask[i] = i >= t && ids[i] != asst.
__global__ void __launch_bounds__(256)
    k_supervision_mask(const int32_t* __restrict__ ids, int64_t n, int64_t t, int asst,
                       uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mask[i] = (i >= t && __ldg(ids + i) != asst) ? 1 : 0;
}
}  // namespace
}  // namespace tp

extern "C" int tp_supervision_mask(const int32_t* d_ids, int64_t n, int64_t first_asst,
                                   int32_t asst_id, uint8_t* d_mask, void* stream) {
  if (n < 0) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "negative length");
  if (first_asst < 0 || first_asst > n)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "first_assistant_index %lld outside [0, %lld]",
                         static_cast<long long>(first_asst), static_cast<long long>(n));
  if (n == 0) return TP_OK;
  if (!d_ids || !d_mask) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "null buffer");
  const int64_t want = (n + 255) / 256;
  const int grid = static_cast<int>(std::min<int64_t>(want, 16LL * std::max(1, tp::device_sm_count())));
  tp::k_supervision_mask<<<grid, 256, 0, tp::as_stream(stream)>>>(d_ids, n, first_asst, asst_id,
                                                                 d_mask);
  return tp::check_launch("tp_supervision_mask");
}
