// K6 — greedy longest-match tokenizer, batched (replaces tokenize, tokenizer.py:135-158).
//
// The reference walks each text left to right: at `pos` it takes the longest
// vocabulary entry (at most max_token_bytes long) that matches the bytes starting at
// `pos`, else the byte-fallback token of data[pos], and jumps past it.  The longest
// match *at a position* does not depend on where the walk came from, so it is computed
// for every byte position of every text in parallel (K6a: one thread per position,
// hash probes from the longest candidate down); the walk itself is then a chain of
// jumps through that table (K6b: one thread per text), and K6c/K6d compact the ids.
//
// Vocabulary table (built on the host by tp_vocab_build, see include/tileprep.h):
//   TpVocabHeader, int32 byte_ids[256], TpVocabSlot slots[n_slots] (open addressing,
//   linear probing, key = token bytes zero-padded to 16 + length).

#include "tp_common.cuh"

#include <cstring>

namespace tp {
namespace {

struct TpVocabHeader {
  uint32_t magic;
  int32_t n_slots;  // power of two
  int32_t max_len;  // longest non-byte token (bytes)
  int32_t n_tokens;
};
struct TpVocabSlot {
  uint64_t k0, k1;  // token bytes, little-endian, zero padded
  int32_t id;       // -1: empty slot
  int32_t len;
};
constexpr uint32_t kVocabMagic = 0x544F4B31u;  // "TOK1"
constexpr int kMaxTokenBytes = 16;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
__host__ __device__ __forceinline__ uint32_t key_hash(uint64_t k0, uint64_t k1, int len) {
  return static_cast<uint32_t>(mix64(k0 ^ mix64(k1 + 0x9E3779B97F4A7C15ULL * (len + 1))));
}

size_t table_bytes(int n_slots) {
  return sizeof(TpVocabHeader) + 256 * sizeof(int32_t) + static_cast<size_t>(n_slots) * sizeof(TpVocabSlot);
}
int slots_for(int n_tokens) {
  int s = 16;
  while (s < 2 * n_tokens) s <<= 1;
  return s;
}

// K6a: longest match at every byte position (one block per text, threads stride the text)
__global__ void k_tok_match(const uint8_t* __restrict__ vocab, const uint8_t* __restrict__ text,
                            const int64_t* __restrict__ text_off, int n_texts,
                            int32_t* __restrict__ m_id, uint8_t* __restrict__ m_len) {
  const TpVocabHeader* hdr = reinterpret_cast<const TpVocabHeader*>(vocab);
  const int32_t* byte_ids = reinterpret_cast<const int32_t*>(vocab + sizeof(TpVocabHeader));
  const TpVocabSlot* slots =
      reinterpret_cast<const TpVocabSlot*>(vocab + sizeof(TpVocabHeader) + 256 * sizeof(int32_t));
  const uint32_t mask = static_cast<uint32_t>(hdr->n_slots - 1);
  const int max_len = hdr->max_len;
  for (int t = blockIdx.x; t < n_texts; t += gridDim.x) {
    const int64_t beg = text_off[t], end = text_off[t + 1];
    for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
      const int64_t left = end - i;
      const int avail = left < max_len ? static_cast<int>(left) : max_len;
      uint8_t b[kMaxTokenBytes];
#pragma unroll
      for (int k = 0; k < kMaxTokenBytes; ++k) b[k] = k < avail ? text[i + k] : 0;
      int id = -1, len = 1;
      for (int L = avail; L >= 1 && id < 0; --L) {
        uint64_t k0 = 0, k1 = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          k0 |= static_cast<uint64_t>(k < L ? b[k] : 0) << (8 * k);
          k1 |= static_cast<uint64_t>(k + 8 < L ? b[k + 8] : 0) << (8 * k);
        }
        for (uint32_t h = key_hash(k0, k1, L) & mask;; h = (h + 1) & mask) {
          const TpVocabSlot s = slots[h];
          if (s.id < 0) break;
          if (s.len == L && s.k0 == k0 && s.k1 == k1) {
            id = s.id;
            len = L;
            break;
          }
        }
      }
      if (id < 0) {  // byte fallback (tokenizer.py:150-155); -1 means none: error
        id = byte_ids[b[0]];
        len = 1;
        if (id < 0) id = -0x100 - static_cast<int>(b[0]);
      }
      m_id[i] = id;
      m_len[i] = static_cast<uint8_t>(len);
    }
  }
}

// K6b: the greedy walk through the match table, one warp per text, in segments of
// kSeg bytes (one lane each) so a long text is walked in parallel:
//  (1) every segment walks speculatively from its first byte to its end, recording the
//      rank (tokens before it) of each position it visits;
//  (2) the true walk enters a segment at one of its first kMaxTokenBytes positions (the
//      first boundary at or after its start); for each such candidate entry the lane
//      walks until it lands on a position its speculative walk visited -- greedy walks
//      are deterministic, so from there the speculative tail is the true one (usually
//      one or two tokens) -- giving (exit, token count) per candidate;
//  (3) lane 0 chains the segments: entry of segment j+1 = exit of segment j for its
//      entry (a table lookup per segment), then a warp scan of the counts places every
//      segment's first id, and each lane re-walks its segment writing the ids.
// A byte with neither a token nor a fallback on the true path makes the text an error.
constexpr int kSeg = 256;
constexpr int kCand = kMaxTokenBytes;

struct SegCand {
  int32_t exit[kCand];
  int32_t cnt[kCand];   // tokens from the candidate entry to the exit; -1: error on the path
  int32_t spec_exit, spec_cnt, spec_err;  // the speculative walk from the segment start
};

__device__ __forceinline__ int64_t seg_index(int64_t beg, int t, int j) {
  return beg / kSeg + t + j;  // unique across texts (texts are disjoint byte ranges)
}

__global__ void __launch_bounds__(128) k_tok_walk(const int64_t* __restrict__ text_off, int n_texts,
                                                  const int32_t* __restrict__ m_id,
                                                  const uint8_t* __restrict__ m_len,
                                                  int32_t* __restrict__ rank,
                                                  SegCand* __restrict__ cand,
                                                  int32_t* __restrict__ seg_entry,
                                                  int32_t* __restrict__ stage_ids,
                                                  int32_t* __restrict__ counts,
                                                  int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_texts; t += warps) {
    const int64_t beg = text_off[t], end = text_off[t + 1];
    const int nseg = static_cast<int>((end - beg + kSeg - 1) / kSeg);
    // (1) speculative walks; positions are text-relative (< 2^31)
    for (int j = lane; j < nseg; j += 32) {
      const int64_t q = beg + static_cast<int64_t>(j) * kSeg;
      const int64_t qe = q + kSeg < end ? q + kSeg : end;
      int64_t pos = q;
      int k = 0, bad = 0;
      while (pos < qe) {
        const int id = m_id[pos];
        rank[pos] = id < 0 ? -2 : k;  // -2: the walk stops here (no token, no fallback)
        if (id < 0) {
          bad = 1;
          break;
        }
        ++k;
        pos += m_len[pos];
      }
      SegCand& sc = cand[seg_index(beg, t, j)];
      sc.spec_exit = static_cast<int32_t>(pos - beg);
      sc.spec_cnt = k;
      sc.spec_err = bad;
    }
    __syncwarp();
    // (2) every candidate entry of every segment
    for (int j = lane; j < nseg; j += 32) {
      const int64_t q = beg + static_cast<int64_t>(j) * kSeg;
      const int64_t qe = q + kSeg < end ? q + kSeg : end;
      SegCand& sc = cand[seg_index(beg, t, j)];
      const int64_t sx = beg + sc.spec_exit;  // the speculative walk's own totals
      const int sk = sc.spec_cnt;
      const bool serr = sc.spec_err != 0;
      for (int c = 0; c < kCand; ++c) {
        int64_t pos = q + c;
        int k = 0;
        int out_cnt = -1;
        int64_t out_exit = pos;
        if (pos >= qe) {  // the entry is already past this segment
          out_cnt = 0;
        } else {
          while (true) {
            if (pos >= qe) {
              out_cnt = k;
              out_exit = pos;
              break;
            }
            const int r = rank[pos];
            if (r >= 0) {  // joined the speculative walk
              out_cnt = serr ? -1 : k + sk - r;
              out_exit = sx;
              break;
            }
            const int id = m_id[pos];
            if (id < 0) break;  // error on this path
            ++k;
            pos += m_len[pos];
          }
        }
        sc.exit[c] = static_cast<int32_t>(out_exit - beg);
        sc.cnt[c] = out_cnt;
      }
    }
    __syncwarp();
    // (3) chain the segments (lane 0), scan, write
    int e_code = 0;
    if (lane == 0) {
      int64_t e = beg;
      for (int j = 0; j < nseg; ++j) {
        const int64_t q = beg + static_cast<int64_t>(j) * kSeg;
        if (e >= end) {
          seg_entry[seg_index(beg, t, j)] = -1;  // nothing left to walk
          continue;
        }
        const SegCand& sc = cand[seg_index(beg, t, j)];
        const int c = static_cast<int>(e - q);
        seg_entry[seg_index(beg, t, j)] = static_cast<int32_t>(e - beg);
        if (sc.cnt[c] < 0) {
          // find the offending byte on the true path (the reference raises there)
          int64_t pos = e;
          while (pos < end && m_id[pos] >= 0) pos += m_len[pos];
          e_code = pos < end ? -m_id[pos] : 0x100;
          break;
        }
        e = beg + sc.exit[c];
      }
    }
    e_code = __shfl_sync(0xffffffffu, e_code, 0);
    if (e_code) {
      if (lane == 0) {
        counts[t] = 0;
        err[t] = e_code;
      }
      continue;
    }
    int carry = 0;
    for (int j0 = 0; j0 < nseg; j0 += 32) {
      const int j = j0 + lane;
      int cnt = 0, e_rel = -1;
      if (j < nseg) {
        e_rel = seg_entry[seg_index(beg, t, j)];
        if (e_rel >= 0) {
          const int64_t q = beg + static_cast<int64_t>(j) * kSeg;
          cnt = cand[seg_index(beg, t, j)].cnt[static_cast<int>(beg + e_rel - q)];
        }
      }
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (e_rel >= 0) {
        const int64_t q = beg + static_cast<int64_t>(j) * kSeg;
        const int64_t qe = q + kSeg < end ? q + kSeg : end;
        int64_t pos = beg + e_rel;
        int k = carry + x - cnt;
        while (pos < qe) {
          stage_ids[beg + k++] = m_id[pos];
          pos += m_len[pos];
        }
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      counts[t] = carry;
      err[t] = 0;
    }
  }
}

// K6c: exclusive scan of the counts -> out_off (one CTA); out_off[n] = total
__global__ void __launch_bounds__(1024) k_tok_scan(const int32_t* __restrict__ counts, int n,
                                                   int32_t* __restrict__ out_off) {
  __shared__ int64_t scratch[33];
  int64_t carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int64_t v = i < n ? counts[i] : 0;
    int64_t total;
    const int64_t ex = block_exclusive_scan<int64_t>(v, scratch, &total);
    if (i < n) out_off[i] = static_cast<int32_t>(carry + ex);
    carry += total;
  }
  if (threadIdx.x == 0) out_off[n] = carry > INT32_MAX ? -1 : static_cast<int32_t>(carry);
}

// K6d: compaction (one block per text)
__global__ void k_tok_compact(const int64_t* __restrict__ text_off, int n_texts,
                              const int32_t* __restrict__ stage_ids,
                              const int32_t* __restrict__ out_off, int32_t* __restrict__ out_ids) {
  if (out_off[n_texts] < 0) return;
  for (int t = blockIdx.x; t < n_texts; t += gridDim.x) {
    const int64_t src = text_off[t];
    const int dst = out_off[t], cnt = out_off[t + 1] - out_off[t];
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) out_ids[dst + k] = stage_ids[src + k];
  }
}

}  // namespace
}  // namespace tp

extern "C" int64_t tp_vocab_table_bytes(int32_t n_tokens) {
  if (n_tokens < 0) return -1;
  return static_cast<int64_t>(tp::table_bytes(tp::slots_for(n_tokens)));
}

extern "C" int tp_vocab_build(const uint8_t* tok_bytes, const int32_t* tok_off,
                              const int32_t* tok_id, int32_t n_tokens, const int32_t* byte_ids,
                              void* host_table, int64_t table_bytes) {
  if (n_tokens < 0 || (n_tokens > 0 && (!tok_bytes || !tok_off || !tok_id)) || !byte_ids ||
      !host_table)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_vocab_build: bad arguments");
  const int slots = tp::slots_for(n_tokens);
  if (table_bytes < static_cast<int64_t>(tp::table_bytes(slots)))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_vocab_build: table needs %lld bytes",
                         static_cast<long long>(tp::table_bytes(slots)));
  uint8_t* base = static_cast<uint8_t*>(host_table);
  auto* hdr = reinterpret_cast<tp::TpVocabHeader*>(base);
  auto* bids = reinterpret_cast<int32_t*>(base + sizeof(tp::TpVocabHeader));
  auto* tab = reinterpret_cast<tp::TpVocabSlot*>(base + sizeof(tp::TpVocabHeader) + 256 * sizeof(int32_t));
  for (int s = 0; s < slots; ++s) tab[s] = tp::TpVocabSlot{0, 0, -1, 0};
  std::memcpy(bids, byte_ids, 256 * sizeof(int32_t));
  int max_len = 1;
  for (int i = 0; i < n_tokens; ++i) {
    const int len = tok_off[i + 1] - tok_off[i];
    if (len < 1 || len > tp::kMaxTokenBytes)
      return tp::set_error(TP_ERR_UNSUPPORTED, "token %d has %d bytes (1..%d supported)", i,
                           len, tp::kMaxTokenBytes);
    uint64_t k0 = 0, k1 = 0;
    for (int k = 0; k < len; ++k) {
      const uint64_t v = tok_bytes[tok_off[i] + k];
      if (k < 8) k0 |= v << (8 * k); else k1 |= v << (8 * (k - 8));
    }
    uint32_t h = tp::key_hash(k0, k1, len) & static_cast<uint32_t>(slots - 1);
    while (tab[h].id >= 0) {
      if (tab[h].len == len && tab[h].k0 == k0 && tab[h].k1 == k1)
        return tp::set_error(TP_ERR_INVALID_ARGUMENT, "duplicate token at index %d", i);
      h = (h + 1) & static_cast<uint32_t>(slots - 1);
    }
    tab[h] = tp::TpVocabSlot{k0, k1, tok_id[i], len};
    max_len = len > max_len ? len : max_len;
  }
  *hdr = tp::TpVocabHeader{tp::kVocabMagic, slots, max_len, n_tokens};
  return TP_OK;
}

namespace {
// workspace: match ids | staged ids | walk ranks (int32 per byte) | match lengths (u8 per
// byte) | counts (int32 per text) | per segment: candidates, true entry
int64_t n_segs(int64_t total_bytes, int32_t n_texts) { return total_bytes / tp::kSeg + n_texts + 1; }
int64_t al256(int64_t v) { return (v + 255) & ~int64_t(255); }
}  // namespace

extern "C" int64_t tp_tokenize_workspace_bytes(int64_t total_bytes, int32_t n_texts) {
  if (total_bytes < 0 || n_texts < 0) return -1;
  const int64_t a = al256(total_bytes * 4);
  const int64_t b = al256(total_bytes);
  const int64_t c = al256(static_cast<int64_t>(n_texts) * 4);
  const int64_t segs = n_segs(total_bytes, n_texts);
  return 3 * a + b + c + al256(segs * static_cast<int64_t>(sizeof(tp::SegCand))) + al256(segs * 4);
}

extern "C" int tp_tokenize(const void* d_vocab, const uint8_t* d_text, const int64_t* d_text_off,
                           int32_t n_texts, int64_t total_bytes, int32_t* d_out_ids,
                           int32_t* d_out_off, int32_t* d_err, void* d_workspace,
                           int64_t workspace_bytes, void* stream) {
  if (n_texts < 0 || total_bytes < 0)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tokenize: negative size");
  if (!d_vocab || !d_text_off || !d_out_off || (n_texts > 0 && !d_err))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tokenize: null buffer");
  if (workspace_bytes < tp_tokenize_workspace_bytes(total_bytes, n_texts) || !d_workspace)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tokenize: workspace too small");
  if (total_bytes > INT32_MAX)
    return tp::set_error(TP_ERR_UNSUPPORTED, "tp_tokenize: more than 2^31 bytes per batch");
  cudaStream_t s = tp::as_stream(stream);
  uint8_t* ws = static_cast<uint8_t*>(d_workspace);
  const int64_t a = al256(total_bytes * 4);
  const int64_t b = al256(total_bytes);
  const int64_t c = al256(static_cast<int64_t>(n_texts) * 4);
  const int64_t segs = n_segs(total_bytes, n_texts);
  int32_t* m_id = reinterpret_cast<int32_t*>(ws);
  int32_t* stage = reinterpret_cast<int32_t*>(ws + a);
  int32_t* rank = reinterpret_cast<int32_t*>(ws + 2 * a);
  uint8_t* m_len = ws + 3 * a;
  int32_t* counts = reinterpret_cast<int32_t*>(ws + 3 * a + b);
  auto* cand = reinterpret_cast<tp::SegCand*>(ws + 3 * a + b + c);
  int32_t* seg_entry = reinterpret_cast<int32_t*>(ws + 3 * a + b + c +
                                                  al256(segs * static_cast<int64_t>(sizeof(tp::SegCand))));
  if (n_texts > 0) {
    const int sms = std::max(1, tp::device_sm_count());
    if (total_bytes > 0) {
      if (!d_text || !d_out_ids)
        return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_tokenize: null text/out buffer");
      tp::k_tok_match<<<std::min(n_texts, 16 * sms), 128, 0, s>>>(
          static_cast<const uint8_t*>(d_vocab), d_text, d_text_off, n_texts, m_id, m_len);
    }
    if (total_bytes > 0 && cudaMemsetAsync(rank, 0xFF, 4 * total_bytes, s) != cudaSuccess)
      return tp::set_error(TP_ERR_CUDA, "tp_tokenize: memset failed");
    tp::k_tok_walk<<<std::min<int>((n_texts + 3) / 4, 16 * sms), 128, 0, s>>>(
        d_text_off, n_texts, m_id, m_len, rank, cand, seg_entry, stage, counts, d_err);
  }
  tp::k_tok_scan<<<1, 1024, 0, s>>>(counts, n_texts, d_out_off);
  if (n_texts > 0 && total_bytes > 0) {
    const int sms = std::max(1, tp::device_sm_count());
    tp::k_tok_compact<<<std::min(n_texts, 8 * sms), 128, 0, s>>>(d_text_off, n_texts, stage,
                                                                 d_out_off, d_out_ids);
  }
  return tp::check_launch("tp_tokenize");
}
