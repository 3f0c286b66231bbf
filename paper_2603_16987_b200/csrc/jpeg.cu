// K7 — device JPEG decode for sm_100a.
//
// Replaces the PIL decode in decode_image / _decode_pass (imgproc.py:213-260) for
// baseline JPEGs, bit-exact with the libjpeg-turbo Pillow uses (oracle/jpeg_oracle.py
// restates it and is pinned to Pillow):
//
//   J1 k_jpeg_unstuff  one CTA per image: drop the 0x00 after every data 0xFF, cut the
//                      entropy-coded data at its RST markers (block scans), so each
//                      restart interval is a plain bit string
//   J2 k_jpeg_huff     cooperative grid, every image's intervals cut into subsequences of
//                      sub_bits bits, one thread each (Huffman codes self-synchronize):
//                      (1) every subsequence decodes speculatively from a guessed state;
//                      (2) rounds: subsequence j re-decodes from subsequence j-1's exit
//                          state (bit position, block slot in the MCU, zigzag index) until
//                          no exit changes -- typically two rounds;
//                      (3) per interval, a scan of the blocks each subsequence completes
//                          gives its first block index;
//                      (4) every subsequence decodes once more, writing its coefficients;
//                      (5) DC prediction: per interval and component, a warp scan of the
//                          DC differences (int16 like libjpeg's JCOEF)
//   J3 k_jpeg_idct     jidctint.c jpeg_idct_islow, 8 threads per block, 64-bit JLONG
//                      arithmetic as libjpeg's on LP64, the jdmaster.c range-limit table
//   J4 k_jpeg_color    jdsample.c fancy upsampling (h2v1 / h2v2, edge replication of
//                      jdmainct.c's context rows) + jdcolor.c ycc_rgb_convert into RGB HWC
//                      uint8 -- the packed-image layout K2 reads
//
// Anything the decoder finds unclean (a bad Huffman code, data that ends before the last
// MCU, a marker other than RST, a coefficient index past 63) marks the image in d_status;
// the caller decodes that one on the host, as the reference does.

#include <cooperative_groups.h>

#include "jpeg_common.cuh"
#include "tp_common.cuh"

namespace cg = cooperative_groups;

namespace tp {
namespace {

using jpeg::JDesc;
using jpeg::JHuff;

__constant__ uint8_t c_zig[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                  12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                  35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                  58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

constexpr int kMaxSteps = 160;  // sync half-rounds before an image is handed to the host
constexpr int kNoErr = 0x7FFFFFFF;

struct Work {
  unsigned* counters;  // [h]: exits changed in half-round h
  long long* exitp;    // per slot: (bit << 16) | (u << 8) | z, bit relative to the interval
  int* blocks;         // blocks completed from the (last) entry to the exit
  int* err;            // block count at the first unclean symbol, kNoErr if none
  int* bstart;         // block index (in the image) at the entry
  int* lastproc;       // half-round this slot last decoded in
  int* changed;        // half-round its exit last changed in
};

__host__ __device__ inline int64_t al256(int64_t v) { return (v + 255) & ~int64_t(255); }

__device__ inline Work work_view(uint8_t* w, int64_t slots) {
  Work v;
  v.counters = reinterpret_cast<unsigned*>(w);
  int64_t o = 4096;
  v.exitp = reinterpret_cast<long long*>(w + o);
  o += al256(8 * slots);
  int* arrs[5];
  for (int i = 0; i < 5; ++i) {
    arrs[i] = reinterpret_cast<int*>(w + o);
    o += al256(4 * slots);
  }
  v.blocks = arrs[0];
  v.err = arrs[1];
  v.bstart = arrs[2];
  v.lastproc = arrs[3];
  v.changed = arrs[4];
  return v;
}

__device__ inline int find_image(const JDesc* d, int n, int64_t g, int which) {
  // largest k with base(k) <= g; which: 0 slot_base, 1 block_base, 2 row_base
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    const int64_t b = which == 0 ? d[mid].slot_base : which == 1 ? d[mid].block_base : d[mid].row_base;
    if (b <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// J1: unstuff

__device__ inline unsigned block_excl_scan(unsigned v, unsigned* sh, unsigned& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned t = lane < nw ? sh[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    if (lane < nw) sh[lane] = t;
  }
  __syncthreads();
  const unsigned before = (warp ? sh[warp - 1] : 0u) + x - v;
  total = sh[nw - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(512) k_jpeg_unstuff(const uint8_t* __restrict__ payload,
                                                      const JDesc* __restrict__ descs, int n,
                                                      uint8_t* __restrict__ work,
                                                      int32_t* __restrict__ status) {
  __shared__ unsigned sh[32];
  __shared__ unsigned carry_kept, carry_rst, bad;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const JDesc& d = descs[k];
    if (d.n_slots == 0) continue;
    const uint8_t* raw = payload + d.raw_off;
    const int64_t len = d.raw_len;
    uint8_t* clean = work + d.clean_off;
    int32_t* seg_start = reinterpret_cast<int32_t*>(work + d.seg_off);
    if (threadIdx.x == 0) {
      carry_kept = 0;
      carry_rst = 0;
      bad = 0;
    }
    __syncthreads();
    constexpr int kPer = 16;
    for (int64_t base = 0; base < len; base += static_cast<int64_t>(blockDim.x) * kPer) {
      const int64_t p0 = base + static_cast<int64_t>(threadIdx.x) * kPer;
      uint32_t keep = 0, rst = 0;  // bit i: byte p0 + i kept / is the 2nd byte of an RST
      int n_keep = 0, n_rst = 0;
      bool my_bad = false;
      if (p0 < len) {
        int prev = p0 > 0 ? raw[p0 - 1] : 0;
        for (int i = 0; i < kPer && p0 + i < len; ++i) {
          const int cur = raw[p0 + i];
          const int nxt = p0 + i + 1 < len ? raw[p0 + i + 1] : -1;  // -1: end (EOI follows)
          bool kp = false;
          if (cur == 0xFF) {
            if (nxt == 0x00) kp = true;  // a data 0xFF (its stuffed 0x00 follows)
            else if (!(nxt == 0xFF || nxt == -1 || (nxt >= 0xD0 && nxt <= 0xD7))) my_bad = true;
          } else if (prev == 0xFF) {
            if (cur >= 0xD0 && cur <= 0xD7) {
              rst |= 1u << i;
              ++n_rst;
            } else if (cur != 0x00) {
              my_bad = true;  // a marker other than RST inside the scan
            }
          } else {
            kp = true;
          }
          if (kp) {
            keep |= 1u << i;
            ++n_keep;
          }
          prev = cur;
        }
      }
      if (my_bad) atomicOr(&bad, 1u);
      unsigned total;
      const unsigned before = block_excl_scan((static_cast<unsigned>(n_rst) << 16) | n_keep, sh, total);
      unsigned ck = carry_kept + (before & 0xFFFF);
      unsigned cr = carry_rst + (before >> 16);
      for (int i = 0; i < kPer; ++i) {
        if (keep >> i & 1) clean[ck++] = raw[p0 + i];
        if (rst >> i & 1) {
          ++cr;
          if (cr < static_cast<unsigned>(d.n_seg)) seg_start[cr] = static_cast<int32_t>(ck);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        carry_kept += total & 0xFFFF;
        carry_rst += total >> 16;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      seg_start[0] = 0;
      seg_start[d.n_seg] = static_cast<int32_t>(carry_kept);
      if (bad || carry_rst != static_cast<unsigned>(d.n_seg - 1)) atomicOr(status + k, TP_JPEG_CORRUPT);
    }
    for (int i = threadIdx.x; i < 64; i += blockDim.x) clean[carry_kept + i] = 0;  // peek slack
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// J2: Huffman decode

struct BitReader {
  const uint32_t* w;  // 4-byte aligned base
  uint32_t wi, hi, lo;
  __device__ void init(const uint8_t* clean) {
    w = reinterpret_cast<const uint32_t*>(clean);
    wi = 0xFFFFFFF0u;  // no word index: neither it nor its successor is ever requested
  }
  __device__ __forceinline__ uint32_t ld(uint32_t i) const { return __byte_perm(w[i], 0, 0x0123); }
  // the 32 bits starting at bit p (big-endian bit order)
  __device__ __forceinline__ uint32_t peek(uint32_t p) {
    const uint32_t i = p >> 5;
    if (i != wi) {
      if (i == wi + 1) {
        hi = lo;
        lo = ld(i + 1);
      } else {
        hi = ld(i);
        lo = ld(i + 1);
      }
      wi = i;
    }
    const uint32_t sh = p & 31;
    return sh ? (hi << sh) | (lo >> (32 - sh)) : hi;
  }
};

__device__ __forceinline__ int huff_decode(const JHuff* __restrict__ t, uint32_t v, int& sym) {
  const uint32_t e = t->fast[v >> (32 - jpeg::kFastBits)];
  if (e) {
    sym = e & 255;
    return static_cast<int>(e >> 8);
  }
  for (int l = jpeg::kFastBits + 1; l <= 16; ++l) {
    const int code = static_cast<int>(v >> (32 - l));
    if (code <= t->maxcode[l]) {
      sym = t->vals[(t->valoff[l] + code) & 255];
      return l;
    }
  }
  return 0;
}

__device__ __forceinline__ int extend(uint32_t bits, int s) {
  return bits < (1u << (s - 1)) ? static_cast<int>(bits) - (1 << s) + 1 : static_cast<int>(bits);
}

struct DecOut {
  uint32_t pos;
  int u, z, blocks, err;
};

// Decode from (pos, u, z) until the position reaches `stop` at a symbol boundary.
// MODE 0: speculative (entry guessed: an unclean symbol skips one bit and restarts the
// state); 1: true entry, counting; 2: true entry, writing coefficients from block
// `block` on, stopping at `block_limit`.  pos, stop and seg_bits are bits from the
// interval start; bit0 is the interval's first bit in the image's clean stream.
template <int MODE>
__device__ DecOut decode_run(const JDesc& d, BitReader& br, uint32_t bit0, uint32_t seg_bits,
                             uint32_t stop, uint32_t pos, int u, int z, int16_t* coef, int block,
                             int block_limit) {
  DecOut o;
  o.blocks = 0;
  o.err = kNoErr;
  int c = d.slot_comp[u];
  const JHuff* dct = &d.dc[d.comp_td[c]];
  const JHuff* act = &d.ac[d.comp_ta[c]];
  if (MODE == 2 && block >= block_limit) stop = pos;
  while (pos < stop) {
    const uint32_t v = br.peek(bit0 + pos);
    int sym;
    const int len = huff_decode(z == 0 ? dct : act, v, sym);
    int r = 0, s = sym;
    if (z != 0) {
      r = sym >> 4;
      s = sym & 15;
    }
    const uint32_t used = static_cast<uint32_t>(len + s);
    const bool ran_out = len != 0 && pos + used > seg_bits;
    if (len == 0 || ran_out || (z != 0 && s != 0 && z + r > 63)) {
      // An unclean symbol.  From a true entry it means a corrupt stream -- or the padding
      // after the interval's last block (harmless: phase 3 compares the block count at
      // the first unclean symbol with the interval's block total).  Either way the
      // decode resynchronises like a speculative one: an entry that is still wrong
      // (its predecessor not yet converged) must be able to fall into the true path.
      if (MODE != 0 && o.err == kNoErr) o.err = o.blocks;
      if (MODE == 2 || ran_out) {
        pos = seg_bits;
        break;
      }
      ++pos;
      u = 0;
      z = 0;
      c = d.slot_comp[0];
      dct = &d.dc[d.comp_td[c]];
      act = &d.ac[d.comp_ta[c]];
      continue;
    }
    if (z == 0) {
      if (MODE == 2) coef[static_cast<int64_t>(block) * 64] =
          static_cast<int16_t>(s ? extend((v << len) >> (32 - s), s) : 0);
      z = 1;
    } else if (s) {
      z += r;
      if (MODE == 2) coef[static_cast<int64_t>(block) * 64 + c_zig[z]] =
          static_cast<int16_t>(extend((v << len) >> (32 - s), s));
      ++z;
    } else if (r == 15) {
      z += 16;
    } else {
      z = 64;
    }
    pos += used;
    if (z >= 64) {
      z = 0;
      ++o.blocks;
      u = u + 1 == d.bmcu ? 0 : u + 1;
      c = d.slot_comp[u];
      dct = &d.dc[d.comp_td[c]];
      act = &d.ac[d.comp_ta[c]];
      if (MODE == 2 && ++block >= block_limit) break;
    }
  }
  o.pos = pos;
  o.u = u;
  o.z = z;
  return o;
}

__device__ __forceinline__ long long pack_state(uint32_t pos, int u, int z) {
  return (static_cast<long long>(pos) << 16) | (u << 8) | z;
}

struct SlotRef {
  int k, s, j;      // image, interval, subsequence within the interval
  uint32_t bit0;    // interval's first bit in the clean stream
  uint32_t seg_bits;
};

__device__ inline bool slot_ref(const JDesc* descs, int n, uint8_t* work, const int32_t* status,
                                int64_t g, SlotRef& r) {
  r.k = find_image(descs, n, g, 0);
  const JDesc& d = descs[r.k];
  const int64_t t = g - d.slot_base;
  if (t < 0 || t >= d.n_slots || status[r.k]) return false;
  const int32_t* seg_start = reinterpret_cast<const int32_t*>(work + d.seg_off);
  const int32_t* sub_prefix = seg_start + d.n_seg + 1;
  if (t >= sub_prefix[d.n_seg]) return false;
  int lo = 0, hi = d.n_seg;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sub_prefix[mid] <= t) lo = mid; else hi = mid;
  }
  r.s = lo;
  r.j = static_cast<int>(t - sub_prefix[lo]);
  r.bit0 = 8u * static_cast<uint32_t>(seg_start[lo]);
  r.seg_bits = 8u * static_cast<uint32_t>(seg_start[lo + 1] - seg_start[lo]);
  return true;
}

__device__ inline int seg_blocks(const JDesc& d, int s) {
  const int n_mcu = d.mcux * d.mcuy;
  const int m = n_mcu - s * d.ri < d.ri ? n_mcu - s * d.ri : d.ri;
  return m * d.bmcu;
}

__global__ void __launch_bounds__(256) k_jpeg_huff(const JDesc* __restrict__ descs, int n,
                                                   int64_t total_slots, int sub_bits,
                                                   uint8_t* __restrict__ work,
                                                   int32_t* __restrict__ status) {
  cg::grid_group grid = cg::this_grid();
  const Work W = work_view(work, total_slots);
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;

  // (0) subsequences per interval (sub_prefix after seg_start)
  for (int64_t k = tid; k < n; k += nthreads) {
    const JDesc& d = descs[k];
    if (d.n_slots == 0 || status[k]) continue;
    const int32_t* seg_start = reinterpret_cast<const int32_t*>(work + d.seg_off);
    int32_t* sub_prefix = const_cast<int32_t*>(seg_start) + d.n_seg + 1;
    int acc = 0;
    for (int s = 0; s < d.n_seg; ++s) {
      sub_prefix[s] = acc;
      const int64_t bits = 8LL * (seg_start[s + 1] - seg_start[s]);
      acc += static_cast<int>(bits > 0 ? (bits + sub_bits - 1) / sub_bits : 1);
    }
    sub_prefix[d.n_seg] = acc;
    if (acc > d.n_slots) atomicOr(status + k, TP_JPEG_CORRUPT);  // cannot happen: clean <= raw
  }
  grid.sync();

  // (1) speculative decode of every subsequence
  for (int64_t g = tid; g < total_slots; g += nthreads) {
    SlotRef r;
    if (!slot_ref(descs, n, work, status, g, r)) continue;
    const JDesc& d = descs[r.k];
    BitReader br;
    br.init(work + d.clean_off);
    const uint32_t start = static_cast<uint32_t>(r.j) * sub_bits;
    const uint32_t stop = min(start + static_cast<uint32_t>(sub_bits), r.seg_bits);
    const DecOut o = r.j == 0 ? decode_run<1>(d, br, r.bit0, r.seg_bits, stop, 0, 0, 0, nullptr, 0, 0)
                              : decode_run<0>(d, br, r.bit0, r.seg_bits, stop, start, 0, 0, nullptr, 0, 0);
    W.exitp[g] = pack_state(o.pos, o.u, o.z);
    W.blocks[g] = o.blocks;
    W.err[g] = o.err;
    W.lastproc[g] = 0;
    W.changed[g] = 1;
  }

  // (2) half-rounds: subsequences of one parity re-decode from their predecessor's exit
  int h = 2;
  for (; h < kMaxSteps; ++h) {
    grid.sync();
    for (int64_t g = tid; g < total_slots; g += nthreads) {
      SlotRef r;
      if (!slot_ref(descs, n, work, status, g, r) || r.j == 0 || (r.j & 1) != (h & 1)) continue;
      if (W.changed[g - 1] < W.lastproc[g]) continue;
      const JDesc& d = descs[r.k];
      BitReader br;
      br.init(work + d.clean_off);
      const long long e = W.exitp[g - 1];
      const uint32_t stop = min(static_cast<uint32_t>(r.j + 1) * sub_bits, r.seg_bits);
      const DecOut o = decode_run<1>(d, br, r.bit0, r.seg_bits, stop, static_cast<uint32_t>(e >> 16),
                                     static_cast<int>((e >> 8) & 255), static_cast<int>(e & 255),
                                     nullptr, 0, 0);
      const long long x = pack_state(o.pos, o.u, o.z);
      W.blocks[g] = o.blocks;
      W.err[g] = o.err;
      W.lastproc[g] = h;
      if (x != W.exitp[g]) {
        W.exitp[g] = x;
        W.changed[g] = h;
        atomicAdd(W.counters + h, 1u);
      }
    }
    grid.sync();
    if (h >= 3 && W.counters[h] == 0 && W.counters[h - 1] == 0) break;
  }
  const bool converged = h < kMaxSteps;
  if (tid == 0) W.counters[1023] = h;  // diagnostics: half-rounds used

  // (3) per interval: first block of every subsequence; unclean streams go to the host
  const int lane = threadIdx.x & 31;
  const int64_t warp = tid >> 5, nwarps = nthreads >> 5;
  for (int64_t k = warp; k < n; k += nwarps) {
    const JDesc& d = descs[k];
    if (d.n_slots == 0 || status[k]) continue;
    const int32_t* seg_start = reinterpret_cast<const int32_t*>(work + d.seg_off);
    const int32_t* sub_prefix = seg_start + d.n_seg + 1;
    bool bad = false;
    for (int s = 0; s < d.n_seg; ++s) {
      const int T = seg_blocks(d, s);
      const int first = s * d.ri * d.bmcu;
      int carry = 0;
      for (int t0 = sub_prefix[s]; t0 < sub_prefix[s + 1]; t0 += 32) {
        const int t = t0 + lane;
        const int64_t g = d.slot_base + t;
        const bool on = t < sub_prefix[s + 1];
        const int b = on ? W.blocks[g] : 0;
        int x = b;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, dd);
          if (lane >= dd) x += y;
        }
        const int before = carry + x - b;
        if (on) {
          W.bstart[g] = first + before;
          const int e = W.err[g];
          if (e != kNoErr && before + e < T) bad = true;
          if (!converged && W.changed[g] >= h - 1) bad = true;
        }
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (carry < T) bad = true;  // the data ends before the interval's last block
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status + k, TP_JPEG_CORRUPT);
  }
  grid.sync();

  // (4) write pass
  for (int64_t g = tid; g < total_slots; g += nthreads) {
    SlotRef r;
    if (!slot_ref(descs, n, work, status, g, r)) continue;
    const JDesc& d = descs[r.k];
    BitReader br;
    br.init(work + d.clean_off);
    uint32_t pos = 0;
    int u = 0, z = 0;
    if (r.j > 0) {
      const long long e = W.exitp[g - 1];
      pos = static_cast<uint32_t>(e >> 16);
      u = static_cast<int>((e >> 8) & 255);
      z = static_cast<int>(e & 255);
    }
    const uint32_t stop = min(static_cast<uint32_t>(r.j + 1) * sub_bits, r.seg_bits);
    const int limit = r.s * d.ri * d.bmcu + seg_blocks(d, r.s);
    decode_run<2>(d, br, r.bit0, r.seg_bits, stop, pos, u, z,
                  reinterpret_cast<int16_t*>(work + d.coef_off), W.bstart[g], limit);
  }
  grid.sync();

  // (5) DC prediction per interval and component (diffs -> values, int16 stores)
  for (int64_t k = warp; k < n; k += nwarps) {
    const JDesc& d = descs[k];
    if (d.n_slots == 0 || status[k]) continue;
    int16_t* coef = reinterpret_cast<int16_t*>(work + d.coef_off);
    const int n_mcu = d.mcux * d.mcuy;
    for (int c = 0; c < d.ncomp; ++c) {
      int u0 = 0;
      while (d.slot_comp[u0] != c) ++u0;
      int nb = 0;
      while (u0 + nb < d.bmcu && d.slot_comp[u0 + nb] == c) ++nb;
      for (int s = 0; s < d.n_seg; ++s) {
        const int m0 = s * d.ri, m1 = min(n_mcu, m0 + d.ri);
        int carry = 0;  // libjpeg's last_dc_val (int), reset at each restart
        for (int mb = m0; mb < m1; mb += 32) {
          const int m = mb + lane;
          int sum = 0;
          if (m < m1)
            for (int b = 0; b < nb; ++b) sum += coef[(static_cast<int64_t>(m) * d.bmcu + u0 + b) * 64];
          int x = sum;
#pragma unroll
          for (int dd = 1; dd < 32; dd <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, dd);
            if (lane >= dd) x += y;
          }
          int run = carry + x - sum;
          if (m < m1)
            for (int b = 0; b < nb; ++b) {
              int16_t* p = coef + (static_cast<int64_t>(m) * d.bmcu + u0 + b) * 64;
              run += *p;
              *p = static_cast<int16_t>(run);
            }
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// J3: ISLOW IDCT (jidctint.c), 8 threads per block

constexpr long long F0298 = 2446, F0390 = 3196, F0541 = 4433, F0765 = 6270, F0899 = 7373,
                    F1175 = 9633, F1501 = 12299, F1847 = 15137, F1961 = 16069, F2053 = 16819,
                    F2562 = 20995, F3072 = 25172;

__device__ __forceinline__ void idct_1d(const long long (&in)[8], long long (&out)[8]) {
  long long z2 = in[2], z3 = in[6];
  long long z1 = (z2 + z3) * F0541;
  const long long tmp2 = z1 + z3 * -F1847;
  const long long tmp3 = z1 + z2 * F0765;
  const long long tmp0 = (in[0] + in[4]) * 8192;  // << CONST_BITS
  const long long tmp1 = (in[0] - in[4]) * 8192;
  const long long tmp10 = tmp0 + tmp3, tmp13 = tmp0 - tmp3, tmp11 = tmp1 + tmp2, tmp12 = tmp1 - tmp2;
  long long t0 = in[7], t1 = in[5], t2 = in[3], t3 = in[1];
  z1 = t0 + t3;
  z2 = t1 + t2;
  z3 = t0 + t2;
  long long z4 = t1 + t3;
  const long long z5 = (z3 + z4) * F1175;
  t0 *= F0298;
  t1 *= F2053;
  t2 *= F3072;
  t3 *= F1501;
  z1 *= -F0899;
  z2 *= -F2562;
  z3 = z3 * -F1961 + z5;
  z4 = z4 * -F0390 + z5;
  t0 += z1 + z3;
  t1 += z2 + z4;
  t2 += z2 + z3;
  t3 += z1 + z4;
  out[0] = tmp10 + t3;
  out[7] = tmp10 - t3;
  out[1] = tmp11 + t2;
  out[6] = tmp11 - t2;
  out[2] = tmp12 + t1;
  out[5] = tmp12 - t1;
  out[3] = tmp13 + t0;
  out[4] = tmp13 - t0;
}

__device__ __forceinline__ uint32_t range_limit(long long x) {
  const uint32_t v = static_cast<uint32_t>(x) & 1023u;  // RANGE_MASK
  return v < 128 ? v + 128 : v < 512 ? 255u : v < 896 ? 0u : v - 896;
}

__global__ void __launch_bounds__(256) k_jpeg_idct(const JDesc* __restrict__ descs, int n,
                                                   int64_t total_blocks, uint8_t* __restrict__ work,
                                                   const int32_t* __restrict__ status) {
  __shared__ int ws[32][64];
  const int sub = threadIdx.x & 7, lb = threadIdx.x >> 3;
  for (int64_t gb0 = static_cast<int64_t>(blockIdx.x) * 32; gb0 < total_blocks;
       gb0 += static_cast<int64_t>(gridDim.x) * 32) {
    const int64_t gb = gb0 + lb;
    const bool on = gb < total_blocks;
    int k = 0;
    const JDesc* d = nullptr;
    bool live = false;
    if (on) {
      k = find_image(descs, n, gb, 1);
      d = descs + k;
      live = d->n_slots > 0 && status[k] == 0;
    }
    const int b = on ? static_cast<int>(gb - d->block_base) : 0;
    int c = 0;
    const int16_t* blk = nullptr;
    if (live) {
      c = d->slot_comp[b % d->bmcu];
      blk = reinterpret_cast<const int16_t*>(work + d->coef_off) + static_cast<int64_t>(b) * 64;
      // pass 1: column `sub` (DEQUANTIZE: short coef x short quant, as ISLOW_MULT_TYPE)
      long long in[8], out[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        in[r] = static_cast<long long>(blk[8 * r + sub]) *
                static_cast<long long>(static_cast<int16_t>(d->quant[c][8 * r + sub]));
      idct_1d(in, out);
#pragma unroll
      for (int r = 0; r < 8; ++r)  // DESCALE(x, CONST_BITS - PASS1_BITS), stored as int
        ws[lb][8 * r + sub] = static_cast<int>((out[r] + (1LL << 10)) >> 11);
    }
    __syncthreads();
    if (live) {
      long long in[8], out[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) in[i] = ws[lb][8 * sub + i];
      idct_1d(in, out);
      const int mcu = b / d->bmcu, u = b % d->bmcu;
      const int my = mcu / d->mcux, mx = mcu % d->mcux;
      const int by = d->ncomp == 1 ? my : my * d->comp_v[c] + d->slot_bv[u];
      const int bx = d->ncomp == 1 ? mx : mx * d->comp_h[c] + d->slot_bh[u];
      uint8_t* dst = work + d->plane_off[c] + static_cast<int64_t>(by * 8 + sub) * d->plane_w[c] + bx * 8;
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // DESCALE(x, CONST_BITS + PASS1_BITS + 3), range limit
        lo |= range_limit((out[i] + (1LL << 17)) >> 18) << (8 * i);
        hi |= range_limit((out[i + 4] + (1LL << 17)) >> 18) << (8 * i);
      }
      *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// J4: upsampling + colour conversion -> RGB HWC

__device__ __forceinline__ int chroma(const uint8_t* __restrict__ p, int pw, int dsw, int dsh, int hx,
                                      int vx, int x, int y) {
  if (hx == 1 && vx == 1) return p[static_cast<int64_t>(y) * pw + x];
  if (dsw <= 2) return p[static_cast<int64_t>(y / vx) * pw + (x >> 1)];  // plain replication
  const int i = x >> 1;
  if (vx == 1) {  // h2v1 fancy
    const uint8_t* row = p + static_cast<int64_t>(y) * pw;
    if (x & 1) return i == dsw - 1 ? row[i] : (row[i] * 3 + row[i + 1] + 2) >> 2;
    return i == 0 ? row[0] : (row[i] * 3 + row[i - 1] + 1) >> 2;
  }
  // h2v2 fancy: nearer row inrow, further row above (even y) / below (odd y), replicated
  const int inrow = y >> 1;
  const int other = (y & 1) ? min(inrow + 1, dsh - 1) : max(inrow - 1, 0);
  const uint8_t* r0 = p + static_cast<int64_t>(inrow) * pw;
  const uint8_t* r1 = p + static_cast<int64_t>(other) * pw;
  const int cs = r0[i] * 3 + r1[i];
  if (x & 1) {
    if (i == dsw - 1) return (cs * 4 + 7) >> 4;
    return (cs * 3 + r0[i + 1] * 3 + r1[i + 1] + 7) >> 4;
  }
  if (i == 0) return (cs * 4 + 8) >> 4;
  return (cs * 3 + r0[i - 1] * 3 + r1[i - 1] + 8) >> 4;
}

__device__ __forceinline__ uint32_t clamp255(int v) { return static_cast<uint32_t>(min(max(v, 0), 255)); }

__global__ void __launch_bounds__(256) k_jpeg_color(const JDesc* __restrict__ descs, int n,
                                                    int64_t total_rows, const uint8_t* __restrict__ work,
                                                    uint8_t* __restrict__ out,
                                                    const int32_t* __restrict__ status) {
  for (int64_t gr = blockIdx.x; gr < total_rows; gr += gridDim.x) {
    const int k = find_image(descs, n, gr, 2);
    const JDesc& d = descs[k];
    if (d.n_slots == 0 || status[k]) continue;
    const int y = static_cast<int>(gr - d.row_base);
    uint8_t* o = out + d.out_off + static_cast<int64_t>(y) * d.width * 3;
    const uint8_t* py = work + d.plane_off[0];
    if (d.ncomp == 1) {
      for (int x = threadIdx.x; x < d.width; x += blockDim.x) {
        const uint8_t g = py[static_cast<int64_t>(y) * d.plane_w[0] + x];
        o[3 * x] = g;
        o[3 * x + 1] = g;
        o[3 * x + 2] = g;
      }
      continue;
    }
    const uint8_t* pcb = work + d.plane_off[1];
    const uint8_t* pcr = work + d.plane_off[2];
    const int hx = d.hmax / d.comp_h[1], vx = d.vmax / d.comp_v[1];
    for (int x = threadIdx.x; x < d.width; x += blockDim.x) {
      const int Y = py[static_cast<int64_t>(y) * d.plane_w[0] + x];
      const int cb = chroma(pcb, d.plane_w[1], d.ds_w[1], d.ds_h[1], hx, vx, x, y) - 128;
      const int cr = chroma(pcr, d.plane_w[2], d.ds_w[2], d.ds_h[2], hx, vx, x, y) - 128;
      // jdcolor.c build_ycc_rgb_table: FIX(x) = x * 65536 + 0.5, ONE_HALF = 32768
      const int r = Y + ((91881 * cr + 32768) >> 16);
      const int g = Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16);
      const int b = Y + ((116130 * cb + 32768) >> 16);
      o[3 * x] = static_cast<uint8_t>(clamp255(r));
      o[3 * x + 1] = static_cast<uint8_t>(clamp255(g));
      o[3 * x + 2] = static_cast<uint8_t>(clamp255(b));
    }
  }
}

__global__ void k_jpeg_status_init(const JDesc* __restrict__ descs, int n, int32_t* status) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    status[k] = descs[k].n_slots > 0 ? TP_JPEG_OK : TP_JPEG_UNSUPPORTED;
}

}  // namespace
}  // namespace tp

extern "C" {

TP_API int tp_jpeg_decode(const uint8_t* d_payload, const void* d_desc, int32_t n,
                          const int64_t* totals, int32_t sub_bits, void* d_work,
                          int64_t work_bytes, uint8_t* d_out, int32_t* d_status, void* stream) {
  using namespace tp;
  if (n < 0 || !totals || (n > 0 && (!d_payload || !d_desc || !d_work || !d_out || !d_status)) ||
      sub_bits < 64 || (sub_bits & 31))
    return set_error(TP_ERR_INVALID_ARGUMENT, "tp_jpeg_decode: bad arguments");
  if (n == 0) return TP_OK;
  cudaStream_t s = as_stream(stream);
  const JDesc* descs = static_cast<const JDesc*>(d_desc);
  uint8_t* work = static_cast<uint8_t*>(d_work);
  const int64_t slots = totals[0], blocks = totals[1], rows = totals[2];
  const int64_t coef_begin = totals[3], coef_end = totals[4];
  if (coef_end > work_bytes || coef_begin < 4096) return set_error(TP_ERR_INVALID_ARGUMENT, "tp_jpeg_decode: workspace too small");
  k_jpeg_status_init<<<(n + 255) / 256, 256, 0, s>>>(descs, n, d_status);
  if (cudaMemsetAsync(work, 0, 4096, s) != cudaSuccess ||
      cudaMemsetAsync(work + coef_begin, 0, coef_end - coef_begin, s) != cudaSuccess)
    return set_error(TP_ERR_CUDA, "tp_jpeg_decode: memset failed");
  const int sms = device_sm_count();
  k_jpeg_unstuff<<<min(n, 4 * sms), 512, 0, s>>>(d_payload, descs, n, work, d_status);
  if (slots > 0) {
    static int per_sm_of[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
      return set_error(TP_ERR_CUDA, "tp_jpeg_decode: no usable device");
    int& per_sm = per_sm_of[dev];
    if (per_sm == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jpeg_huff, 256, 0);
      if (per_sm <= 0) return set_error(TP_ERR_CUDA, "tp_jpeg_decode: decode kernel does not fit");
    }
    int grid = per_sm * sms;
    const int64_t need = (slots + 255) / 256;
    if (need < grid) grid = static_cast<int>(need > 0 ? need : 1);
    int nn = n;
    int64_t ts = slots;
    int sb = sub_bits;
    int32_t* st = d_status;
    void* args[] = {&descs, &nn, &ts, &sb, &work, &st};
    cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_jpeg_huff), grid, 256,
                                                args, 0, s);
    if (e != cudaSuccess) return set_error(TP_ERR_CUDA, "tp_jpeg_decode: %s", cudaGetErrorString(e));
  }
  if (blocks > 0) {
    const int64_t g = (blocks + 31) / 32;
    k_jpeg_idct<<<static_cast<unsigned>(g < 32 * sms ? g : 32 * sms), 256, 0, s>>>(descs, n, blocks, work, d_status);
  }
  if (rows > 0) {
    k_jpeg_color<<<static_cast<unsigned>(rows < 64 * sms ? rows : 64 * sms), 256, 0, s>>>(descs, n, rows, work, d_out, d_status);
  }
  return check_launch("tp_jpeg_decode");
}

}  // extern "C"
