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
//                      (3) per interval, scans of the blocks and of the per-component DC
//                          difference sums each subsequence decodes give its first block
//                          index and its entry DC predictors;
//                      (4) every subsequence decodes once more, writing its coefficients
//                          with DC values predicted in place (int16, libjpeg's JCOEF)
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
constexpr int kMaxHops = 1;  // subsequences one thread re-decodes per half-round (longer
                              // chains measured slower: one thread's serial decodes)
constexpr int kCkpts = 7;  // checkpoints per subsequence (every sub_bits / 8 bits)

struct Work {
  unsigned* counters;  // [h]: exits changed in half-round h; [512 + h]: decodes in it;
                       // [1023]: half-rounds used
  unsigned long long* stamps;  // [8] phase timestamps (globaltimer), diagnostics
  long long* exitp;    // per slot: (bit << 16) | (u << 8) | z, bit relative to the interval
  long long* entry;    // per slot: the entry state its counts below were decoded from
  int4* dcs;           // per slot: DC difference sums per component (.y .z .w), then
                       // (phase 3) the interval's running DC of each component at the entry
  int* blocks;         // blocks completed from the entry to the exit
  int* err;            // block count at the first unclean symbol, kNoErr if none
  int* errpos;         // its bit position
  int* bstart;         // block index (in the image) at the entry
  int* claim;          // half-round in which a thread last took this slot (one decode each)
  long long* ck_state; // [slot][kCkpts] checkpoint states
  int4* ck_acc;        // [slot][kCkpts] checkpoint accumulators
};

__host__ __device__ inline int64_t al256(int64_t v) { return (v + 255) & ~int64_t(255); }

__device__ inline Work work_view(uint8_t* w, int64_t slots) {
  Work v;
  v.counters = reinterpret_cast<unsigned*>(w);
  v.stamps = reinterpret_cast<unsigned long long*>(w + 3968);
  int64_t o = 4096;
  v.exitp = reinterpret_cast<long long*>(w + o);
  o += al256(8 * slots);
  v.entry = reinterpret_cast<long long*>(w + o);
  o += al256(8 * slots);
  v.dcs = reinterpret_cast<int4*>(w + o);
  o += al256(16 * slots);
  int* arrs[5];
  for (int i = 0; i < 5; ++i) {
    arrs[i] = reinterpret_cast<int*>(w + o);
    o += al256(4 * slots);
  }
  v.blocks = arrs[0];
  v.err = arrs[1];
  v.errpos = arrs[2];
  v.bstart = arrs[3];
  v.claim = arrs[4];
  v.ck_state = reinterpret_cast<long long*>(w + o);
  o += al256(8 * kCkpts * slots);
  v.ck_acc = reinterpret_cast<int4*>(w + o);
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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

// The scan is cut into chunks of kChunk raw bytes (one CTA each, many per image): a
// counting pass, then a writing pass that places each chunk's kept bytes after the kept
// bytes of the image's earlier chunks.  A thread owns 16 raw bytes per step (one 16-byte
// load; a step without a 0xFF byte keeps all 16), the CTA compacts them in shared memory
// and stores the step's output with consecutive threads writing consecutive bytes.
constexpr int kUnstuffThreads = 512;
constexpr int kChunk = 32768;  // raw bytes per CTA (4 steps of 512 x 16)

struct ByteFlags {
  uint32_t keep, rst;  // bit i: byte i kept / byte i is the second byte of an RST marker
  bool bad;            // a marker other than RST inside the scan
};

__device__ __forceinline__ ByteFlags flag_bytes(const uint8_t* raw, int64_t p0, int64_t len) {
  ByteFlags f{0u, 0u, false};
  if (p0 >= len) return f;
  const int nb = len - p0 < 16 ? static_cast<int>(len - p0) : 16;
  uint32_t w[4] = {0, 0, 0, 0};
  if (nb == 16) {
    const uint4 q = *reinterpret_cast<const uint4*>(raw + p0);
    w[0] = q.x;
    w[1] = q.y;
    w[2] = q.z;
    w[3] = q.w;
  } else {
    for (int i = 0; i < nb; ++i) w[i >> 2] |= static_cast<uint32_t>(raw[p0 + i]) << (8 * (i & 3));
  }
  const int prev0 = p0 > 0 ? raw[p0 - 1] : 0;
  bool any_ff = prev0 == 0xFF;
#pragma unroll
  for (int i = 0; i < 4; ++i) any_ff |= __vcmpeq4(w[i], 0xFFFFFFFFu) != 0;
  if (!any_ff) {  // the common case: no 0xFF anywhere near
    f.keep = nb == 16 ? 0xFFFFu : (1u << nb) - 1u;
    return f;
  }
  int prev = prev0;
  for (int i = 0; i < nb; ++i) {
    const int cur = (w[i >> 2] >> (8 * (i & 3))) & 255;
    int nxt;
    if (i + 1 < nb) nxt = (w[(i + 1) >> 2] >> (8 * ((i + 1) & 3))) & 255;
    else nxt = p0 + i + 1 < len ? raw[p0 + i + 1] : -1;  // -1: end (EOI follows)
    if (cur == 0xFF) {
      if (nxt == 0x00) f.keep |= 1u << i;  // a data 0xFF (its stuffed 0x00 follows)
      else if (!(nxt == 0xFF || nxt == -1 || (nxt >= 0xD0 && nxt <= 0xD7))) f.bad = true;
    } else if (prev == 0xFF) {
      if (cur >= 0xD0 && cur <= 0xD7) f.rst |= 1u << i;
      else if (cur != 0x00) f.bad = true;
    } else {
      f.keep |= 1u << i;
    }
    prev = cur;
  }
  return f;
}

__device__ inline int find_chunk_image(const JDesc* d, int n, int64_t c) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (d[mid].chunk_base <= c) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kUnstuffThreads) k_jpeg_unstuff_count(
    const uint8_t* __restrict__ payload, const JDesc* __restrict__ descs, int n,
    int2* __restrict__ chunk_counts, int32_t* __restrict__ status) {
  __shared__ int sk[kUnstuffThreads / 32], sr[kUnstuffThreads / 32];
  __shared__ int sbad;
  const int64_t c = blockIdx.x;
  const int k = find_chunk_image(descs, n, c);
  const JDesc& d = descs[k];
  const int64_t c0 = (c - d.chunk_base) * kChunk;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  int kept = 0, rst = 0;
  bool bad = false;
  for (int step = 0; step < kChunk / (16 * kUnstuffThreads); ++step) {
    const int64_t p0 = c0 + (static_cast<int64_t>(step) * kUnstuffThreads + threadIdx.x) * 16;
    const ByteFlags f = flag_bytes(payload + d.raw_off, p0, d.raw_len);
    kept += __popc(f.keep);
    rst += __popc(f.rst);
    bad |= f.bad;
  }
  kept = __reduce_add_sync(0xffffffffu, kept);
  rst = __reduce_add_sync(0xffffffffu, rst);
  if (bad) sbad = 1;
  if ((threadIdx.x & 31) == 0) {
    sk[threadIdx.x >> 5] = kept;
    sr[threadIdx.x >> 5] = rst;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tk = 0, tr = 0;
    for (int w = 0; w < kUnstuffThreads / 32; ++w) {
      tk += sk[w];
      tr += sr[w];
    }
    chunk_counts[c] = make_int2(tk, tr);
    if (sbad) atomicOr(status + k, TP_JPEG_CORRUPT);
  }
}

__global__ void __launch_bounds__(kUnstuffThreads) k_jpeg_unstuff_write(
    const uint8_t* __restrict__ payload, const JDesc* __restrict__ descs, int n,
    const int2* __restrict__ chunk_counts, uint8_t* __restrict__ work,
    int32_t* __restrict__ status) {
  __shared__ unsigned sh[32];
  __shared__ uint8_t sout[16 * kUnstuffThreads];
  __shared__ int carry_k, carry_r;
  const int64_t c = blockIdx.x;
  const int k = find_chunk_image(descs, n, c);
  const JDesc& d = descs[k];
  const int64_t ci = c - d.chunk_base;
  const int64_t c0 = ci * kChunk;
  uint8_t* clean = work + d.clean_off;
  int32_t* seg_start = reinterpret_cast<int32_t*>(work + d.seg_off);
  if (threadIdx.x == 0) {
    int tk = 0, tr = 0;
    for (int64_t j = d.chunk_base; j < c; ++j) {
      const int2 v = chunk_counts[j];
      tk += v.x;
      tr += v.y;
    }
    carry_k = tk;
    carry_r = tr;
  }
  __syncthreads();
  const uint8_t* raw = payload + d.raw_off;
  for (int step = 0; step < kChunk / (16 * kUnstuffThreads); ++step) {
    const int64_t sbase = c0 + static_cast<int64_t>(step) * kUnstuffThreads * 16;
    if (sbase >= d.raw_len) break;  // uniform across the CTA
    const int64_t p0 = sbase + static_cast<int64_t>(threadIdx.x) * 16;
    const ByteFlags f = flag_bytes(raw, p0, d.raw_len);
    unsigned total;
    const unsigned before = block_excl_scan((static_cast<unsigned>(__popc(f.rst)) << 16) |
                                                static_cast<unsigned>(__popc(f.keep)), sh, total);
    unsigned o = before & 0xFFFF;
    unsigned r = carry_r + (before >> 16);
    for (int i = 0; i < 16; ++i) {
      if (f.keep >> i & 1) sout[o++] = raw[p0 + i];
      if (f.rst >> i & 1) {
        ++r;
        if (r < static_cast<unsigned>(d.n_seg)) seg_start[r] = static_cast<int32_t>(carry_k + o);
      }
    }
    __syncthreads();
    const int nk = static_cast<int>(total & 0xFFFF);
    for (int i = threadIdx.x; i < nk; i += kUnstuffThreads) clean[carry_k + i] = sout[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_k += nk;
      carry_r += static_cast<int>(total >> 16);
    }
    __syncthreads();
  }
  if (ci == d.n_chunks - 1) {  // the image's last chunk closes the interval table
    if (threadIdx.x == 0) {
      seg_start[0] = 0;
      seg_start[d.n_seg] = carry_k;
      if (carry_r != d.n_seg - 1) atomicOr(status + k, TP_JPEG_CORRUPT);
    }
    for (int i = threadIdx.x; i < 64; i += kUnstuffThreads) clean[carry_k + i] = 0;  // peek slack
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
  // pull the bits [b0, b1) into L1 ahead of the serial decode: its loads then hit L1
  // instead of paying the L2 latency every 32 bits
  __device__ __forceinline__ void prefetch(uint32_t b0, uint32_t b1) const {
    const char* p = reinterpret_cast<const char*>(w);
    for (uint32_t byte = (b0 >> 3) & ~127u; byte < ((b1 + 7) >> 3) + 8; byte += 128)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p + byte));
  }
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

__device__ __forceinline__ int extend(uint32_t bits, int s) {  // T.81 F.12 EXTEND, s >= 1
  return bits < (1u << ((s - 1) & 31)) ? static_cast<int>(bits) - (1 << s) + 1 : static_cast<int>(bits);
}

struct DecOut {
  uint32_t pos;
  int u, z, blocks, err;
  int symbols;  // decoded in this call (diagnostics)
  int dc[jpeg::kMaxComps];  // sum of the DC differences decoded, per component
};

// The per-image fields the symbol loop needs, in registers: per block slot of the MCU its
// component, and per component its DC / AC tables.
struct Tabs {
  const JHuff* base;   // [4]: dc0 dc1 ac0 ac1 (a shared-memory copy or the descriptor's own)
  uint32_t slot_comp;  // 2 bits per block slot of the MCU: its component
  uint32_t dcid, acid; // bit c: table id of component c
  int bmcu;
  __device__ void load(const JDesc& d, const JHuff* tables) {
    base = tables;
    bmcu = d.bmcu;
    slot_comp = 0;
    for (int u = 0; u < d.bmcu; ++u) slot_comp |= static_cast<uint32_t>(d.slot_comp[u]) << (2 * u);
    dcid = acid = 0;
    for (int c = 0; c < d.ncomp; ++c) {
      dcid |= static_cast<uint32_t>(d.comp_td[c] & 1) << c;
      acid |= static_cast<uint32_t>(d.comp_ta[c] & 1) << c;
    }
  }
  __device__ __forceinline__ int comp(int u) const { return (slot_comp >> (2 * u)) & 3; }
  __device__ __forceinline__ const JHuff* dct(int c) const { return base + ((dcid >> c) & 1); }
  __device__ __forceinline__ const JHuff* act(int c) const { return base + 2 + ((acid >> c) & 1); }
};

// Checkpoints of one subsequence: the decoder's state at the first symbol boundary at or
// after each checkpoint position, with the blocks and DC sums accumulated from the entry
// to there.  A later decode of the same subsequence from another entry that reaches a
// checkpoint in the recorded state has rejoined the recorded path: everything after it is
// known, so the decode stops there (a re-decode usually costs a few hundred bits, not
// sub_bits).
struct Ckpt {
  long long* state;  // [kCkpts], -1 = not recorded
  int4* acc;         // [kCkpts] (blocks, dc0, dc1, dc2) from the entry
  uint32_t first, step;
  bool compare;      // a previous decode of this subsequence exists (its totals below)
  long long prev_exit;
  int prev_blocks, prev_err;
  uint32_t prev_errpos;
  int4 prev_dc;
};

__device__ __forceinline__ long long pack_state(uint32_t pos, int u, int z) {
  return (static_cast<long long>(pos) << 16) | (u << 8) | z;
}

// Decode from (pos, u, z) until the position reaches `stop` at a symbol boundary.
// MODE 0: speculative (entry guessed); 1: true entry, counting; 2: true entry, writing
// coefficients from block `block` on (stopping at `block_limit`), DC values predicted
// from `pred` (the interval's running DC of each component at this entry).  pos, stop
// and seg_bits are bits from the interval start; bit0 is the interval's first bit in
// the image's clean stream.  CK: record / compare checkpoints (MODE 0 and 1).
template <int MODE, bool CK>
__device__ DecOut decode_run(const Tabs& T, BitReader& br, uint32_t bit0, uint32_t seg_bits,
                             uint32_t stop, uint32_t pos, int u, int z, int16_t* coef, int block,
                             int block_limit, const int* pred_in, const Ckpt* ck = nullptr,
                             uint32_t* errpos = nullptr) {
  DecOut o;
  o.blocks = 0;
  o.err = kNoErr;
  o.symbols = 0;
  uint32_t epos = 0xFFFFFFFFu;
  // running DC per component: the predictors (MODE 2) or the sums of differences
  int p0 = MODE == 2 ? pred_in[0] : 0, p1 = MODE == 2 ? pred_in[1] : 0,
      p2 = MODE == 2 ? pred_in[2] : 0;
  int c = T.comp(u);
  const JHuff* dct = T.dct(c);
  const JHuff* act = T.act(c);
  int ci = 0;
  uint32_t next_cp = CK ? ck->first : 0xFFFFFFFFu;
  if (MODE == 2 && block >= block_limit) stop = pos;
  if (pos < stop) br.prefetch(bit0 + pos, bit0 + stop);
  while (pos < stop) {
    if (CK && pos >= next_cp) {
      const long long st = pack_state(pos, u, z);
      if (ck->compare && ck->state[ci] == st) {  // rejoined the recorded path
        const int4 a = ck->acc[ci];
        const int4 now = make_int4(o.blocks, p0, p1, p2);
        if (o.err == kNoErr && ck->prev_err != kNoErr && ck->prev_errpos >= pos) {
          o.err = ck->prev_err - a.x + o.blocks;
          epos = ck->prev_errpos;
        }
        o.blocks += ck->prev_blocks - a.x;
        p0 += ck->prev_dc.y - a.y;
        p1 += ck->prev_dc.z - a.z;
        p2 += ck->prev_dc.w - a.w;
        // later checkpoints hold accumulators of the recorded decode: rebase them
        for (int i = ci; i < kCkpts; ++i) {
          if (ck->state[i] < 0) break;
          const int4 b = ck->acc[i];
          ck->acc[i] = make_int4(b.x - a.x + now.x, b.y - a.y + now.y, b.z - a.z + now.z,
                                 b.w - a.w + now.w);
        }
        o.pos = static_cast<uint32_t>(ck->prev_exit >> 16);
        o.u = static_cast<int>((ck->prev_exit >> 8) & 255);
        o.z = static_cast<int>(ck->prev_exit & 255);
        o.dc[0] = p0;
        o.dc[1] = p1;
        o.dc[2] = p2;
        if (errpos) *errpos = epos;
        return o;
      }
      ck->state[ci] = st;
      ck->acc[ci] = make_int4(o.blocks, p0, p1, p2);
      ++ci;
      next_cp = ci < kCkpts ? ck->first + ci * ck->step : 0xFFFFFFFFu;
    }
    ++o.symbols;
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
      if (MODE != 0 && o.err == kNoErr) {
        o.err = o.blocks;
        epos = pos;
      }
      if (MODE == 2 || ran_out) {
        pos = seg_bits;
        break;
      }
      ++pos;
      u = 0;
      z = 0;
      c = T.comp(0);
      dct = T.dct(c);
      act = T.act(c);
      continue;
    }
    // the symbol's effect without branching on its kind (lanes of a warp decode different
    // streams): DC (z == 0, r = 0: the value is the difference), AC with a value (z += r,
    // the coefficient, z += 1), ZRL (r = 15, s = 0: z += 16 = r + 1) or EOB (the block ends)
    const bool dc = z == 0;
    const int val = s ? extend((v << len) >> ((32 - s) & 31), s) : 0;
    const int dcv = dc ? val : 0;
    // libjpeg: last_dc_val[ci] += diff (int), the block keeps (JCOEF) last_dc_val
    p0 += c == 0 ? dcv : 0;
    p1 += c == 1 ? dcv : 0;
    p2 += c == 2 ? dcv : 0;
    if (MODE == 2) {
      if (dc)
        coef[static_cast<int64_t>(block) * 64] = static_cast<int16_t>(c == 0 ? p0 : c == 1 ? p1 : p2);
      else if (s)
        coef[static_cast<int64_t>(block) * 64 + c_zig[z + r]] = static_cast<int16_t>(val);
    }
    const int zn = (dc || s != 0 || r == 15) ? z + r + 1 : 64;
    pos += used;
    const bool bend = zn >= 64;
    z = bend ? 0 : zn;
    o.blocks += bend ? 1 : 0;
    u = bend ? (u + 1 == T.bmcu ? 0 : u + 1) : u;
    c = T.comp(u);
    dct = T.dct(c);
    act = T.act(c);
    if (MODE == 2 && bend && ++block >= block_limit) break;
  }
  if (CK)
    for (int i = ci; i < kCkpts; ++i) ck->state[i] = -1;  // not reached by this decode
  o.pos = pos;
  o.u = u;
  o.z = z;
  o.dc[0] = p0;
  o.dc[1] = p1;
  o.dc[2] = p2;
  if (errpos) *errpos = epos;
  return o;
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

// Huffman tables of the (at most two) images a CTA's chunk of 256 slots belongs to, in
// shared memory; slots of a third image in the same chunk (tiny images) read the
// descriptor's tables from global memory.
struct ChunkTables {
  JHuff tab[2][4];
  int img[2];
};

__device__ inline const JHuff* chunk_tables(ChunkTables& ct, const JDesc* descs, int n,
                                            int64_t base, int64_t total, int my_k) {
  const int k0 = find_image(descs, n, base, 0);
  const int k1 = find_image(descs, n, min(base + static_cast<int64_t>(blockDim.x) - 1, total - 1), 0);
  __syncthreads();  // the previous chunk's readers are done
  for (int side = 0; side < 2; ++side) {
    const int k = side == 0 ? k0 : k1;
    if (side == 1 && k1 == k0) break;
    if (ct.img[side] == k) continue;  // still loaded (same value in every thread)
    const int4* src = reinterpret_cast<const int4*>(descs[k].dc);
    int4* dst = reinterpret_cast<int4*>(ct.tab[side]);
    constexpr int kWords = static_cast<int>(4 * sizeof(JHuff) / 16);
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ct.img[0] = k0;
    ct.img[1] = k1;
  }
  // (every thread read ct.img before the first barrier above; the writes land after it)
  return my_k == k0 ? ct.tab[0] : my_k == k1 ? ct.tab[1] : descs[my_k].dc;
}

__device__ inline void init_ckpt(Ckpt& ck, const Work& W, int64_t g, int j, int sub_bits) {
  ck.state = W.ck_state + g * kCkpts;
  ck.acc = W.ck_acc + g * kCkpts;
  ck.step = static_cast<uint32_t>(sub_bits) / (kCkpts + 1);
  ck.first = static_cast<uint32_t>(j) * sub_bits + ck.step;
  ck.compare = false;
}

__device__ __forceinline__ void unpack_state(long long e, uint32_t& pos, int& u, int& z) {
  pos = static_cast<uint32_t>(e >> 16);
  u = static_cast<int>((e >> 8) & 255);
  z = static_cast<int>(e & 255);
}

// block-wide exclusive scan of 4 ints (x: block counts, y..w: DC sums)
__device__ inline int4 block_scan4(int4 v, int4* sh, int4& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int4 x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int4 y;
    y.x = __shfl_up_sync(0xffffffffu, x.x, d);
    y.y = __shfl_up_sync(0xffffffffu, x.y, d);
    y.z = __shfl_up_sync(0xffffffffu, x.z, d);
    y.w = __shfl_up_sync(0xffffffffu, x.w, d);
    if (lane >= d) {
      x.x += y.x;
      x.y += y.y;
      x.z += y.z;
      x.w += y.w;
    }
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  int4 pre = make_int4(0, 0, 0, 0);
  for (int w = 0; w < warp; ++w) {
    pre.x += sh[w].x;
    pre.y += sh[w].y;
    pre.z += sh[w].z;
    pre.w += sh[w].w;
  }
  total = make_int4(0, 0, 0, 0);
  for (int w = 0; w < nw; ++w) {
    total.x += sh[w].x;
    total.y += sh[w].y;
    total.z += sh[w].z;
    total.w += sh[w].w;
  }
  __syncthreads();
  return make_int4(pre.x + x.x - v.x, pre.y + x.y - v.y, pre.z + x.z - v.z, pre.w + x.w - v.w);
}

#ifndef TP_JPEG_HUFF_MINB  // resident CTAs per SM the register allocation must allow
#define TP_JPEG_HUFF_MINB 1
#endif
__global__ void __launch_bounds__(256, TP_JPEG_HUFF_MINB) k_jpeg_huff(const JDesc* __restrict__ descs, int n,
                                                   int64_t total_slots, int sub_bits,
                                                   int lead_bits, uint8_t* __restrict__ work,
                                                   int32_t* __restrict__ status) {
  cg::grid_group grid = cg::this_grid();
  __shared__ ChunkTables ct;
  __shared__ int4 scan_sh[8];
  __shared__ int bad_sh;
  const Work W = work_view(work, total_slots);
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (threadIdx.x == 0) ct.img[0] = ct.img[1] = -1;
  if (tid == 0) W.stamps[0] = gtimer();
  const uint32_t overlap = lead_bits > 0 ? static_cast<uint32_t>(lead_bits)
                                         : static_cast<uint32_t>(sub_bits);  // speculative lead-in

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

  // (1) every subsequence: a speculative lead-in of `overlap` bits before its start (from a
  // guessed state; from the interval start, exactly, when that is closer), which almost
  // always falls into the true path, then the counting decode of its own bits
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < total_slots; base += nthreads) {
    const int64_t g = base + threadIdx.x;
    SlotRef r;
    const bool on = g < total_slots && slot_ref(descs, n, work, status, g, r);
    const JHuff* tabs = chunk_tables(ct, descs, n, base, total_slots, on ? r.k : -1);
    if (!on) continue;
    const JDesc& d = descs[r.k];
    Tabs T;
    T.load(d, tabs);
    BitReader br;
    br.init(work + d.clean_off);
    const uint32_t start = static_cast<uint32_t>(r.j) * sub_bits;
    const uint32_t stop = min(start + static_cast<uint32_t>(sub_bits), r.seg_bits);
    uint32_t pos = 0;
    int u = 0, z = 0;
    if (r.j > 0) {
      const uint32_t lead = start > overlap ? start - overlap : 0u;
      const DecOut s0 = decode_run<0, false>(T, br, r.bit0, r.seg_bits, start, lead, 0, 0, nullptr,
                                             0, 0, nullptr);
      pos = s0.pos;
      u = s0.u;
      z = s0.z;
    }
    Ckpt ck;
    init_ckpt(ck, W, g, r.j, sub_bits);
    uint32_t ep;
    const DecOut o = decode_run<1, true>(T, br, r.bit0, r.seg_bits, stop, pos, u, z, nullptr, 0, 0,
                                         nullptr, &ck, &ep);
    W.entry[g] = pack_state(pos, u, z);
    W.exitp[g] = pack_state(o.pos, o.u, o.z);
    W.blocks[g] = o.blocks;
    W.err[g] = o.err;
    W.errpos[g] = static_cast<int>(ep);
    W.dcs[g] = make_int4(0, o.dc[0], o.dc[1], o.dc[2]);
    W.claim[g] = 0;
  }
  if (tid == 0) W.stamps[1] = gtimer();

  // (2) half-rounds: a subsequence whose recorded entry is not its predecessor's exit
  // re-decodes from that exit (stopping as soon as it rejoins its recorded path); one
  // parity per half-round, so no exit is read while it is rewritten
  int h = 2;
  for (; h < kMaxSteps; ++h) {
    grid.sync();
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < total_slots; base += nthreads) {
      const int64_t g = base + threadIdx.x;
      SlotRef r;
      bool need = g < total_slots && slot_ref(descs, n, work, status, g, r) && r.j > 0 &&
                  (r.j & 1) == (h & 1) && W.exitp[g - 1] != W.entry[g];
      if (!__syncthreads_or(need)) continue;
      const JHuff* tabs = chunk_tables(ct, descs, n, base, total_slots, need ? r.k : -1);
      if (!need) continue;
      const JDesc& d = descs[r.k];
      Tabs T;
      T.load(d, tabs);
      BitReader br;
      br.init(work + d.clean_off);
      const int32_t* sub_prefix =
          reinterpret_cast<const int32_t*>(work + d.seg_off) + d.n_seg + 1;
      const int n_sub = sub_prefix[r.s + 1] - sub_prefix[r.s];
      long long e = W.exitp[g - 1];
      // a changed exit is carried into the next subsequence(s) right away: that one has
      // the other parity, so no other thread decodes it in this half-round, and a chain
      // of subsequences that missed their lead-in is resolved in one half-round, not one
      // half-round per link (the successor of the chain is re-checked next half-round)
      for (int hop = 0, j = r.j; hop < kMaxHops && j < n_sub; ++hop, ++j) {
        const int64_t gg = g + hop;
        if (hop > 0 && W.entry[gg] == e) break;
        // one decode per slot and half-round: a chain running into a slot another thread
        // took (or the other way round) stops; the next half-round re-checks it
        if (atomicMax(W.claim + gg, h) == h) break;
        atomicAdd(W.counters + 512 + h, 1u);
        uint32_t pos;
        int u, z;
        unpack_state(e, pos, u, z);
        const uint32_t stop = min(static_cast<uint32_t>(j + 1) * sub_bits, r.seg_bits);
        Ckpt ck;
        init_ckpt(ck, W, gg, j, sub_bits);
        ck.compare = true;
        ck.prev_exit = W.exitp[gg];
        ck.prev_blocks = W.blocks[gg];
        ck.prev_err = W.err[gg];
        ck.prev_errpos = static_cast<uint32_t>(W.errpos[gg]);
        ck.prev_dc = W.dcs[gg];
        uint32_t ep;
        const long long c0 = clock64();
        const DecOut o = decode_run<1, true>(T, br, r.bit0, r.seg_bits, stop, pos, u, z, nullptr,
                                             0, 0, nullptr, &ck, &ep);
        if (h < 128) {  // diagnostics: the longest re-decode of this half-round
          atomicMax(W.counters + 256 + h, static_cast<unsigned>(o.symbols));
          atomicMax(W.counters + 384 + h, static_cast<unsigned>(min(clock64() - c0, 0x7FFFFFFFLL)));
        }
        const long long x = pack_state(o.pos, o.u, o.z);
        W.entry[gg] = e;
        W.blocks[gg] = o.blocks;
        W.err[gg] = o.err;
        W.errpos[gg] = static_cast<int>(ep);
        W.dcs[gg] = make_int4(0, o.dc[0], o.dc[1], o.dc[2]);
        if (x == W.exitp[gg]) break;
        W.exitp[gg] = x;
        atomicAdd(W.counters + h, 1u);
        e = x;
      }
    }
    grid.sync();
    if (tid == 0 && h < 64) reinterpret_cast<unsigned long long*>(W.counters + 640)[h] = gtimer();
    if (h >= 3 && W.counters[h] == 0 && W.counters[h - 1] == 0) break;
  }
  const bool converged = h < kMaxSteps;
  if (tid == 0) {
    W.counters[1023] = h;
    W.stamps[2] = gtimer();
  }

  // (3) per interval (one CTA per image): first block and entry DC predictors of every
  //     subsequence (block scans); unclean streams go to the host
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const JDesc& d = descs[k];
    if (d.n_slots == 0 || status[k]) continue;
    const int32_t* seg_start = reinterpret_cast<const int32_t*>(work + d.seg_off);
    const int32_t* sub_prefix = seg_start + d.n_seg + 1;
    bool bad = false;
    for (int s = 0; s < d.n_seg; ++s) {
      const int T = seg_blocks(d, s);
      const int first = s * d.ri * d.bmcu;
      int4 carry = make_int4(0, 0, 0, 0);  // DC predictors reset at each restart
      for (int t0 = sub_prefix[s]; t0 < sub_prefix[s + 1]; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const int64_t g = d.slot_base + t;
        const bool on = t < sub_prefix[s + 1];
        int4 v = make_int4(0, 0, 0, 0);
        if (on) {
          const int4 dv = W.dcs[g];
          v = make_int4(W.blocks[g], dv.y, dv.z, dv.w);
        }
        int4 tot;
        const int4 ex = block_scan4(v, scan_sh, tot);
        if (on) {
          const int before = carry.x + ex.x;
          W.bstart[g] = first + before;
          W.dcs[g] = make_int4(0, carry.y + ex.y, carry.z + ex.z, carry.w + ex.w);
          const int e = W.err[g];
          if (e != kNoErr && before + e < T) bad = true;
          if (!converged && t > sub_prefix[s] && W.exitp[g - 1] != W.entry[g]) bad = true;
        }
        carry.x += tot.x;
        carry.y += tot.y;
        carry.z += tot.z;
        carry.w += tot.w;
      }
      if (carry.x < T) bad = true;  // the data ends before the interval's last block
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status + k, TP_JPEG_CORRUPT);
  }
  grid.sync();
  if (tid == 0) W.stamps[3] = gtimer();

  // (4) write pass: coefficients, with the DC values predicted in place
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < total_slots; base += nthreads) {
    const int64_t g = base + threadIdx.x;
    SlotRef r;
    const bool on = g < total_slots && slot_ref(descs, n, work, status, g, r);
    const JHuff* tabs = chunk_tables(ct, descs, n, base, total_slots, on ? r.k : -1);
    if (!on) continue;
    const JDesc& d = descs[r.k];
    Tabs T;
    T.load(d, tabs);
    BitReader br;
    br.init(work + d.clean_off);
    uint32_t pos;
    int u, z;
    unpack_state(W.entry[g], pos, u, z);
    const uint32_t stop = min(static_cast<uint32_t>(r.j + 1) * sub_bits, r.seg_bits);
    const int limit = r.s * d.ri * d.bmcu + seg_blocks(d, r.s);
    const int4 pv = W.dcs[g];
    const int pred[3] = {pv.y, pv.z, pv.w};
    decode_run<2, false>(T, br, r.bit0, r.seg_bits, stop, pos, u, z,
                         reinterpret_cast<int16_t*>(work + d.coef_off), W.bstart[g], limit, pred);
  }
  if (tid == 0) W.stamps[4] = gtimer();
  (void)bad_sh;
}

// ---------------------------------------------------------------------------
// J3: ISLOW IDCT (jidctint.c), 8 threads per block

constexpr int F0298 = 2446, F0390 = 3196, F0541 = 4433, F0765 = 6270, F0899 = 7373, F1175 = 9633,
              F1501 = 12299, F1847 = 15137, F1961 = 16069, F2053 = 16819, F2562 = 20995,
              F3072 = 25172;

// One jidctint.c butterfly.  libjpeg computes in JLONG (64-bit on LP64); T = int is
// exact whenever the inputs are bounded as the callers check (|in| <= 2^13 keeps every
// intermediate below 2^30.3), T = long long otherwise (corrupt-looking coefficients).
template <typename T>
__device__ __forceinline__ void idct_1d(const T (&in)[8], T (&out)[8]) {
  T z2 = in[2], z3 = in[6];
  T z1 = (z2 + z3) * F0541;
  const T tmp2 = z1 + z3 * -F1847;
  const T tmp3 = z1 + z2 * F0765;
  const T tmp0 = (in[0] + in[4]) * 8192;  // << CONST_BITS
  const T tmp1 = (in[0] - in[4]) * 8192;
  const T tmp10 = tmp0 + tmp3, tmp13 = tmp0 - tmp3, tmp11 = tmp1 + tmp2, tmp12 = tmp1 - tmp2;
  T t0 = in[7], t1 = in[5], t2 = in[3], t3 = in[1];
  z1 = t0 + t3;
  z2 = t1 + t2;
  z3 = t0 + t2;
  T z4 = t1 + t3;
  const T z5 = (z3 + z4) * F1175;
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

__device__ __forceinline__ uint32_t range_limit(int x) {
  const uint32_t v = static_cast<uint32_t>(x) & 1023u;  // RANGE_MASK
  return v < 128 ? v + 128 : v < 512 ? 255u : v < 896 ? 0u : v - 896;
}

// pass 1 of one column: DEQUANTIZE (short coef x short quant, ISLOW_MULT_TYPE) then the
// butterfly, DESCALE(x, CONST_BITS - PASS1_BITS) into the int workspace
__device__ __forceinline__ void idct_col(const int (&dq)[8], int (&ws)[8]) {
  int m = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) m = max(m, abs(dq[r]));
  if (m <= (1 << 13)) {
    int out[8];
    idct_1d<int>(dq, out);
#pragma unroll
    for (int r = 0; r < 8; ++r) ws[r] = (out[r] + (1 << 10)) >> 11;
  } else {
    long long in[8], out[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) in[r] = dq[r];
    idct_1d<long long>(in, out);
#pragma unroll
    for (int r = 0; r < 8; ++r) ws[r] = static_cast<int>((out[r] + (1LL << 10)) >> 11);
  }
}

// pass 2 of one row: butterfly, DESCALE(x, CONST_BITS + PASS1_BITS + 3), range limit
__device__ __forceinline__ void idct_row(const int (&w)[8], uint32_t& lo, uint32_t& hi) {
  int m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) m = max(m, abs(w[i]));
  int px[8];
  if (m <= (1 << 13)) {
    int out[8];
    idct_1d<int>(w, out);
#pragma unroll
    for (int i = 0; i < 8; ++i) px[i] = (out[i] + (1 << 17)) >> 18;
  } else {
    long long in[8], out[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) in[i] = w[i];
    idct_1d<long long>(in, out);
#pragma unroll
    for (int i = 0; i < 8; ++i) px[i] = static_cast<int>((out[i] + (1LL << 17)) >> 18);
  }
  lo = hi = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    lo |= range_limit(px[i]) << (8 * i);
    hi |= range_limit(px[i + 4]) << (8 * i);
  }
}

// q = a / b, r = a % b for 0 <= a < 2^24, b >= 1, through a float reciprocal and one
// correction step (an integer division is ~20 instructions on the GPU)
__device__ __forceinline__ void div_small(int a, int b, int& q, int& r) {
  q = __float2int_rz(__int2float_rn(a) * __frcp_rn(__int2float_rn(b)));
  r = a - q * b;
  if (r < 0) {
    --q;
    r += b;
  } else if (r >= b) {
    ++q;
    r -= b;
  }
}

// One thread per block: the 64 coefficients in registers (eight 16-byte loads), eight
// column transforms then eight row transforms, eight 8-byte row stores.  (Eight threads per
// block spent ~4x more instructions on per-thread set-up than on the transforms.)
__global__ void __launch_bounds__(128) k_jpeg_idct(const JDesc* __restrict__ descs, int n,
                                                   int64_t total_blocks, uint8_t* __restrict__ work,
                                                   const int32_t* __restrict__ status) {
  int ck_img = -1;
  int64_t ck_lo = 0, ck_hi = 0;
  for (int64_t gb = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; gb < total_blocks;
       gb += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!(ck_img >= 0 && gb >= ck_lo && gb < ck_hi)) {  // consecutive blocks: same image
      ck_img = find_image(descs, n, gb, 1);
      ck_lo = descs[ck_img].block_base;
      ck_hi = ck_lo + descs[ck_img].n_blocks;
    }
    const JDesc* d = descs + ck_img;
    if (d->n_slots == 0 || status[ck_img] != 0) continue;
    const int b = static_cast<int>(gb - d->block_base);
    int mcu, u;
    div_small(b, d->bmcu, mcu, u);
    const int c = d->slot_comp[u];
    const uint4* src = reinterpret_cast<const uint4*>(
        reinterpret_cast<const int16_t*>(work + d->coef_off) + static_cast<int64_t>(b) * 64);
    const uint4* qsrc = reinterpret_cast<const uint4*>(d->quant[c]);
    int blk[8][8];  // [row][col], dequantized, then the workspace, then the output
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint4 cv = src[r], qv = qsrc[r];
      const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w}, qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)  // DEQUANTIZE: short coef x short quant (ISLOW_MULT_TYPE)
        blk[r][i] = static_cast<int>(static_cast<int16_t>(cw[i >> 1] >> (16 * (i & 1)))) *
                    static_cast<int>(static_cast<int16_t>(qw[i >> 1] >> (16 * (i & 1))));
    }
#pragma unroll
    for (int col = 0; col < 8; ++col) {  // pass 1: columns
      int in[8], w[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) in[r] = blk[r][col];
      idct_col(in, w);
#pragma unroll
      for (int r = 0; r < 8; ++r) blk[r][col] = w[r];
    }
    int my, mx;
    div_small(mcu, d->mcux, my, mx);
    const int by = d->ncomp == 1 ? my : my * d->comp_v[c] + d->slot_bv[u];
    const int bx = d->ncomp == 1 ? mx : mx * d->comp_h[c] + d->slot_bh[u];
    uint8_t* dst = work + d->plane_off[c] + static_cast<int64_t>(by * 8) * d->plane_w[c] + bx * 8;
#pragma unroll
    for (int r = 0; r < 8; ++r) {  // pass 2: rows
      uint32_t lo, hi;
      idct_row(blk[r], lo, hi);
      *reinterpret_cast<uint2*>(dst + static_cast<int64_t>(r) * d->plane_w[c]) = make_uint2(lo, hi);
    }
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

__device__ __forceinline__ uint32_t ycc_px(int Y, int cb, int cr) {
  // jdcolor.c build_ycc_rgb_table: FIX(x) = x * 65536 + 0.5, ONE_HALF = 32768
  const int r = Y + ((91881 * cr + 32768) >> 16);
  const int g = Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16);
  const int b = Y + ((116130 * cb + 32768) >> 16);
  return clamp255(r) | (clamp255(g) << 8) | (clamp255(b) << 16);
}

// One CTA per output row; each thread 4 consecutive pixels (12 bytes, three 32-bit stores
// when the row is 4-byte aligned, which it is whenever the width is a multiple of 4).
__global__ void __launch_bounds__(256) k_jpeg_color(const JDesc* __restrict__ descs, int n,
                                                    int64_t total_rows, const uint8_t* __restrict__ work,
                                                    uint8_t* __restrict__ out,
                                                    const int32_t* __restrict__ status) {
  int k = -1;
  int64_t lo = 0, hi = 0;
  for (int64_t gr = blockIdx.x; gr < total_rows; gr += gridDim.x) {
    if (!(k >= 0 && gr >= lo && gr < hi)) {  // rows of one image are consecutive
      k = find_image(descs, n, gr, 2);
      lo = descs[k].row_base;
      hi = lo + descs[k].height;
    }
    const JDesc& d = descs[k];
    if (d.n_slots == 0 || status[k]) continue;
    const int y = static_cast<int>(gr - d.row_base);
    const int W = d.width;
    uint8_t* o = out + d.out_off + static_cast<int64_t>(y) * W * 3;
    const bool aligned = (reinterpret_cast<uintptr_t>(o) & 3) == 0;
    const uint8_t* py = work + d.plane_off[0] + static_cast<int64_t>(y) * d.plane_w[0];
    const int hx = d.ncomp == 1 ? 1 : d.hmax / d.comp_h[1], vx = d.ncomp == 1 ? 1 : d.vmax / d.comp_v[1];
    const uint8_t* pcb = work + d.plane_off[d.ncomp == 1 ? 0 : 1];
    const uint8_t* pcr = work + d.plane_off[d.ncomp == 1 ? 0 : 2];
    // the chroma rows this output row reads: nearer row and (h2v2) the further one, the
    // jdmainct.c context rows replicating the edges
    const int dsw = d.ds_w[1], dsh = d.ds_h[1];
    const int crow = vx == 2 ? y >> 1 : y;
    const int orow = vx == 2 ? ((y & 1) ? min(crow + 1, dsh - 1) : max(crow - 1, 0)) : crow;
    const int64_t pw1 = d.plane_w[1];
    const uint8_t* cb0 = pcb + crow * pw1;
    const uint8_t* cb1 = pcb + orow * pw1;
    const uint8_t* cr0 = pcr + crow * pw1;
    const uint8_t* cr1 = pcr + orow * pw1;
    const bool fancy = hx == 2 && dsw > 2;
    // 8 pixels per thread: one 8-byte Y load; for the fancy paths the chroma column sums
    // at 4t - 1 .. 4t + 4 come from one aligned word per row and plane plus its two
    // neighbours (clamped at the plane's real edges, which reproduces jdsample.c's first
    // and last column cases)
    for (int x0 = 8 * threadIdx.x; x0 < W; x0 += 8 * blockDim.x) {
      const uint2 yv = *reinterpret_cast<const uint2*>(py + x0);  // planes are 8-padded
      uint32_t px[8];
      if (d.ncomp == 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) px[i] = (((i < 4 ? yv.x : yv.y) >> (8 * (i & 3))) & 255) * 0x010101u;
      } else if (fancy) {
        const int i0 = x0 >> 1;  // chroma columns i0 .. i0 + 3
        int cb[6], cr[6];        // column sums at i0 - 1 .. i0 + 4
        if (i0 >= 1 && i0 + 4 <= dsw - 1) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(cb0 + i0);
          const uint32_t r0 = *reinterpret_cast<const uint32_t*>(cr0 + i0);
          const uint32_t b1 = vx == 2 ? *reinterpret_cast<const uint32_t*>(cb1 + i0) : 0u;
          const uint32_t r1 = vx == 2 ? *reinterpret_cast<const uint32_t*>(cr1 + i0) : 0u;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int bb0 = (b0 >> (8 * q)) & 255, rr0 = (r0 >> (8 * q)) & 255;
            cb[q + 1] = vx == 2 ? bb0 * 3 + static_cast<int>((b1 >> (8 * q)) & 255) : bb0;
            cr[q + 1] = vx == 2 ? rr0 * 3 + static_cast<int>((r1 >> (8 * q)) & 255) : rr0;
          }
          cb[0] = vx == 2 ? cb0[i0 - 1] * 3 + cb1[i0 - 1] : cb0[i0 - 1];
          cr[0] = vx == 2 ? cr0[i0 - 1] * 3 + cr1[i0 - 1] : cr0[i0 - 1];
          cb[5] = vx == 2 ? cb0[i0 + 4] * 3 + cb1[i0 + 4] : cb0[i0 + 4];
          cr[5] = vx == 2 ? cr0[i0 + 4] * 3 + cr1[i0 + 4] : cr0[i0 + 4];
        } else {
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const int ii = min(max(i0 - 1 + q, 0), dsw - 1);
            cb[q] = vx == 2 ? cb0[ii] * 3 + cb1[ii] : cb0[ii];
            cr[q] = vx == 2 ? cr0[ii] * 3 + cr1[ii] : cr0[ii];
          }
        }
        const int sh = vx == 2 ? 4 : 2;
        const int be = vx == 2 ? 8 : 1, bo = vx == 2 ? 7 : 2;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int q = 1 + (i >> 1);              // this column's sum
          const int nb = (i & 1) ? q + 1 : q - 1;  // the neighbour it blends with
          const int bias = (i & 1) ? bo : be;
          const int ccb = ((cb[q] * 3 + cb[nb] + bias) >> sh) - 128;
          const int ccr = ((cr[q] * 3 + cr[nb] + bias) >> sh) - 128;
          px[i] = ycc_px(((i < 4 ? yv.x : yv.y) >> (8 * (i & 3))) & 255, ccb, ccr);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int x = min(x0 + i, W - 1);
          const int ci = hx == 2 ? x >> 1 : x;  // 4:4:4, or plain replication (dsw <= 2)
          px[i] = ycc_px(((i < 4 ? yv.x : yv.y) >> (8 * (i & 3))) & 255, cb0[ci] - 128, cr0[ci] - 128);
        }
      }
      if (aligned && x0 + 8 <= W) {
        uint32_t* o32 = reinterpret_cast<uint32_t*>(o + 3 * x0);
#pragma unroll
        for (int h4 = 0; h4 < 2; ++h4) {
          const uint32_t* p4 = px + 4 * h4;
          o32[3 * h4] = p4[0] | (p4[1] << 24);
          o32[3 * h4 + 1] = (p4[1] >> 8) | (p4[2] << 16);
          o32[3 * h4 + 2] = (p4[2] >> 16) | (p4[3] << 8);
        }
      } else {
        for (int i = 0; i < 8 && x0 + i < W; ++i) {
          o[3 * (x0 + i)] = static_cast<uint8_t>(px[i]);
          o[3 * (x0 + i) + 1] = static_cast<uint8_t>(px[i] >> 8);
          o[3 * (x0 + i) + 2] = static_cast<uint8_t>(px[i] >> 16);
        }
      }
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
  const int64_t chunks = totals[5];
  if (chunks > 0) {
    int2* counts = reinterpret_cast<int2*>(work + totals[6]);
    k_jpeg_unstuff_count<<<static_cast<unsigned>(chunks), kUnstuffThreads, 0, s>>>(d_payload, descs, n, counts, d_status);
    k_jpeg_unstuff_write<<<static_cast<unsigned>(chunks), kUnstuffThreads, 0, s>>>(d_payload, descs, n, counts, work, d_status);
  }
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
    int lb = static_cast<int>(totals[7]);  // speculative lead-in bits (0: sub_bits)
    int32_t* st = d_status;
    void* args[] = {&descs, &nn, &ts, &sb, &lb, &work, &st};
    cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_jpeg_huff), grid, 256,
                                                args, 0, s);
    if (e != cudaSuccess) return set_error(TP_ERR_CUDA, "tp_jpeg_decode: %s", cudaGetErrorString(e));
  }
  if (blocks > 0) {
    const int64_t g = (blocks + 127) / 128;
    k_jpeg_idct<<<static_cast<unsigned>(g < 32 * sms ? g : 32 * sms), 128, 0, s>>>(descs, n, blocks, work, d_status);
  }
  if (rows > 0) {
    k_jpeg_color<<<static_cast<unsigned>(rows < 64 * sms ? rows : 64 * sms), 256, 0, s>>>(descs, n, rows, work, d_out, d_status);
  }
  return check_launch("tp_jpeg_decode");
}

}  // extern "C"
