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
        // the r-th marker must be RST(r mod 8); libjpeg resynchronizes on any other
        // (jdmarker.c read_restart_marker / jpeg_resync_to_restart): left to the host
        if (raw[p0 + i] != 0xD0 + (r & 7)) atomicOr(status + k, TP_JPEG_CORRUPT);
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
#ifndef TP_JPEG_NOSTORE  // measurement only: the write pass without its stores (wrong output)
#define TP_JPEG_NOSTORE 0
#endif
#ifndef TP_JPEG_STAGED  // write pass: blocks staged in shared memory, one bulk store each
#define TP_JPEG_STAGED 1
#endif

// The write pass's coefficient staging: one 128-byte block per thread in shared memory
// (144-byte stride: 16-byte aligned for the bulk copy, lanes spread over the banks; the
// pad takes the dummy store of EOB / ZRL symbols, so every symbol stores unconditionally).
// A block that completes inside the thread's range leaves with one cp.async.bulk (128
// bytes, a whole line); the partial blocks at a subsequence's two ends store just their
// own coefficient range [zlo, z) -- the neighbouring subsequence stores the rest -- so the
// coefficient buffer needs no zeroing (the 400 MB memset of a 64 x 1080p batch is gone).
// 64 x 1080p: K7 2.70 -> 2.57 ms (scattered 2-byte global stores + memset before;
// profiles/r02/jpeg/ab_staged_write.log).
#ifndef TP_JPEG_STAGE_BULK  // 1: a block leaves through cp.async.bulk; 0: plain 16-byte stores
#define TP_JPEG_STAGE_BULK 1
#endif
#ifndef TP_JPEG_STAGE_SLOTS  // 128-byte blocks staged per thread (2: the copy out of one
#define TP_JPEG_STAGE_SLOTS 1  // overlaps the decode into the other, but the extra 32 KB of
#endif                         // shared memory per CTA costs the decode its L1: slower)
constexpr int kStageStride = 128 * TP_JPEG_STAGE_SLOTS + 16;  // bytes per thread
struct Stage {
  uint8_t* base;  // this thread's 2 x 128 bytes
  int slot;       // the current block's slot
};

__device__ __forceinline__ void stage_zero(uint8_t* p) {
  uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
  for (int i = 0; i < 8; ++i) q[i] = make_uint4(0u, 0u, 0u, 0u);
}

__device__ __forceinline__ void bulk_store128(void* gdst, const void* ssrc) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> async proxy
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(gdst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc)))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int MODE, bool CK>
__device__ DecOut decode_run(const Tabs& T, BitReader& br, uint32_t bit0, uint32_t seg_bits,
                             uint32_t stop, uint32_t pos, int u, int z, int16_t* coef, int block,
                             int block_limit, const int* pred_in, const Ckpt* ck = nullptr,
                             uint32_t* errpos = nullptr, Stage* stage = nullptr) {
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
  // staged write pass: the current block's coefficients from zlo on are this thread's
  const bool staged = MODE == 2 && TP_JPEG_STAGED && !TP_JPEG_NOSTORE;
  int zlo = z;
  int16_t* stg = staged ? reinterpret_cast<int16_t*>(stage->base + 128 * stage->slot) : nullptr;
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
    if (staged) {  // one unconditional store (EOB / ZRL write a zero into the pad)
      int16_t* at = dc ? stg : s ? stg + z + r : reinterpret_cast<int16_t*>(stage->base + 128 * TP_JPEG_STAGE_SLOTS);
      *at = static_cast<int16_t>(dc ? (c == 0 ? p0 : c == 1 ? p1 : p2) : val);  // zigzag order
    } else if (MODE == 2 && !TP_JPEG_NOSTORE) {
      if (dc)
        coef[static_cast<int64_t>(block) * 64] = static_cast<int16_t>(c == 0 ? p0 : c == 1 ? p1 : p2);
      else if (s)
        coef[static_cast<int64_t>(block) * 64 + z + r] = static_cast<int16_t>(val);  // zigzag order
    }
    const int zn = (dc || s != 0 || r == 15) ? z + r + 1 : 64;
    pos += used;
    const bool bend = zn >= 64;
    if (staged && bend) {  // the block is complete: out it goes, the other slot comes in
      int16_t* dst = coef + static_cast<int64_t>(block) * 64;
      if (zlo == 0 && TP_JPEG_STAGE_BULK) {
        bulk_store128(dst, stg);
      } else if (zlo == 0) {  // eight 16-byte stores: a whole line from one lane
        const uint4* q = reinterpret_cast<const uint4*>(stg);
        uint4* g4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int i = 0; i < 8; ++i) __stcs(g4 + i, q[i]);
      } else {
        for (int i = zlo; i < 64; ++i) dst[i] = stg[i];
      }
      stage->slot = TP_JPEG_STAGE_SLOTS == 2 ? stage->slot ^ 1 : 0;
      stg = reinterpret_cast<int16_t*>(stage->base + 128 * stage->slot);
      if (TP_JPEG_STAGE_BULK) bulk_wait_read<TP_JPEG_STAGE_SLOTS - 1>();  // its last copy read it
      stage_zero(reinterpret_cast<uint8_t*>(stg));
      zlo = 0;
    }
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
  if (staged && z != zlo) {  // the block the next subsequence finishes: [zlo, z) is ours
    int16_t* dst = coef + static_cast<int64_t>(block) * 64;
    for (int i = zlo; i < z; ++i) dst[i] = stg[i];
    stage_zero(reinterpret_cast<uint8_t*>(stg));
  }
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
  extern __shared__ __align__(16) uint8_t stage_mem[];
  Stage stage{stage_mem + kStageStride * threadIdx.x, 0};
  if (TP_JPEG_STAGED) {
    stage_zero(stage.base);
    if (TP_JPEG_STAGE_SLOTS == 2) stage_zero(stage.base + 128);
  }
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
    const DecOut o = decode_run<2, false>(T, br, r.bit0, r.seg_bits, stop, pos, u, z,
                                          reinterpret_cast<int16_t*>(work + d.coef_off),
                                          W.bstart[g], limit, pred, nullptr, nullptr, &stage);
    // This pass walks the true path exactly once and stops at the interval's last block,
    // so an unclean symbol here is damage that libjpeg would conceal.  (Phase 3 can miss
    // one: a re-decode that rejoins a recorded path inherits that path's first error only,
    // and a path that fell into the true one after an early error of its own had it there.)
    if (o.err != kNoErr) atomicOr(status + r.k, TP_JPEG_CORRUPT);
  }
  if (TP_JPEG_STAGED && TP_JPEG_STAGE_BULK) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (tid == 0) W.stamps[4] = gtimer();
}

// ---------------------------------------------------------------------------
// J3: ISLOW IDCT (jidctint.c), one thread per block

constexpr int F0298 = 2446, F0390 = 3196, F0541 = 4433, F0765 = 6270, F0899 = 7373, F1175 = 9633,
              F1501 = 12299, F1847 = 15137, F1961 = 16069, F2053 = 16819, F2562 = 20995,
              F3072 = 25172;

// zigzag index of each natural-order coefficient (the inverse of c_zig): the write pass
// stores coefficients in zigzag order, the IDCT picks them into natural order at compile time
__device__ constexpr int kNat2Zig[64] = {0,  1,  5,  6,  14, 15, 27, 28, 2,  4,  7,  13, 16, 26, 29, 42,
                              3,  8,  12, 17, 25, 30, 41, 43, 9,  11, 18, 24, 31, 40, 44, 53,
                              10, 19, 23, 32, 39, 45, 52, 54, 20, 22, 33, 38, 46, 51, 55, 60,
                              21, 34, 37, 47, 50, 56, 59, 61, 35, 36, 48, 49, 57, 58, 62, 63};

// One jidctint.c butterfly.  libjpeg computes in JLONG (64-bit on LP64); int is exact for
// the inputs the caller lets through (|in| < 2^13 keeps every intermediate below 2^30.3).
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

// The sample limit with CENTERJSAMPLE folded into the descale (x128 = x + 128).  The
// decoder the reference runs is Pillow's libjpeg-turbo, whose x86-64 SIMD ISLOW IDCT
// (jsimd_idct_islow: packssdw, packsswb, + CENTERJSAMPLE) saturates; jdmaster.c's
// range-limit table agrees with that for x in [-512, 511] and wraps beyond (only damaged
// streams get there), so the saturation is what Pillow returns.
__device__ __forceinline__ uint32_t range_limit128(int x128) {
  return static_cast<uint32_t>(min(max(x128, 0), 255));
}

// |v| < 2^13 for all 64 values (min / max trees, three-input VIMNMX3).  The SIMD IDCT keeps
// dequantized coefficients and the pass-1 workspace in 16-bit lanes (pmullw, paddw of
// coefficient pairs, the DC-only << PASS1_BITS, packssdw); under this bound none of those
// overflow and it equals jidctint.c.  A block outside it came from a damaged stream:
// the image goes to Pillow.
__device__ __forceinline__ bool all_small(const int (&v)[8][8]) {
  int mx = v[0][0], mn = v[0][0];
#pragma unroll
  for (int i = 1; i < 64; i += 2) {
    const int a = v[i >> 3][i & 7], b = i + 1 < 64 ? v[(i + 1) >> 3][(i + 1) & 7] : a;
    mx = max(mx, max(a, b));
    mn = min(mn, min(a, b));
  }
  return mx < (1 << 13) && mn > -(1 << 13);
}

// pass 1 (columns): DESCALE(x, CONST_BITS - PASS1_BITS) into the int workspace, in place
template <typename T>
__device__ __forceinline__ void idct_pass1(int (&blk)[8][8]) {
#pragma unroll
  for (int col = 0; col < 8; ++col) {
    T in[8], out[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) in[r] = blk[r][col];
    idct_1d<T>(in, out);
#pragma unroll
    for (int r = 0; r < 8; ++r) blk[r][col] = static_cast<int>((out[r] + T(1 << 10)) >> 11);
  }
}

// pass 2 (rows): DESCALE(x, CONST_BITS + PASS1_BITS + 3) + 128, range limit, 8 bytes a row
template <typename T>
__device__ __forceinline__ void idct_pass2(const int (&blk)[8][8], uint32_t (&lo)[8], uint32_t (&hi)[8]) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    T in[8], out[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) in[i] = blk[r][i];
    idct_1d<T>(in, out);
    uint32_t px[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      px[i] = range_limit128(static_cast<int>((out[i] + T((1 << 17) + (128 << 18))) >> 18));
    lo[r] = __byte_perm(__byte_perm(px[0], px[1], 0x0040), __byte_perm(px[2], px[3], 0x0040), 0x5410);
    hi[r] = __byte_perm(__byte_perm(px[4], px[5], 0x0040), __byte_perm(px[6], px[7], 0x0040), 0x5410);
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

// One thread per block: the 64 zigzag-ordered coefficients in registers (eight 16-byte
// loads), DEQUANTIZE (short coef x short quant, ISLOW_MULT_TYPE) into natural order,
// eight column transforms then eight row transforms, eight 8-byte row stores.  Each CTA
// takes a contiguous range of blocks (one image lookup per CTA, not per block); each pass
// checks its 64 inputs once against the SIMD-exact bound (all_small).
constexpr int kIdctThreads = 128;

__global__ void __launch_bounds__(kIdctThreads) k_jpeg_idct(const JDesc* __restrict__ descs, int n,
                                                            int64_t total_blocks, int64_t per_cta,
                                                            uint8_t* __restrict__ work,
                                                            int32_t* __restrict__ status) {
  const int64_t b_lo = static_cast<int64_t>(blockIdx.x) * per_cta;
  const int64_t b_hi = min(total_blocks, b_lo + per_cta);
  if (b_lo >= b_hi) return;
  int k = find_image(descs, n, b_lo, 1);
  int64_t img_hi = descs[k].block_base + descs[k].n_blocks;
  for (int64_t gb = b_lo + threadIdx.x; gb < b_hi; gb += kIdctThreads) {
    while (gb >= img_hi && k + 1 < n) {  // images' blocks are consecutive
      ++k;
      img_hi = descs[k].block_base + descs[k].n_blocks;
    }
    const JDesc* d = descs + k;
    if (d->n_slots == 0 || status[k] != 0) continue;
    const int b = static_cast<int>(gb - d->block_base);
    int mcu, u;
    div_small(b, d->bmcu, mcu, u);
    const int c = d->slot_comp[u];
    const uint4* src = reinterpret_cast<const uint4*>(
        reinterpret_cast<const int16_t*>(work + d->coef_off) + static_cast<int64_t>(b) * 64);
    uint32_t cw[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = src[i];
      cw[4 * i] = v.x;
      cw[4 * i + 1] = v.y;
      cw[4 * i + 2] = v.z;
      cw[4 * i + 3] = v.w;
    }
    const int4* q4 = reinterpret_cast<const int4*>(d->quant[c]);
    int blk[8][8];  // [row][col]: dequantized, then the workspace
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int4 qv = q4[i];
      const int qs[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int nat = 4 * i + e, zz = kNat2Zig[nat];
        const uint32_t w = cw[zz >> 1];
        const int coef = (zz & 1) ? static_cast<int>(w) >> 16 : static_cast<int>(static_cast<int16_t>(w));
        blk[nat >> 3][nat & 7] = coef * qs[e];
      }
    }
    if (!all_small(blk)) {
      atomicOr(status + k, TP_JPEG_CORRUPT);
      continue;
    }
    idct_pass1<int>(blk);
    if (!all_small(blk)) {
      atomicOr(status + k, TP_JPEG_CORRUPT);
      continue;
    }
    uint32_t lo[8], hi[8];
    idct_pass2<int>(blk, lo, hi);
    int my, mx;
    div_small(mcu, d->mcux, my, mx);
    const int by = d->ncomp == 1 ? my : my * d->comp_v[c] + d->slot_bv[u];
    const int bx = d->ncomp == 1 ? mx : mx * d->comp_h[c] + d->slot_bh[u];
    const int64_t pw = d->plane_w[c];
    uint8_t* dst = work + d->plane_off[c] + static_cast<int64_t>(by * 8) * pw + bx * 8;
#pragma unroll
    for (int r = 0; r < 8; ++r) *reinterpret_cast<uint2*>(dst + r * pw) = make_uint2(lo[r], hi[r]);
  }
}

// ---------------------------------------------------------------------------
// J4: upsampling + colour conversion -> RGB HWC

// jdcolor.c ycc_rgb_convert of one pixel (build_ycc_rgb_table: FIX(x) = x * 65536 + 0.5,
// ONE_HALF = 32768, the tables' CENTERJSAMPLE folded into the constants) -> bytes
// [R, G, B, 0].  R and B are clamped as two 16-bit lanes (add.s16x2 + max.s16x2.relu,
// min.s16x2), G as one 32-bit lane.  ypair = Y | Y << 16.
__device__ __forceinline__ uint32_t ycc_px(uint32_t ypair, int y, int cb, int cr) {
  const int roff = (91881 * cr + (32768 - 91881 * 128)) >> 16;
  const int boff = (116130 * cb + (32768 - 116130 * 128)) >> 16;
  const int goff = (-22554 * cb - 46802 * cr + (32768 + (22554 + 46802) * 128)) >> 16;
  uint32_t rb = __viaddmax_s16x2_relu(__byte_perm(static_cast<uint32_t>(roff), static_cast<uint32_t>(boff), 0x5410),
                                      ypair, 0u);
  asm("min.s16x2 %0, %0, %1;" : "+r"(rb) : "r"(0x00FF00FFu));
  const int g = min(__viaddmax_s32_relu(goff, y, 0), 255);
  return __byte_perm(rb, static_cast<uint32_t>(g), 0x1240);
}

// 4 RGB pixels -> 3 words
__device__ __forceinline__ void pack3(const uint32_t* p4, uint32_t* w3) {
  w3[0] = __byte_perm(p4[0], p4[1], 0x4210);
  w3[1] = __byte_perm(p4[1], p4[2], 0x5421);
  w3[2] = __byte_perm(p4[2], p4[3], 0x6542);
}

__device__ __forceinline__ uint32_t ld32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }

constexpr int kColorThreads = 256;

enum ColorMode { kGray = 0, kH2V2 = 1, kH2V1 = 2, kH1V1 = 3, kRepl = 4 };

struct ColorRow {
  const uint8_t *py, *cb0, *cb1, *cr0, *cr1;  // Y row; chroma nearer / further rows
  int W, dsw;
};

// The raw samples 8 output pixels x0 .. x0 + 7 read (chroma columns i0 .. i0 + 3 and
// their neighbours), loaded one step ahead of their use (the row loop is software
// pipelined: the loads of step s + 1 are in flight while step s converts).
struct Raw8 {
  uint2 y;
  uint32_t nb, fb, nr, fr;  // chroma words: nearer / further row, Cb / Cr
  uint32_t eb[4], er[4];    // neighbour columns (fancy): near L, near R, far L, far R
  uint32_t sel;             // the byte selector repeating the last real column
};

// fancy upsampling (h2v1 / h2v2) loads of one plane; the neighbour bytes are combined
// only when converted, so nothing here waits for the loads
template <bool V2>
__device__ __forceinline__ void load_fancy(const uint8_t* near, const uint8_t* far, uint32_t& n, uint32_t& f,
                                           uint32_t (&e)[4]) {
  // the columns before and after the word, at immediate offsets from one address (the
  // edge cases are selected when converting; the plane has slack before and after it)
  n = ld32(near);
  e[0] = near[-1];
  e[1] = near[4];
  if (V2) {
    f = ld32(far);
    e[2] = far[-1];
    e[3] = far[4];
  } else {
    f = e[2] = e[3] = 0;
  }
}

template <int MODE>
__device__ __forceinline__ void load8(const ColorRow& c, int x0, Raw8& r) {
  r.y = *reinterpret_cast<const uint2*>(c.py + x0);  // planes are 8-padded
  if (MODE == kH2V2 || MODE == kH2V1) {
    const int i0 = x0 >> 1;
    const int lim = c.dsw - 1 - i0;  // >= 0; < 3 only at the plane's right edge
    r.sel = lim >= 3 ? 0x3210u : static_cast<uint32_t>((0x0000221011100000ull >> (16 * min(lim, 2))) & 0xFFFFu);
    load_fancy<MODE == kH2V2>(c.cb0 + i0, c.cb1 + i0, r.nb, r.fb, r.eb);
    load_fancy<MODE == kH2V2>(c.cr0 + i0, c.cr1 + i0, r.nr, r.fr, r.er);
  }
}

// jdsample.c fancy upsampling of one chroma plane for the 8 output pixels, as 16-bit lanes:
// out[0] = (px0, px4), [1] = (px1, px5), [2] = (px2, px6), [3] = (px3, px7).  h2v2 (V2):
// column sums 3 * nearer + further, then (3 * this + neighbour + 8 or 7) >> 4; h2v1:
// (3 * this + neighbour + 1 or 2) >> 2.  Columns past the plane's last real column repeat
// it (its own neighbour, through `sel`), the column before the first is the first
// (clamped neighbour loads): jdsample.c's edge cases.
template <bool V2>
__device__ __forceinline__ void fancy4(uint32_t nw, uint32_t fw, uint32_t sel, const uint32_t (&e)[4],
                                       bool first, bool last, uint32_t (&out)[4]) {
  uint32_t L = e[0], R = e[1];
  if (V2) {
    L = L * 3 + e[2];
    R = R * 3 + e[3];
  }
  const uint32_t n = __byte_perm(nw, 0, sel);
  uint32_t csE = __byte_perm(n, 0, 0x4240), csO = __byte_perm(n, 0, 0x4341);  // cols (0, 2), (1, 3)
  if (V2) {
    const uint32_t f = __byte_perm(fw, 0, sel);
    csE = csE * 3 + __byte_perm(f, 0, 0x4240);
    csO = csO * 3 + __byte_perm(f, 0, 0x4341);
  }
  if (first) L = csE & 0xFFFFu;  // column -1 is column 0
  if (last) R = csO >> 16;       // past the last real column: the last one (sel repeats it)
  const uint32_t LE = csO * 65536u + L;          // cols (-1, 1)
  const uint32_t RO = R * 65536u + (csE >> 16);  // cols (2, 4)
  constexpr uint32_t Be = V2 ? 0x00080008u : 0x00010001u, Bo = V2 ? 0x00070007u : 0x00020002u;
  constexpr int S = V2 ? 4 : 2;
  const uint32_t t3E = csE * 3, t3O = csO * 3;
  out[0] = ((t3E + LE + Be) >> S) & 0x00FF00FFu;
  out[1] = ((t3E + csO + Bo) >> S) & 0x00FF00FFu;
  out[2] = ((t3O + csE + Be) >> S) & 0x00FF00FFu;
  out[3] = ((t3O + RO + Bo) >> S) & 0x00FF00FFu;
}

// RGB of the 8 pixels x0 .. x0 + 7 of one row (x0 < W; pixels past W are don't-cares)
template <int MODE>
__device__ __forceinline__ void color8(const ColorRow& c, int x0, const Raw8& r, uint32_t (&px)[8]) {
  const uint32_t yw[2] = {r.y.x, r.y.y};
  if (MODE == kGray) {
#pragma unroll
    for (int i = 0; i < 8; ++i) px[i] = ((yw[i >> 2] >> (8 * (i & 3))) & 255) * 0x010101u;
    return;
  }
  int cbv[8], crv[8];
  if (MODE == kH2V2 || MODE == kH2V1) {
    uint32_t ub[4], ur[4];
    const int i0 = x0 >> 1;
    const bool first = i0 == 0, last = i0 + 4 > c.dsw - 1;
    fancy4<MODE == kH2V2>(r.nb, r.fb, r.sel, r.eb, first, last, ub);
    fancy4<MODE == kH2V2>(r.nr, r.fr, r.sel, r.er, first, last, ur);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cbv[i] = static_cast<int>((ub[i & 3] >> (16 * (i >> 2))) & 0xFFu);
      crv[i] = static_cast<int>((ur[i & 3] >> (16 * (i >> 2))) & 0xFFu);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int x = min(x0 + i, c.W - 1);
      const int ci = MODE == kRepl ? x >> 1 : x;  // plain replication (dsw <= 2), or 4:4:4
      cbv[i] = c.cb0[ci];
      crv[i] = c.cr0[ci];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ypair = __byte_perm(yw[i >> 2], 0, 0x4040 + 0x0101 * (i & 3));
    px[i] = ycc_px(ypair, static_cast<int>(ypair & 255u), cbv[i], crv[i]);
  }
}

// one step of a row: 8 pixels per lane, 256 per warp; rows starting 16-byte aligned (width
// a multiple of 16) are staged in the warp's shared memory and written with 16-byte
// stores, others with 32-bit (4-byte aligned rows) or byte stores
template <int MODE>
__device__ __forceinline__ void color_step(const ColorRow& c, uint8_t* o, uint8_t* stage, int xw, bool row16,
                                           bool row4, const Raw8& raw) {
  const int lane = threadIdx.x & 31;
  const int x0 = xw + 8 * lane;
  uint32_t px[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (x0 < c.W) color8<MODE>(c, x0, raw, px);
  uint32_t w[6];
  pack3(px, w);
  pack3(px + 4, w + 3);
  if (row16) {
    uint2* st = reinterpret_cast<uint2*>(stage + 24 * lane);
    st[0] = make_uint2(w[0], w[1]);
    st[1] = make_uint2(w[2], w[3]);
    st[2] = make_uint2(w[4], w[5]);
    __syncwarp();
    uint8_t* ow = o + 3 * static_cast<int64_t>(xw);
    const int nbytes = 3 * min(256, c.W - xw);
    if (nbytes == 768) {  // a full step: 48 chunks of 16 bytes
      reinterpret_cast<uint4*>(ow)[lane] = reinterpret_cast<const uint4*>(stage)[lane];
      if (lane < 16)
        reinterpret_cast<uint4*>(ow)[32 + lane] = reinterpret_cast<const uint4*>(stage)[32 + lane];
    } else {
      for (int i = lane; i < (nbytes >> 4); i += 32)
        reinterpret_cast<uint4*>(ow)[i] = reinterpret_cast<const uint4*>(stage)[i];
      for (int i = (nbytes & ~15) + lane; i < nbytes; i += 32) ow[i] = stage[i];
    }
    __syncwarp();
  } else if (x0 < c.W) {
    if (row4 && x0 + 8 <= c.W) {
      uint32_t* o32 = reinterpret_cast<uint32_t*>(o + 3 * x0);
#pragma unroll
      for (int i = 0; i < 6; ++i) o32[i] = w[i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (x0 + i < c.W) {
          o[3 * (x0 + i)] = static_cast<uint8_t>(px[i]);
          o[3 * (x0 + i) + 1] = static_cast<uint8_t>(px[i] >> 8);
          o[3 * (x0 + i) + 2] = static_cast<uint8_t>(px[i] >> 16);
        }
      }
    }
  }
}

// one output row by one warp, step by step; the loads of the next step are in flight while
// a step converts
template <int MODE>
__device__ __forceinline__ void color_row(const ColorRow& c, uint8_t* o, uint8_t* stage) {
  const int lane = threadIdx.x & 31;
  const uintptr_t oa = reinterpret_cast<uintptr_t>(o);
  const bool row16 = (oa & 15) == 0, row4 = (oa & 3) == 0;
  Raw8 raw;
  if (8 * lane < c.W) load8<MODE>(c, 8 * lane, raw);
  for (int xw = 0; xw < c.W; xw += 256) {
    Raw8 next;
    if (xw + 256 + 8 * lane < c.W) load8<MODE>(c, xw + 256 + 8 * lane, next);
    color_step<MODE>(c, o, stage, xw, row16, row4, raw);
    raw = next;
  }
}

// Each CTA takes a contiguous range of output rows, its warps one row each at a time; an
// image's geometry and colour mode are set up once per image and warp (warp-uniform), each
// mode runs its own specialised row code.
__global__ void __launch_bounds__(kColorThreads, 2) k_jpeg_color(const JDesc* __restrict__ descs, int n,
                                                              int64_t total_rows, int64_t per_cta,
                                                              const uint8_t* __restrict__ work,
                                                              uint8_t* __restrict__ out,
                                                              const int32_t* __restrict__ status) {
  __shared__ __align__(16) uint8_t stage[kColorThreads / 32][32 * 24];
  constexpr int kWarps = kColorThreads / 32;
  const int warp = threadIdx.x >> 5;
  const int64_t r_lo = static_cast<int64_t>(blockIdx.x) * per_cta;
  const int64_t r_hi = min(total_rows, r_lo + per_cta);
  if (r_lo + warp >= r_hi) return;
  int k = find_image(descs, n, r_lo + warp, 2) - 1;
  int64_t img_lo = 0, img_hi = -1;
  bool skip = true;
  int mode = kGray, vx = 1, dsh = 1;
  int64_t pw0 = 0, pw1 = 0;
  const uint8_t *pY = nullptr, *pcb = nullptr, *pcr = nullptr;
  uint8_t* o_img = nullptr;
  ColorRow c;
  c.W = 0;
  c.dsw = 1;
  uint8_t* st = stage[warp];
  for (int64_t gr = r_lo + warp; gr < r_hi; gr += kWarps) {
    while (gr >= img_hi && k + 1 < n) {  // the next image: geometry once (warp-uniform)
      ++k;
      const JDesc& d = descs[k];
      img_lo = d.row_base;
      img_hi = img_lo + d.height;
      skip = d.n_slots == 0 || status[k] != 0;
      c.W = d.width;
      const int ncomp = d.ncomp;
      const int hx = ncomp == 1 ? 1 : d.hmax / d.comp_h[1];
      vx = ncomp == 1 ? 1 : d.vmax / d.comp_v[1];
      c.dsw = d.ds_w[1];
      dsh = d.ds_h[1];
      mode = ncomp == 1 ? kGray : hx == 1 ? kH1V1 : c.dsw <= 2 ? kRepl : vx == 2 ? kH2V2 : kH2V1;
      pw0 = d.plane_w[0];
      pw1 = d.plane_w[1];
      pY = work + d.plane_off[0];
      pcb = work + d.plane_off[ncomp == 1 ? 0 : 1];
      pcr = work + d.plane_off[ncomp == 1 ? 0 : 2];
      o_img = out + d.out_off;
    }
    if (skip) continue;
    const int y = static_cast<int>(gr - img_lo);
    uint8_t* o = o_img + static_cast<int64_t>(y) * c.W * 3;
    c.py = pY + static_cast<int64_t>(y) * pw0;
    // the chroma rows this output row reads: nearer row and (h2v2) the further one, the
    // jdmainct.c context rows replicating the edges
    const int crow = vx == 2 ? y >> 1 : y;
    const int orow = vx == 2 ? ((y & 1) ? min(crow + 1, dsh - 1) : max(crow - 1, 0)) : crow;
    c.cb0 = pcb + crow * pw1;
    c.cb1 = pcb + orow * pw1;
    c.cr0 = pcr + crow * pw1;
    c.cr1 = pcr + orow * pw1;
    switch (mode) {
      case kH2V2: color_row<kH2V2>(c, o, st); break;
      case kH2V1: color_row<kH2V1>(c, o, st); break;
      case kH1V1: color_row<kH1V1>(c, o, st); break;
      case kRepl: color_row<kRepl>(c, o, st); break;
      default: color_row<kGray>(c, o, st); break;
    }
  }
}

// resident CTAs per SM of a kernel at `threads` threads (cached per device in `cache`)
template <typename K>
int resident_per_sm(K* kernel, int threads, int dev, int (&cache)[64]) {
  int& v = cache[dev];
  if (v == 0) {
    int r = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kernel, threads, 0);
    v = r > 0 ? r : 1;
  }
  return v;
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
  // (the coefficients need no zeroing when the write pass stages blocks: it stores every
  // coefficient of every block, zeros included)
  if (cudaMemsetAsync(work, 0, 4096, s) != cudaSuccess ||
      (!TP_JPEG_STAGED && cudaMemsetAsync(work + coef_begin, 0, coef_end - coef_begin, s) != cudaSuccess))
    return set_error(TP_ERR_CUDA, "tp_jpeg_decode: memset failed");
  const int sms = device_sm_count();
  const int64_t chunks = totals[5];
  if (chunks > 0) {
    int2* counts = reinterpret_cast<int2*>(work + totals[6]);
    k_jpeg_unstuff_count<<<static_cast<unsigned>(chunks), kUnstuffThreads, 0, s>>>(d_payload, descs, n, counts, d_status);
    k_jpeg_unstuff_write<<<static_cast<unsigned>(chunks), kUnstuffThreads, 0, s>>>(d_payload, descs, n, counts, work, d_status);
  }
  static int idct_occ[64], color_occ[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
    return set_error(TP_ERR_CUDA, "tp_jpeg_decode: no usable device");
  if (slots > 0) {
    static int per_sm_of[64];
    int& per_sm = per_sm_of[dev];
    const int dyn = TP_JPEG_STAGED ? kStageStride * 256 : 0;
    if (per_sm == 0) {
      if (dyn > 0 &&
          cudaFuncSetAttribute(k_jpeg_huff, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess)
        return set_error(TP_ERR_CUDA, "tp_jpeg_decode: decode kernel shared memory");
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jpeg_huff, 256, dyn);
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
                                                args, dyn, s);
    if (e != cudaSuccess) return set_error(TP_ERR_CUDA, "tp_jpeg_decode: %s", cudaGetErrorString(e));
  }
  if (blocks > 0) {
    // contiguous ranges of whole thread-rows, one wave of resident CTAs
    const int64_t target = static_cast<int64_t>(resident_per_sm(k_jpeg_idct, kIdctThreads, dev, idct_occ)) * sms;
    int64_t per = (blocks + target - 1) / target;
    per = (per + kIdctThreads - 1) / kIdctThreads * kIdctThreads;
    const int64_t g = (blocks + per - 1) / per;
    k_jpeg_idct<<<static_cast<unsigned>(g), kIdctThreads, 0, s>>>(descs, n, blocks, per, work, d_status);
  }
  if (rows > 0) {
    // contiguous row ranges, one wave of resident CTAs
    const int64_t target = static_cast<int64_t>(resident_per_sm(k_jpeg_color, kColorThreads, dev, color_occ)) * sms;
    const int64_t per = (rows + target - 1) / target;
    const int64_t g = (rows + per - 1) / per;
    k_jpeg_color<<<static_cast<unsigned>(g), kColorThreads, 0, s>>>(descs, n, rows, per, work, d_out, d_status);
  }
  return check_launch("tp_jpeg_decode");
}

}  // extern "C"
