// K8 — device PNG decode: zlib/deflate inflate (RFC 1951) and
// PNG scanline unfiltering (PNG spec §9) on the B200, replacing the Pillow decode of
// decode_image / _decode_pass (vlmfp/imgproc.py:213-260) for 8-bit L / RGB / P images.
//
// Deflate is a serial format: a block's Huffman codes are only known after its header,
// and a block's end only after decoding it.  The parallel decode follows the
// block-finder design of rapidgzip (Knespel & Brunst 2023):
//   find     one warp per unit (kUnitBits of compressed stream): the first bit position
//            in the unit that carries a plausible block header -- a dynamic header whose
//            code-length code is complete and whose literal/length and distance codes are
//            complete (zlib always writes complete codes), or a stored header whose
//            LEN/NLEN agree and which is followed by another plausible header;
//   inflate  one thread per unit decodes from its start to the first block boundary at
//            or past the next unit's start, into tokens (literal packs, matches, stored
//            blocks), with its own Huffman tables in shared memory;
//   chain    one warp per image checks that every unit ended exactly where the next one
//            starts (a false header is passed by the preceding unit's decode: that start
//            is dropped and the preceding unit is decoded again, up to kRounds rounds),
//            and scans the units' inflated lengths into offsets;
//   expand   one warp per unit turns tokens into bytes (u16 per byte): a back reference
//            that reaches before the unit's start becomes a marker into the 32 KB window
//            before the unit (256 + window position), copied through later references;
//   window   one CTA per image resolves the last 32 KB of each unit in order (each
//            unit's window is then final), `final` resolves everything else in parallel;
//   unfilter one CTA per image: thread = scanline, a wavefront over 4-byte chunks (row y
//            reconstructs chunk i one step after row y-1), L and P expanded to RGB.
// Everything the decode does not take cleanly sets d_status[k]: the host decodes that
// image with Pillow, so pixels (or the error) are the reference's.

#include "png_common.cuh"
#include "tp_common.cuh"

namespace {

using namespace tp::png;

constexpr int kLitRoot = 9;
constexpr int kLitCap = 852;  // zlib's ENOUGH_LENS for a 9-bit root: worst-case entries
constexpr int kDistRoot = 6;
constexpr int kInflateThreads = 96;
// per-thread shared memory: literal/length table (u16), distance root table (u8),
// distance code counts (u8[16]) and symbols in canonical order (u8[32])
constexpr int kDistBytes = (1 << kDistRoot) + 16 + 32;
constexpr int kThreadSmem = kLitCap * 2 + kDistBytes;
static_assert(kThreadSmem % 4 == 0, "table alignment");

// ---------------------------------------------------------------------------
// bit reader: deflate packs bits LSB first; the stream is 4-byte aligned in the payload
// with 16 readable bytes after it

struct Bits {
  const uint32_t* w;
  int64_t wi;
  uint64_t buf;
  int n;
  __device__ __forceinline__ void init(const uint32_t* words, int64_t bit) {
    w = words;
    wi = bit >> 5;
    const int s = static_cast<int>(bit & 31);
    buf = static_cast<uint64_t>(__ldg(w + wi)) >> s;
    n = 32 - s;
    ++wi;
    refill();
  }
  __device__ __forceinline__ void refill() {
    if (n <= 32) {
      buf |= static_cast<uint64_t>(__ldg(w + wi)) << n;
      n += 32;
      ++wi;
    }
  }
  __device__ __forceinline__ uint32_t peek(int k) const {
    return static_cast<uint32_t>(buf) & ((1u << k) - 1u);
  }
  __device__ __forceinline__ void drop(int k) {
    buf >>= k;
    n -= k;
  }
  __device__ __forceinline__ int64_t pos() const { return wi * 32 - n; }
};

// 64 bits starting at bit p (for the finder's header probes)
__device__ __forceinline__ uint64_t peek64(const uint32_t* w, int64_t p) {
  const int64_t i = p >> 5;
  const uint32_t s = static_cast<uint32_t>(p & 31);
  const uint32_t w0 = __ldg(w + i), w1 = __ldg(w + i + 1), w2 = __ldg(w + i + 2);
  const uint32_t lo = __funnelshift_r(w0, w1, s), hi = __funnelshift_r(w1, w2, s);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint32_t rev_bits(uint32_t code, int len) {
  return __brev(code) >> (32 - len);
}

// length / distance bases (RFC 1951 §3.2.5), computed instead of tabled: lanes index
// them with their own symbols, and a divergent constant-memory read serialises
__device__ __forceinline__ void length_base(int i, int& base, int& extra) {  // i = sym - 257
  if (i < 8) {
    base = 3 + i;
    extra = 0;
  } else if (i < 28) {
    extra = (i - 4) >> 2;
    base = ((4 + (i & 3)) << extra) + 3;
  } else {
    base = 258;
    extra = 0;
  }
}
__device__ __forceinline__ void dist_base(int d, int& base, int& extra) {
  if (d < 4) {
    base = 1 + d;
    extra = 0;
  } else {
    extra = (d - 2) >> 1;
    base = ((2 + (d & 1)) << extra) + 1;
  }
}

// Kraft check with zlib's rule (inftrees.c): over-subscribed is an error; an incomplete
// set is only allowed when the longest code has length 1 (or there are no codes at all).
__device__ bool kraft_ok(const uint8_t* lens, int n, int maxbits, int* count) {
  for (int l = 0; l <= 15; ++l) count[l] = 0;
  for (int s = 0; s < n; ++s) ++count[lens[s]];
  int maxl = 0;
  for (int l = 1; l <= 15; ++l)
    if (count[l]) maxl = l;
  if (maxl == 0) return true;
  if (maxl > maxbits) return false;
  int left = 1;
  for (int l = 1; l <= 15; ++l) {
    left <<= 1;
    left -= count[l];
    if (left < 0) return false;
  }
  return left == 0 || maxl == 1;
}

// Precode (code-length code) lookup: 7-bit index -> (len << 5) | sym, 0 = invalid.
// Returns false unless the code is complete (zlib rejects incomplete code-length codes).
__device__ bool build_precode(const uint8_t* cl, uint8_t* tab) {
  int count[16];
  for (int l = 0; l < 8; ++l) count[l] = 0;
  for (int s = 0; s < 19; ++s) ++count[cl[s]];
  int left = 1;
  for (int l = 1; l <= 7; ++l) {
    left <<= 1;
    left -= count[l];
    if (left < 0) return false;
  }
  if (left != 0) return false;
  int next[8];
  int code = 0;
  count[0] = 0;
  for (int l = 1; l <= 7; ++l) {
    code = (code + count[l - 1]) << 1;
    next[l] = code;
  }
  for (int s = 0; s < 19; ++s) {
    const int l = cl[s];
    if (!l) continue;
    const uint32_t r = rev_bits(static_cast<uint32_t>(next[l]++), l);
    for (uint32_t i = r; i < 128; i += 1u << l) tab[i] = static_cast<uint8_t>((l << 5) | s);
  }
  return true;
}

// Dynamic block header (RFC 1951 §3.2.7): code lengths into lens[0, hlit + hdist).
// Leaves the reader after the header.  tab: 128 bytes of scratch for the precode.
__device__ bool read_dynamic_lengths(Bits& br, uint8_t* lens, uint8_t* tab, int& hlit,
                                     int& hdist, int64_t limit) {
  br.refill();
  hlit = static_cast<int>(br.peek(5)) + 257;
  br.drop(5);
  hdist = static_cast<int>(br.peek(5)) + 1;
  br.drop(5);
  const int hclen = static_cast<int>(br.peek(4)) + 4;
  br.drop(4);
  if (hlit > 286 || hdist > 30) return false;
  uint8_t cl[19];
  for (int i = 0; i < 19; ++i) cl[i] = 0;
  const uint8_t kOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
  for (int i = 0; i < hclen; ++i) {
    br.refill();
    cl[kOrder[i]] = static_cast<uint8_t>(br.peek(3));
    br.drop(3);
  }
  if (!build_precode(cl, tab)) return false;
  const int total = hlit + hdist;
  int i = 0;
  while (i < total) {
    if (br.pos() > limit) return false;  // the reader stays within the stream's padding
    br.refill();
    const uint8_t e = tab[br.peek(7)];
    if (!e) return false;
    br.drop(e >> 5);
    const int sym = e & 31;
    if (sym < 16) {
      lens[i++] = static_cast<uint8_t>(sym);
      continue;
    }
    int rep;
    uint8_t val = 0;
    if (sym == 16) {
      if (i == 0) return false;
      val = lens[i - 1];
      rep = 3 + static_cast<int>(br.peek(2));
      br.drop(2);
    } else if (sym == 17) {
      rep = 3 + static_cast<int>(br.peek(3));
      br.drop(3);
    } else {
      rep = 11 + static_cast<int>(br.peek(7));
      br.drop(7);
    }
    if (i + rep > total) return false;
    while (rep--) lens[i++] = val;
  }
  return lens[256] != 0;  // a block without end-of-block cannot be decoded
}

// Literal/length table, 9-bit root + subtables (u16 entries):
//   direct   bit 15 = 0, bits 14..11 total code length, bits 8..0 symbol
//   pointer  bit 15 = 1, bits 14..12 subtable index bits, bits 11..0 subtable offset
//   invalid  0xFFFF
__device__ bool build_lit(const uint8_t* lens, int n, uint16_t* tbl) {
  int count[16];
  if (!kraft_ok(lens, n, 15, count)) return false;
  int next[16];
  int code = 0;
  count[0] = 0;
  int left = 1;
  for (int l = 1; l <= 15; ++l) {
    code = (code + count[l - 1]) << 1;
    next[l] = code;
    left = (left << 1) - count[l];
  }
  if (left != 0)  // incomplete (allowed for a lone 1-bit code): missing codes are invalid
    for (int i = 0; i < (1 << kLitRoot); ++i) tbl[i] = 0xFFFF;
  int nlong = 0;
  for (int l = kLitRoot + 1; l <= 15; ++l) nlong += count[l];
  int snext[16];
  for (int l = 0; l < 16; ++l) snext[l] = next[l];
  for (int s = 0; s < n; ++s) {
    const int l = lens[s];
    if (!l || l > kLitRoot) continue;
    const uint32_t r = rev_bits(static_cast<uint32_t>(snext[l]++), l);
    const uint16_t e = static_cast<uint16_t>((l << 11) | s);
    for (uint32_t i = r; i < (1u << kLitRoot); i += 1u << l) tbl[i] = e;
  }
  if (!nlong) return true;
  // long codes in canonical order (length, then symbol) have non-decreasing 9-bit
  // prefixes, so codes sharing a prefix are consecutive and the last is the longest
  int off = 1 << kLitRoot;
  int cur = -1, cur_max = 0;
  auto close_group = [&](int prefix, int maxl) -> bool {
    const int bits = maxl - kLitRoot;
    if (off + (1 << bits) > kLitCap) return false;
    tbl[rev_bits(static_cast<uint32_t>(prefix), kLitRoot)] =
        static_cast<uint16_t>(0x8000 | (bits << 12) | off);
    if (left != 0)
      for (int i = 0; i < (1 << bits); ++i) tbl[off + i] = 0xFFFF;
    off += 1 << bits;
    return true;
  };
  for (int l = kLitRoot + 1; l <= 15; ++l) {
    if (!count[l]) continue;
    int c = next[l];
    for (int s = 0; s < n; ++s) {
      if (lens[s] != l) continue;
      const int prefix = c >> (l - kLitRoot);
      if (prefix != cur) {
        if (cur >= 0 && !close_group(cur, cur_max)) return false;
        cur = prefix;
      }
      cur_max = l;
      ++c;
    }
  }
  if (!close_group(cur, cur_max)) return false;
  for (int l = kLitRoot + 1; l <= 15; ++l) {
    if (!count[l]) continue;
    for (int s = 0; s < n; ++s) {
      if (lens[s] != l) continue;
      const int c = snext[l]++;
      const int prefix = c >> (l - kLitRoot);
      const uint16_t p = tbl[rev_bits(static_cast<uint32_t>(prefix), kLitRoot)];
      const int bits = (p >> 12) & 7, base = p & 0xFFF;
      const int rest = l - kLitRoot;
      const uint32_t r = rev_bits(static_cast<uint32_t>(c) & ((1u << rest) - 1u), rest);
      const uint16_t e = static_cast<uint16_t>((l << 11) | s);
      for (uint32_t i = r; i < (1u << bits); i += 1u << rest) tbl[base + i] = e;
    }
  }
  return true;
}

// Distance code: 6-bit root of (len << 5) | sym bytes (0xFF: longer code or invalid),
// plus counts per length and the symbols in canonical order for the longer codes.
__device__ bool build_dist(const uint8_t* lens, int n, uint8_t* dt) {
  int count[16];
  if (!kraft_ok(lens, n, 15, count)) return false;
  uint8_t* root = dt;
  uint8_t* dcount = dt + (1 << kDistRoot);
  uint8_t* dsym = dcount + 16;
  for (int i = 0; i < (1 << kDistRoot); ++i) root[i] = 0xFF;
  int next[16], idx[16];
  int code = 0, k = 0;
  count[0] = 0;
  for (int l = 1; l <= 15; ++l) {
    code = (code + count[l - 1]) << 1;
    next[l] = code;
    idx[l] = k;
    k += count[l];
    dcount[l] = static_cast<uint8_t>(count[l]);
  }
  dcount[0] = 0;
  for (int s = 0; s < n; ++s) {
    const int l = lens[s];
    if (!l) continue;
    dsym[idx[l]++] = static_cast<uint8_t>(s);
    const int c = next[l]++;
    if (l <= kDistRoot) {
      const uint32_t r = rev_bits(static_cast<uint32_t>(c), l);
      for (uint32_t i = r; i < (1u << kDistRoot); i += 1u << l)
        root[i] = static_cast<uint8_t>((l << 5) | s);
    }
  }
  return true;
}

// distance symbol; -1: invalid code
__device__ __forceinline__ int decode_dist(Bits& br, const uint8_t* dt) {
  const uint8_t e = dt[br.peek(kDistRoot)];
  if (e != 0xFF) {
    br.drop(e >> 5);
    return e & 31;
  }
  const uint8_t* dcount = dt + (1 << kDistRoot);
  const uint8_t* dsym = dcount + 16;
  const uint32_t bits = br.peek(15);
  int code = 0, first = 0, index = 0;
  for (int l = 1; l <= 15; ++l) {
    code |= static_cast<int>((bits >> (l - 1)) & 1u);
    const int cnt = dcount[l];
    if (code - first < cnt) {
      br.drop(l);
      return dsym[index + code - first];
    }
    index += cnt;
    first = (first + cnt) << 1;
    code <<= 1;
  }
  return -1;
}

// Quick probe of a dynamic header at bit p: field ranges and a complete code-length code.
__device__ __forceinline__ bool dynamic_probe(const uint32_t* w, int64_t p) {
  const uint64_t x = peek64(w, p);
  if (((x >> 1) & 3) != 2) return false;
  if (((x >> 3) & 31) > 29 || ((x >> 8) & 31) > 29) return false;
  const int hclen = static_cast<int>((x >> 13) & 15) + 4;
  const uint64_t y = peek64(w, p + 17);
  int sum = 0;
  for (int i = 0; i < hclen; ++i) {
    const int l = static_cast<int>((y >> (3 * i)) & 7);
    if (l) sum += 128 >> l;
  }
  return sum == 128;
}

__device__ bool dynamic_full(const uint32_t* w, int64_t p, int64_t in_bits) {
  Bits br;
  br.init(w, p + 3);
  uint8_t lens[320];
  uint8_t tab[128];
  int hlit, hdist;
  if (!read_dynamic_lengths(br, lens, tab, hlit, hdist, in_bits)) return false;
  if (br.pos() > in_bits) return false;
  int count[16];
  return kraft_ok(lens, hlit, 15, count) && kraft_ok(lens + hlit, hdist, 15, count);
}

// stored header at p (BTYPE 00): zero padding to the byte boundary, LEN == ~NLEN;
// *next = bit of the following block
__device__ __forceinline__ bool stored_probe(const uint32_t* w, int64_t p, int64_t in_bits,
                                             int64_t* next) {
  const uint64_t x = peek64(w, p);
  if (((x >> 1) & 3) != 0) return false;
  const int64_t q = (p + 3 + 7) & ~int64_t(7);
  const int pad = static_cast<int>(q - (p + 3));
  if (pad && ((x >> 3) & ((1ull << pad) - 1)) != 0) return false;
  const uint64_t v = peek64(w, q);
  const uint32_t len = static_cast<uint32_t>(v & 0xFFFF), nlen = static_cast<uint32_t>((v >> 16) & 0xFFFF);
  if ((len ^ nlen) != 0xFFFF) return false;
  *next = q + 32 + 8 * static_cast<int64_t>(len);
  return *next <= in_bits;
}

// 0: no header at p; 1: dynamic header; 2: stored header (canonical start: its LEN byte)
__device__ int header_candidate(const uint32_t* w, int64_t p, int64_t in_bits) {
  if (p + 3 > in_bits) return 0;
  if (dynamic_probe(w, p)) return dynamic_full(w, p, in_bits) ? 1 : 0;
  int64_t nxt;
  if (!stored_probe(w, p, in_bits, &nxt)) return 0;
  if (nxt == in_bits - 32) return 2;  // the last block: the Adler-32 trailer follows
  // a stored block must be followed by another plausible header
  if (nxt + 3 > in_bits) return 0;
  if (dynamic_probe(w, nxt)) return dynamic_full(w, nxt, in_bits) ? 2 : 0;
  int64_t nxt2;
  return stored_probe(w, nxt, in_bits, &nxt2) ? 2 : 0;
}

__device__ __forceinline__ int unit_image(const PDesc* __restrict__ desc, int n, int u) {
  int lo = 0, hi = n;  // largest k with unit_base <= u
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (desc[mid].unit_base <= u) lo = mid; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// find: one warp per unit

__global__ void k_png_find(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc,
                           int n, PUnit* __restrict__ units, int U) {
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= U) return;
  const int k = unit_image(desc, n, u);
  const PDesc& d = desc[k];
  const int local = u - d.unit_base;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(payload + d.in_off);
  int64_t start = -1;
  int stored = 0;
  if (local == 0) {
    start = 16;  // after the zlib header
  } else {
    const int64_t lo = static_cast<int64_t>(local) * kUnitBits;
    const int64_t hi = min(lo + kUnitBits, d.in_bits);
    for (int64_t p0 = lo; p0 < hi; p0 += 32) {
      const int64_t p = p0 + lane;
      const int kind = p < hi ? header_candidate(w, p, d.in_bits) : 0;
      const unsigned m = __ballot_sync(0xffffffffu, kind != 0);
      if (m) {
        const int l = __ffs(m) - 1;
        start = p0 + l;
        stored = (__ballot_sync(0xffffffffu, kind == 2) >> l) & 1;
        if (stored) start = (start + 3 + 7) & ~int64_t(7);
        break;
      }
    }
  }
  if (lane == 0) {
    PUnit& o = units[u];
    o.start = start;
    o.end = -1;
    o.out_len = 0;
    o.out_off = 0;
    o.ntok = 0;
    o.status = kUnitOk;
    o.final_ = 0;
    o.dirty = start >= 0;
    o.stored = stored;
  }
}

// ---------------------------------------------------------------------------
// inflate: one thread per unit

__global__ void __launch_bounds__(kInflateThreads)
    k_png_inflate(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc, int n,
                  PUnit* __restrict__ units, int U, uint32_t* __restrict__ toks,
                  const int32_t* __restrict__ img_status) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= U) return;
  PUnit& me = units[u];
  if (!me.dirty) return;
  const int k = unit_image(desc, n, u);
  const PDesc& d = desc[k];
  if (img_status[k] != kImgOk) return;
  const int64_t start = me.start;
  // stop: the next unit's start (the first block boundary at or past it ends this unit)
  int64_t stop = -1;
  const int ulast = d.unit_base + d.n_units;
  for (int j = u + 1; j < ulast; ++j) {
    const int64_t s = units[j].start;
    if (s >= 0) {
      stop = s;
      break;
    }
  }
  const bool last = stop < 0;
  const int64_t in_bits = d.in_bits;
  uint16_t* lt = reinterpret_cast<uint16_t*>(smem + threadIdx.x * kThreadSmem);
  uint8_t* dt = smem + threadIdx.x * kThreadSmem + kLitCap * 2;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(payload + d.in_off);
  uint32_t* tk = toks + d.tok_off + (start >> 1);
  const int64_t cap = last ? d.in_bits / 2 + 256 - (start >> 1) : (stop >> 1) - (start >> 1);
  int64_t ntok = 0, out = 0;
  int status = kUnitOk, fin = 0;
  uint32_t pack = 0;
  int pc = 0;
  auto emit = [&](uint32_t t) -> bool {
    if (ntok >= cap) return false;
    tk[ntok++] = t;
    return true;
  };
  Bits br;
  br.init(w, start);
  bool stored_start = me.stored != 0;  // the first block's LEN field is at `start`
  int64_t end = start;
  while (true) {
    const int64_t pos = br.pos();
    uint32_t hdr = 0;
    int btype = 0;
    if (stored_start) {
      end = pos;
    } else {
      if (pos + 3 > in_bits) {
        status = kUnitOverrun;
        break;
      }
      br.refill();
      hdr = br.peek(3);
      btype = static_cast<int>(hdr >> 1);
      // canonical block position: a stored block's is its LEN byte
      end = btype == 0 ? (pos + 3 + 7) & ~int64_t(7) : pos;
      if (!last && end >= stop) break;
      br.drop(3);
    }
    if (btype == 0) {  // stored
      if (!stored_start) br.drop(br.n & 7);  // to the byte boundary (pos % 8 = -n % 8)
      stored_start = false;
      const int64_t q = br.pos();
      br.refill();
      const uint32_t v32 = static_cast<uint32_t>(br.buf);  // n >= 33 after the refill
      const uint32_t len = v32 & 0xFFFF, nlen = v32 >> 16;
      if ((len ^ nlen) != 0xFFFF) {
        status = kUnitBadStored;
        break;
      }
      const int64_t data_bit = q + 32;
      const int64_t next = data_bit + 8 * static_cast<int64_t>(len);
      if (next > in_bits) {
        status = kUnitOverrun;
        break;
      }
      if (pc) {
        if (!emit((static_cast<uint32_t>(pc) << 24) | pack)) { status = kUnitTokens; break; }
        pc = 0;
        pack = 0;
      }
      if (len) {
        if (!emit(kTokStored | static_cast<uint32_t>(data_bit >> 3))) { status = kUnitTokens; break; }
        out += len;
      }
      br.init(w, next);
      // only the final block is followed directly by the Adler-32 trailer (the BFINAL bit
      // of a stored start is not read: a canonical start skips its header)
      if (next == in_bits - 32) hdr |= 1;
    } else if (btype == 1 || btype == 2) {
      if (btype == 1) {  // fixed codes (RFC 1951 §3.2.6)
        uint8_t lens[320];
        for (int i = 0; i < 144; ++i) lens[i] = 8;
        for (int i = 144; i < 256; ++i) lens[i] = 9;
        for (int i = 256; i < 280; ++i) lens[i] = 7;
        for (int i = 280; i < 288; ++i) lens[i] = 8;
        for (int i = 0; i < 32; ++i) lens[288 + i] = 5;
        if (!build_lit(lens, 288, lt) || !build_dist(lens + 288, 32, dt)) {
          status = kUnitBadCode;
          break;
        }
      } else {
        uint8_t lens[320];
        int hlit, hdist;
        // the precode table lives in the (not yet built) literal table's space
        if (!read_dynamic_lengths(br, lens, reinterpret_cast<uint8_t*>(lt), hlit, hdist, in_bits) ||
            !build_lit(lens, hlit, lt) || !build_dist(lens + hlit, hdist, dt)) {
          status = kUnitBadCode;
          break;
        }
      }
      bool ok = true;
      while (true) {
        if (br.pos() > in_bits) { ok = false; status = kUnitOverrun; break; }
        br.refill();
        uint32_t e = lt[br.peek(kLitRoot)];
        if (e & 0x8000u) {
          const int sub = (e >> 12) & 7;
          if (sub == 7) { ok = false; break; }
          e = lt[(e & 0xFFFu) + (br.peek(kLitRoot + sub) >> kLitRoot)];
          if (e & 0x8000u) { ok = false; break; }
        }
        br.drop((e >> 11) & 15);
        const int s = static_cast<int>(e & 511u);
        if (s < 256) {
          pack |= static_cast<uint32_t>(s) << (8 * pc);
          if (++pc == 3) {
            if (ntok >= cap) { ok = false; status = kUnitTokens; break; }
            tk[ntok++] = (3u << 24) | pack;
            pc = 0;
            pack = 0;
          }
          ++out;
          continue;
        }
        if (s == 256) break;
        if (s > 285) { ok = false; break; }
        int base, extra;
        length_base(s - 257, base, extra);
        const int len = base + static_cast<int>(br.peek(extra));
        br.drop(extra);
        br.refill();
        const int ds = decode_dist(br, dt);
        if (ds < 0 || ds > 29) { ok = false; break; }
        int dbase, dextra;
        dist_base(ds, dbase, dextra);
        const int dist = dbase + static_cast<int>(br.peek(dextra));
        br.drop(dextra);
        if (pc) {
          if (ntok >= cap) { ok = false; status = kUnitTokens; break; }
          tk[ntok++] = (static_cast<uint32_t>(pc) << 24) | pack;
          pc = 0;
          pack = 0;
        }
        if (ntok >= cap) { ok = false; status = kUnitTokens; break; }
        tk[ntok++] = kTokMatch | (static_cast<uint32_t>(len - 3) << 16) | static_cast<uint32_t>(dist - 1);
        out += len;
      }
      if (!ok) {
        if (status == kUnitOk) status = kUnitBadCode;
        break;
      }
      if (br.pos() > in_bits) {
        status = kUnitOverrun;
        break;
      }
    } else {
      status = kUnitBadCode;
      break;
    }
    if (hdr & 1) {
      fin = 1;
      break;
    }
  }
  if (status == kUnitOk && pc) {
    if (ntok < cap) tk[ntok++] = (static_cast<uint32_t>(pc) << 24) | pack;
    else status = kUnitTokens;
  }
  // a token overflow is judged by how far the decode got (past the next start or not)
  me.end = (last || status == kUnitTokens) ? br.pos() : end;
  me.ntok = static_cast<int32_t>(ntok);
  me.out_len = out;
  me.status = status;
  me.final_ = fin;
  me.dirty = 0;
}

// ---------------------------------------------------------------------------
// chain: one warp per image (lane 0 walks; the units are few)

__global__ void k_png_chain(const PDesc* __restrict__ desc, int n, PUnit* __restrict__ units,
                            int32_t* __restrict__ img_status, int last_round) {
  const int k = blockIdx.x;
  if (k >= n || threadIdx.x != 0) return;
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const int u0 = d.unit_base, u1 = d.unit_base + d.n_units;
  int64_t off = 0;
  int u = u0;  // unit 0 always starts at a real block
  // the start found for unit v is not a block start: the decode of u passed it
  auto drop_successor = [&](PUnit& cu, int v) {
    units[v].start = -1;
    units[v].dirty = 0;
    cu.dirty = 1;  // decode u again, up to the next start
    if (last_round) img_status[k] = kImgChain;
  };
  while (true) {
    PUnit& cu = units[u];
    if (cu.dirty) {  // re-decoded next round
      if (last_round) img_status[k] = kImgChain;
      return;
    }
    int v = u + 1;
    while (v < u1 && units[v].start < 0) ++v;
    const bool has_v = v < u1;
    if (cu.status == kUnitTokens && has_v && cu.end > units[v].start) {
      drop_successor(cu, v);
      return;
    }
    if (cu.status != kUnitOk) {
      img_status[k] = kImgInflate;
      return;
    }
    if (!has_v) {
      if (!cu.final_) {
        img_status[k] = kImgNotFinal;
        return;
      }
      cu.out_off = off;
      off += cu.out_len;
      units[u0].final_end = cu.end;
      break;
    }
    if (cu.final_) {  // a header was found past the end of the final block
      units[v].start = -1;
      units[v].dirty = 0;
      continue;  // look for u's next successor
    }
    if (cu.end == units[v].start) {
      cu.out_off = off;
      off += cu.out_len;
      u = v;
      continue;
    }
    drop_successor(cu, v);
    return;
  }
  if (off != d.raw_len) img_status[k] = kImgLength;
}

// ---------------------------------------------------------------------------
// expand: one warp per unit, tokens -> u16 bytes (>= 256: window markers)

__global__ void k_png_expand(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc,
                             int n, const PUnit* __restrict__ units, int U,
                             const uint32_t* __restrict__ toks, uint16_t* __restrict__ T,
                             int32_t* __restrict__ img_status) {
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= U) return;
  const int k = unit_image(desc, n, u);
  const PDesc& d = desc[k];
  if (img_status[k] != kImgOk) return;
  const PUnit cu = units[u];
  if (cu.start < 0 || cu.out_len == 0) return;
  const uint32_t* tk = toks + d.tok_off + (cu.start >> 1);
  const uint8_t* zs = payload + d.in_off;
  uint16_t* img = T + d.raw_off;
  const int64_t ws = cu.out_off;          // unit start (image-relative)
  const int64_t wbase = ws - kWindow;     // marker 256 + i refers to image byte wbase + i
  int64_t cur = ws;
  bool bad = false;
  for (int b = 0; b < cu.ntok; b += 32) {
    const int i = b + lane;
    const uint32_t t = i < cu.ntok ? tk[i] : 0u;
    const uint32_t type = t >> 30;
    int len = 0;
    if (i < cu.ntok) {
      if (type == 0) {
        len = static_cast<int>((t >> 24) & 3);
      } else if (type == 1) {
        len = static_cast<int>((t >> 16) & 255) + 3;
      } else {
        const uint32_t at = t & 0x3FFFFFFFu;
        len = zs[at - 4] | (zs[at - 3] << 8);
      }
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int64_t at = cur + incl - len;
    if (i < cu.ntok && type == 0)
      for (int j = 0; j < len; ++j) img[at + j] = static_cast<uint16_t>((t >> (8 * j)) & 255);
    __syncwarp();
    unsigned m = __ballot_sync(0xffffffffu, i < cu.ntok && type != 0);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t tt = __shfl_sync(0xffffffffu, t, l);
      const int64_t dst = __shfl_sync(0xffffffffu, at, l);
      const int ln = __shfl_sync(0xffffffffu, len, l);
      if ((tt >> 30) == 2) {
        const uint8_t* src = zs + (tt & 0x3FFFFFFFu);
        for (int j = lane; j < ln; j += 32) img[dst + j] = src[j];
      } else {
        const int dist = static_cast<int>(tt & 0xFFFFu) + 1;
        for (int j = lane; j < ln; j += 32) {
          const int64_t s = dst - dist + (dist >= ln ? j : j % dist);
          uint16_t v;
          if (s >= ws) {
            v = img[s];
          } else if (s >= 0 && s >= wbase) {
            v = static_cast<uint16_t>(256 + (s - wbase));
          } else {
            v = 0;
            bad = true;
          }
          img[dst + j] = v;
        }
      }
      __syncwarp();
    }
    cur += total;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(img_status + k, kImgDistance);
}

// ---------------------------------------------------------------------------
// window: one CTA per image, units in order; each unit's last 32 KB resolved

__global__ void k_png_window(const PDesc* __restrict__ desc, int n, const PUnit* __restrict__ units,
                             const uint16_t* __restrict__ T, uint8_t* __restrict__ R,
                             const int32_t* __restrict__ img_status) {
  const int k = blockIdx.x;
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const uint16_t* t = T + d.raw_off;
  uint8_t* r = R + d.raw_off;
  for (int u = d.unit_base; u < d.unit_base + d.n_units; ++u) {
    const PUnit cu = units[u];
    if (cu.start < 0 || cu.out_len == 0) continue;
    const int64_t os = cu.out_off, oe = os + cu.out_len;
    const int64_t lo = max(os, oe - kWindow);
    const int64_t wb = os - kWindow;
    for (int64_t p = lo + threadIdx.x; p < oe; p += blockDim.x) {
      const uint32_t v = t[p];
      r[p] = v < 256 ? static_cast<uint8_t>(v) : r[wb + (v - 256)];
    }
    __syncthreads();
  }
}

// final: one CTA per unit, the bytes before the unit's last 32 KB
__global__ void k_png_final(const PDesc* __restrict__ desc, int n, const PUnit* __restrict__ units,
                            int U, const uint16_t* __restrict__ T, uint8_t* __restrict__ R,
                            const int32_t* __restrict__ img_status) {
  const int u = blockIdx.x;
  if (u >= U) return;
  const int k = unit_image(desc, n, u);
  const PDesc& d = desc[k];
  if (img_status[k] != kImgOk) return;
  const PUnit cu = units[u];
  if (cu.start < 0 || cu.out_len <= kWindow) return;
  const uint16_t* t = T + d.raw_off;
  uint8_t* r = R + d.raw_off;
  const int64_t os = cu.out_off, hi = os + cu.out_len - kWindow, wb = os - kWindow;
  for (int64_t p = os + threadIdx.x; p < hi; p += blockDim.x) {
    const uint32_t v = t[p];
    r[p] = v < 256 ? static_cast<uint8_t>(v) : r[wb + (v - 256)];
  }
}

// ---------------------------------------------------------------------------
// Adler-32 (RFC 1950 §8) of the inflated bytes, checked when the stream holds the four
// trailer bytes after the final block.  Pillow's zlib verifies the trailer whenever it
// is in the data it was fed (a wrong one raises "broken data stream"), and says nothing
// when the stream ends before it (tests/test_gpu_png.py, bad payloads).  Thread t sums
// its contiguous segment: s1 = sum d_i, s2 = sum (n - i) d_i; b = n + sum s2, a = 1 + sum s1.

constexpr uint32_t kAdlerMod = 65521;
constexpr int kAdlerThreads = 1024;

__global__ void __launch_bounds__(kAdlerThreads)
    k_png_adler(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc, int n,
                const PUnit* __restrict__ units, const uint8_t* __restrict__ R,
                int32_t* __restrict__ img_status) {
  __shared__ uint64_t red[2][kAdlerThreads / 32];
  const int k = blockIdx.x;
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const int64_t fin = units[d.unit_base].final_end;
  const int64_t at = (fin + 7) >> 3;  // trailer bytes, big-endian
  if (at + 4 > (d.in_bits >> 3)) return;
  const int64_t len = d.raw_len;
  const int64_t seg = (len + blockDim.x - 1) / blockDim.x;
  const int64_t s0 = min(len, seg * static_cast<int64_t>(threadIdx.x)), s1e = min(len, s0 + seg);
  const uint8_t* r = R + d.raw_off;
  uint64_t a = 0, b = 0;  // a: sum d_i; b: sum (s1e - i) d_i, reduced every 4096 bytes
  int64_t i = s0;
  while (i < s1e) {
    const int64_t e = min(s1e, i + 4096);
    uint64_t la = 0, lb = 0;
    for (int64_t j = i; j < e; ++j) {
      const uint32_t v = r[j];
      la += v;
      lb += static_cast<uint64_t>(s1e - j) * v;
    }
    a = (a + la) % kAdlerMod;
    b = (b + lb) % kAdlerMod;
    i = e;
  }
  // this segment's weight in the whole: (n - i) = (s1e - i) + (n - s1e)
  b = (b + (static_cast<uint64_t>(len - s1e) % kAdlerMod) * a) % kAdlerMod;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][warp] = a;
    red[1][warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t A = 1, B = static_cast<uint64_t>(len) % kAdlerMod;
    for (int w = 0; w < (blockDim.x >> 5); ++w) {
      A += red[0][w];
      B += red[1][w];
    }
    A %= kAdlerMod;
    B %= kAdlerMod;
    const uint8_t* z = payload + d.in_off + at;
    const uint32_t want = (uint32_t(z[0]) << 24) | (uint32_t(z[1]) << 16) | (uint32_t(z[2]) << 8) | z[3];
    if (((B << 16) | A) != want) atomicOr(img_status + k, kImgAdler);
  }
}

// ---------------------------------------------------------------------------
// unfilter (PNG §9.2) + L/P -> RGB: one CTA per image, thread = scanline

__device__ __forceinline__ uint32_t paeth(uint32_t a, uint32_t b, uint32_t c) {
  const int p = static_cast<int>(a) + static_cast<int>(b) - static_cast<int>(c);
  const int pa = abs(p - static_cast<int>(a)), pb = abs(p - static_cast<int>(b)),
            pc = abs(p - static_cast<int>(c));
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

constexpr int kUnfilterThreads = 1024;

__global__ void __launch_bounds__(kUnfilterThreads)
    k_png_unfilter(const PDesc* __restrict__ desc, int n, uint8_t* __restrict__ R,
                   uint8_t* __restrict__ out, int32_t* __restrict__ img_status) {
  __shared__ uint32_t xch[2][kUnfilterThreads];
  __shared__ uint8_t pal[768];
  const int k = blockIdx.x;
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const int tid = threadIdx.x;
  const int W = d.width, H = d.height, bpp = d.bpp;
  const bool is_p = d.ctype == 3;
  for (int i = tid; i < 768; i += blockDim.x) pal[i] = d.pal[i];
  const int64_t rowbytes = static_cast<int64_t>(W) * bpp, stride = rowbytes + 1;
  const int nch = static_cast<int>((rowbytes + 3) >> 2);
  uint8_t* raw = R + d.raw_off;
  uint8_t* o = out + d.out_off;
  const int G = blockDim.x;
  bool bad_filter = false, bad_pal = false;
  __syncthreads();
  for (int g0 = 0; g0 < H; g0 += G) {
    const int rows = min(G, H - g0);
    const int y = g0 + tid;
    const bool has_row = tid < rows;
    uint8_t* row = raw + static_cast<int64_t>(y) * stride;
    const uint32_t ft = has_row ? row[0] : 0u;
    if (ft > 4) bad_filter = true;
    const uint8_t* prior = y > 0 ? row - stride : nullptr;  // recon (written in place below)
    uint32_t up_prev = 0, cur_prev = 0;
    const int steps = nch + rows - 1;
    for (int t = 0; t < steps; ++t) {
      const int i = t - tid;
      if (has_row && i >= 0 && i < nch) {
        uint32_t up = 0;
        if (tid == 0) {
          if (prior)
            for (int j = 0; j < 4; ++j) {
              const int64_t x = 4 * static_cast<int64_t>(i) + j;
              if (x < rowbytes) up |= static_cast<uint32_t>(prior[1 + x]) << (8 * j);
            }
        } else {
          up = xch[(t - 1) & 1][tid - 1];
        }
        uint32_t rec = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t x = 4 * static_cast<int64_t>(i) + j;
          if (x >= rowbytes) break;
          const uint32_t f = row[1 + x];
          // a = recon[x - bpp], b = up[x], c = up[x - bpp] (0 before the row start)
          uint32_t a = 0, c = 0;
          if (x >= bpp) {
            const int s = j - bpp;  // position of x - bpp relative to this chunk
            a = s >= 0 ? (rec >> (8 * s)) & 255u : (cur_prev >> (8 * (s + 4))) & 255u;
            c = s >= 0 ? (up >> (8 * s)) & 255u : (up_prev >> (8 * (s + 4))) & 255u;
          }
          const uint32_t b = (up >> (8 * j)) & 255u;
          uint32_t pred;
          switch (ft) {
            case 1: pred = a; break;
            case 2: pred = b; break;
            case 3: pred = (a + b) >> 1; break;
            case 4: pred = paeth(a, b, c); break;
            default: pred = 0;
          }
          const uint32_t v = (f + pred) & 255u;
          rec |= v << (8 * j);
          if (bpp == 3) {
            o[static_cast<int64_t>(y) * rowbytes + x] = static_cast<uint8_t>(v);
          } else {
            uint8_t* px = o + (static_cast<int64_t>(y) * W + x) * 3;
            if (is_p) {
              if (static_cast<int>(v) >= d.pal_n) bad_pal = true;
              px[0] = pal[3 * v];
              px[1] = pal[3 * v + 1];
              px[2] = pal[3 * v + 2];
            } else {
              px[0] = px[1] = px[2] = static_cast<uint8_t>(v);
            }
          }
        }
        if (tid == rows - 1)  // the next group's first row reads this row's recon
          for (int j = 0; j < 4; ++j) {
            const int64_t x = 4 * static_cast<int64_t>(i) + j;
            if (x < rowbytes) row[1 + x] = static_cast<uint8_t>(rec >> (8 * j));
          }
        xch[t & 1][tid] = rec;
        up_prev = up;
        cur_prev = rec;
      }
      __syncthreads();
    }
  }
  if (bad_filter) atomicOr(img_status + k, kImgFilter);
  if (bad_pal) atomicOr(img_status + k, kImgPalette);
}

}  // namespace

extern "C" TP_API int tp_png_decode(const uint8_t* d_payload, const void* d_desc, int32_t n,
                                    const int64_t* totals, void* d_work, int64_t work_bytes,
                                    uint8_t* d_out, int32_t* d_status, void* stream) {
  if (n < 0 || (n > 0 && (!d_payload || !d_desc || !totals || !d_work || !d_out || !d_status)))
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_png_decode: null argument");
  if (n == 0) return TP_OK;
  if (work_bytes < totals[7])
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_png_decode: workspace %lld < %lld bytes",
                         (long long)work_bytes, (long long)totals[7]);
  cudaStream_t s = tp::as_stream(stream);
  const PDesc* desc = static_cast<const PDesc*>(d_desc);
  uint8_t* work = static_cast<uint8_t*>(d_work);
  const int U = static_cast<int>(totals[0]);
  PUnit* units = reinterpret_cast<PUnit*>(work + totals[3]);
  uint32_t* toks = reinterpret_cast<uint32_t*>(work + totals[4]);
  uint16_t* T = reinterpret_cast<uint16_t*>(work + totals[5]);
  uint8_t* R = work + totals[6];
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_png_inflate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kInflateThreads * kThreadSmem);
    attr_set = true;
  }
  cudaMemsetAsync(d_status, 0, sizeof(int32_t) * n, s);
  if (U > 0) {
    k_png_find<<<(U + 7) / 8, 256, 0, s>>>(d_payload, desc, n, units, U);
    for (int r = 0; r < kRounds; ++r) {
      k_png_inflate<<<(U + kInflateThreads - 1) / kInflateThreads, kInflateThreads,
                      kInflateThreads * kThreadSmem, s>>>(d_payload, desc, n, units, U, toks,
                                                           d_status);
      k_png_chain<<<n, 32, 0, s>>>(desc, n, units, d_status, r == kRounds - 1);
    }
    k_png_expand<<<(U + 7) / 8, 256, 0, s>>>(d_payload, desc, n, units, U, toks, T, d_status);
    k_png_window<<<n, 1024, 0, s>>>(desc, n, units, T, R, d_status);
    k_png_final<<<U, 256, 0, s>>>(desc, n, units, U, T, R, d_status);
    k_png_adler<<<n, kAdlerThreads, 0, s>>>(d_payload, desc, n, units, R, d_status);
    k_png_unfilter<<<n, kUnfilterThreads, 0, s>>>(desc, n, R, d_out, d_status);
  }
  return tp::check_launch("tp_png_decode");
}
