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

#include <cstdlib>

#include "png_common.cuh"
#include "tp_common.cuh"

namespace {

using namespace tp::png;

// 10-bit root: a photo-like PNG's rarer literals have 10-12 bit codes, and with a 9-bit
// root a third of the warp's decode steps took the subtable branch for some lane
constexpr int kLitRoot = 10;
constexpr int kLitCap = 1332;  // zlib's `enough 286 10 15`: worst-case entries, root 10
constexpr int kDistRoot = 6;
// distance table: root of 2^kDistRoot bytes, code counts (u8[16]) and the symbols in
// canonical order (u8[32])
constexpr int kDistBytes = (1 << kDistRoot) + 16 + 32;

// ---------------------------------------------------------------------------
// bit reader: deflate packs bits LSB first; the stream is 16-byte aligned in the payload
// with 64 readable bytes after it

struct Bits {
  // 64-bit bit buffer refilled one 32-bit word at a time through the read-only path
  // (the words of a lane's subsequence are L1 hits after the first)
  const uint32_t* w;
  int64_t wi;  // next word to load
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
__device__ bool build_lit(const uint8_t* lens, int n, uint16_t* tbl, uint16_t* sorted) {
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
  // the long codes in canonical order (length, then symbol), by one counting-sort pass
  // instead of a scan of every symbol per length
  int loff[16];
  for (int l = 0, o = 0; l <= 15; ++l) {
    loff[l] = o;
    if (l > kLitRoot) o += count[l];
  }
  for (int s = 0; s < n; ++s) {
    const int l = lens[s];
    if (l > kLitRoot) sorted[loff[l]++] = static_cast<uint16_t>(s);
  }
  // their 10-bit prefixes are non-decreasing, so codes sharing a prefix are consecutive
  // and the last of a group is its longest
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
  {
    int l = kLitRoot + 1, c = next[l], left_in_l = count[l];
    for (int k = 0; k < nlong; ++k) {
      while (left_in_l == 0) {
        ++l;
        c = next[l];
        left_in_l = count[l];
      }
      const int prefix = c >> (l - kLitRoot);
      if (prefix != cur) {
        if (cur >= 0 && !close_group(cur, cur_max)) return false;
        cur = prefix;
      }
      cur_max = l;
      ++c;
      --left_in_l;
    }
  }
  if (!close_group(cur, cur_max)) return false;
  {
    int l = kLitRoot + 1, left_in_l = count[l];
    for (int k = 0; k < nlong; ++k) {
      while (left_in_l == 0) {
        ++l;
        left_in_l = count[l];
      }
      --left_in_l;
      const int s = sorted[k];
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

// Full check of a dynamic header at p (after the quick probe): decode the code lengths
// with the code-length code and require complete literal/length and distance codes
// (zlib always writes complete codes) with an end-of-block code.  Kraft sums run while
// decoding, so random bits fail within a few lengths; no length array is kept.
// tab: 128 bytes of scratch (shared memory) for the code-length code.
__device__ bool dynamic_full(const uint32_t* w, int64_t p, int64_t in_bits, uint8_t* tab) {
  Bits br;
  br.init(w, p + 3);
  const int hlit = static_cast<int>(br.peek(5)) + 257;
  br.drop(5);
  const int hdist = static_cast<int>(br.peek(5)) + 1;
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
  int lit_left = 1 << 15, dist_left = 1 << 15;
  int prev = 0, i = 0;
  bool eob = false;
  auto put = [&](int l, int rep) -> bool {
    for (int r = 0; r < rep; ++r, ++i) {
      if (!l) continue;
      if (i < hlit) {
        lit_left -= (1 << 15) >> l;
        if (lit_left < 0) return false;
        if (i == 256) eob = true;
      } else {
        dist_left -= (1 << 15) >> l;
        if (dist_left < 0) return false;
      }
    }
    return true;
  };
  while (i < total) {
    if (br.pos() > in_bits) return false;
    br.refill();
    const uint8_t e = tab[br.peek(7)];
    br.drop(e >> 5);
    const int sym = e & 31;
    int l = 0, rep = 1;
    if (sym < 16) {
      l = sym;
    } else if (sym == 16) {
      if (i == 0) return false;
      l = prev;
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
    if (!put(l, rep)) return false;
    prev = l;
  }
  return eob && lit_left == 0 && dist_left == 0;
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
  // LEN = 0 (a flush marker) is left out: PNG encoders do not flush mid-stream, and the
  // raw data of stored blocks of smooth images is full of 00 00 FF FF
  if ((len ^ nlen) != 0xFFFF || len == 0) return false;
  *next = q + 32 + 8 * static_cast<int64_t>(len);
  return *next <= in_bits;
}

// 0: no header at p; 1: dynamic header; 2: stored header (canonical start: its LEN byte)
__device__ int header_candidate(const uint32_t* w, int64_t p, int64_t in_bits, uint8_t* tab) {
  if (p + 3 > in_bits) return 0;
  if (dynamic_probe(w, p)) return dynamic_full(w, p, in_bits, tab) ? 1 : 0;
  int64_t nxt;
  if (!stored_probe(w, p, in_bits, &nxt)) return 0;
  if (nxt == in_bits - 32) return 2;  // the last block: the Adler-32 trailer follows
  // a stored block must be followed by another plausible header
  if (nxt + 3 > in_bits) return 0;
  if (dynamic_probe(w, nxt)) return dynamic_full(w, nxt, in_bits, tab) ? 2 : 0;
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

constexpr int kFindThreads = 256;

// bits [k, k + 32) of the 128-bit little-endian window (w3 w2 w1 w0), k in [0, 96]
__device__ __forceinline__ uint32_t win32(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                          uint32_t k) {
  const uint32_t s = k & 31;
  const uint32_t lo = k < 32 ? w0 : k < 64 ? w1 : w2, hi = k < 32 ? w1 : k < 64 ? w2 : w3;
  return __funnelshift_r(lo, hi, s);
}

// One warp per unit; each lane tests the 32 positions of one word per step (a warp
// step covers 1024 positions).  Stage 1 is bit-parallel over the word: BTYPE = 2 and
// HLIT, HDIST <= 29 (~22% of random positions pass).  Stage 2 sums the code-length
// code's Kraft terms with a 9-bit table (three 3-bit lengths per lookup); ~0.09% of
// random positions have a complete code.  Those go to the full check (decoding the code
// lengths: hundreds of dependent steps when the random lengths are mostly zeros), which
// the warp runs 32 candidates at a time, one per lane, from a per-warp queue -- run
// inline they would serialise the warp once per step.  Stored blocks are tested per byte
// boundary (LEN == ~NLEN).  Any true block start will do; the warp takes the first
// success of its first successful batch.
constexpr int kFindQueue = 32;
#ifndef TP_PNG_QFLUSH  // queued candidates that trigger a batch of full checks
#define TP_PNG_QFLUSH 24
#endif

// Each unit is scanned by kFindParts warps, one per quarter: a unit's start is the first
// header found in its lowest quarter that has one (k_png_find_select).  A warp stops early
// once a lower quarter of its unit has found a header.  The scratch (per unit: found
// position per quarter, lowest successful quarter) lives in the unit's token staging,
// which the inflate only uses later.
constexpr int kFindParts = 4;  // at most; the launch picks 1-4 by the number of units
static_assert(kUnitBits % (3 * 4 * 1024) == 0, "1-4 parts of whole 1024-bit steps");
struct FindScratch {
  long long pos[kFindParts];  // found start | 1 << 62 for a stored start; -1: none
  int lowest;                 // lowest quarter with a start (kFindParts: none yet)
};
// Work counters of the finder and the inflate rounds: the first 1 + kRounds ints of the
// unfilter's progress area (>= 64 ints; the unfilter zeroes it before its own use)
constexpr int kSchedInts = 1 + kRounds;
#ifndef TP_PNG_INFLATE_DYN  // the same for the inflate's units (per round)
#define TP_PNG_INFLATE_DYN 1
#endif
#ifndef TP_PNG_FIND_DYN  // 1: a resident grid of finder warps taking (unit, part) items in
#define TP_PNG_FIND_DYN 1  // order from a counter; 0: one warp per item (a partial last wave)
#endif
__device__ __forceinline__ FindScratch* find_scratch(uint32_t* stage, int u) {
  return reinterpret_cast<FindScratch*>(reinterpret_cast<uint8_t*>(stage) + u * kStageBytesPerUnit);
}

__global__ void k_png_find_init(uint32_t* stage, int U, int* sched) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < kSchedInts) sched[u] = 0;
  if (u >= U) return;
  FindScratch* f = find_scratch(stage, u);
  for (int p = 0; p < kFindParts; ++p) f->pos[p] = -1;
  f->lowest = kFindParts;
}

__global__ void k_png_find_select(PUnit* __restrict__ units, uint32_t* stage, int U, int parts,
                                  int debug) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= U) return;
  const FindScratch* f = find_scratch(stage, u);
  long long v = -1;
  for (int p = 0; p < parts && v < 0; ++p) v = f->pos[p];
  int64_t start = v < 0 ? -1 : (v & ((1ll << 62) - 1));
  // test hook (tests/test_gpu_png.py): every third found start moved one bit on, a false
  // header the chain check must catch -- the preceding unit's decode passes it, the start
  // is dropped and that unit decodes again in the next round
  if ((debug & 1) && start > 16 && u % 3 == 1 && (v >> 62) == 0) start += 1;
  PUnit& o = units[u];
  o.start = start;
  o.end = -1;
  o.out_len = 0;
  o.out_off = 0;
  o.ntok = 0;
  o.status = kUnitOk;
  o.final_ = 0;
  o.dirty = start >= 0;
  o.stored = v >= 0 && (v >> 62) != 0;
  o.nmark = 0;  // expand skips units without output: the window pass must see no list
  o.fixups = 0;
  o.rounds = 0;
  o.redo = 0;
}

__global__ void __launch_bounds__(kFindThreads)
    k_png_find(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc, int n,
               PUnit* __restrict__ units, int U, uint32_t* stage, int parts, int* sched) {
  __shared__ uint8_t tabs[kFindThreads][128];  // code-length code of a lane's full check
  __shared__ uint8_t kraft9[512];              // Kraft terms of three 3-bit lengths
  __shared__ int64_t queue[kFindThreads / 32][kFindQueue];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    int sum = 0;
    for (int f = 0; f < 3; ++f) {
      const int l = (i >> (3 * f)) & 7;
      if (l) sum += 128 >> l;
    }
    kraft9[i] = static_cast<uint8_t>(sum);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // units need very different scan lengths (the distance from the unit start to the next
  // block header): warps take items from a counter instead of one fixed item each
  int* next_item = sched;
  for (int it = 0;; ++it) {
  int gw;
  if (TP_PNG_FIND_DYN) {
    int v = 0;
    if (lane == 0) v = atomicAdd(next_item, 1);
    gw = __shfl_sync(0xffffffffu, v, 0);
  } else {
    if (it > 0) break;
    gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  }
  const int u = gw / parts, part = gw % parts;
  if (u >= U) break;
  FindScratch* fs = find_scratch(stage, u);
  int64_t* q = queue[threadIdx.x >> 5];
  const int k = unit_image(desc, n, u);
  const PDesc& d = desc[k];
  const int local = u - d.unit_base;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(payload + d.in_off);
  uint8_t* tab = tabs[threadIdx.x];
  int64_t start = -1;
  int stored = 0;
  if (local == 0) {
    if (part == 0) start = 16;  // after the zlib header
  } else {
    const int64_t part_bits = kUnitBits / parts;
    const int64_t lo = static_cast<int64_t>(local) * kUnitBits + part * part_bits;
    const int64_t hi = min(lo + part_bits, d.in_bits - 3);
    int qn = 0;  // queued candidates (warp-uniform)
    int nsteps = 0;  // steps of this warp (the early-exit check runs every fourth)
    // run the queued full checks, one per lane; the first success is the start
    auto flush = [&]() -> bool {
      __syncwarp();
      const bool ok = lane < qn && dynamic_full(w, q[lane], d.in_bits, tab);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      qn = 0;
      __syncwarp();
      if (!m) return false;
      start = q[__ffs(m) - 1];
      return true;
    };
    for (int64_t p0 = lo; p0 < hi; p0 += 1024) {
      ++nsteps;
      // a lower quarter of this unit has its start: this one is not needed
      if (part > 0 && (nsteps & 3) == 1 &&
          __shfl_sync(0xffffffffu, lane == 0 ? *reinterpret_cast<volatile int*>(&fs->lowest) : 0, 0) < part)
        break;
      const int64_t wi = (p0 >> 5) + lane;
      const int64_t pw = wi << 5;  // this lane's first position
      int64_t found = -1;
      int64_t mine[2];
      int nmine = 0;
      if (pw < hi) {
        const uint32_t w0 = __ldg(w + wi), w1 = __ldg(w + wi + 1), w2 = __ldg(w + wi + 2),
                       w3 = __ldg(w + wi + 3);
        auto bits = [&](uint32_t kk) { return win32(w0, w1, w2, w3, kk); };
        const uint32_t lim = hi - pw >= 32 ? 0xFFFFFFFFu : ((1u << (hi - pw)) - 1u);
        uint32_t cand = ~bits(1) & bits(2) & ~(bits(4) & bits(5) & bits(6) & bits(7)) &
                        ~(bits(9) & bits(10) & bits(11) & bits(12)) & lim;
        while (cand) {
          const uint32_t b = __ffs(cand) - 1;
          cand &= cand - 1;
          const int hclen = static_cast<int>((bits(b + 13) & 15)) + 4;
          const uint64_t y = (static_cast<uint64_t>(bits(b + 49)) << 32) | bits(b + 17);
          const uint64_t ym = y & ((1ull << (3 * hclen)) - 1);
          int sum = 0;
#pragma unroll
          for (int g = 0; g < 7; ++g) sum += kraft9[(ym >> (9 * g)) & 511];
          if (sum == 128 && nmine < 2) mine[nmine++] = pw + b;
        }
        // stored: LEN / NLEN at the byte boundaries q in (pw + 3, pw + 42]
        const uint32_t none = ~bits(1) & ~bits(2) & lim;  // BTYPE = 00 positions
        for (uint32_t qb = 8; qb <= 40 && found < 0; qb += 8) {
          const uint32_t v = bits(qb);
          if (((v & 0xFFFF) ^ (v >> 16)) != 0xFFFF || (v & 0xFFFF) == 0) continue;
          // a header position p in [q - 10, q - 3] of this word, zero-padded to q
          for (int pb = static_cast<int>(qb) - 10; pb <= static_cast<int>(qb) - 3; ++pb) {
            if (pb < 0 || pb > 31 || !((none >> pb) & 1)) continue;
            const int pad = static_cast<int>(qb) - (pb + 3);
            if (pad && (bits(pb + 3) & ((1u << pad) - 1)) != 0) continue;
            if (header_candidate(w, pw + pb, d.in_bits, tab) == 2) {
              found = pw + qb;  // canonical start: the LEN byte
              break;
            }
          }
        }
      }
      const unsigned ms = __ballot_sync(0xffffffffu, found >= 0);
      if (ms) {
        start = __shfl_sync(0xffffffffu, found, __ffs(ms) - 1);
        stored = 1;
        break;
      }
      // queue this step's candidates (at most two per lane; more only cost parallelism)
      for (int c = 0; c < 2; ++c) {
        const bool has = c < nmine;
        const unsigned mh = __ballot_sync(0xffffffffu, has);
        if (!mh) break;
        const int slot = qn + __popc(mh & ((1u << lane) - 1u));
        if (has && slot < kFindQueue) q[slot] = mine[c];
        qn = min(kFindQueue, qn + __popc(mh));
        if (qn >= TP_PNG_QFLUSH && flush()) break;
      }
      if (start >= 0) break;
    }
    if (start < 0 && qn > 0) flush();
  }
  if (lane == 0 && start >= 0) {
    fs->pos[part] = start | (stored ? (1ll << 62) : 0);
    atomicMin(&fs->lowest, part);
  }
  }  // items
}

// ---------------------------------------------------------------------------
// inflate: one warp per unit.  Block headers (and stored blocks) are read by lane 0,
// which builds the block's Huffman tables in the warp's shared memory.  A block's data
// is decoded in rounds of 32 subsequences of kSubBits bits, one per lane: lane 0 starts
// at the round's true position, lane j at a speculative position kLeadBits before its
// nominal start, and takes the first symbol boundary at or past the nominal start as its
// entry (Huffman codes self-synchronise, so after the lead-in it is almost always on the
// true symbol grid).  Lanes whose entry differs from their predecessor's exit are decoded
// again from that exit, lowest first, until the subsequences tile the round; then every
// lane decodes its subsequence once more, writing its tokens at its prefix-sum offset.

#ifndef TP_PNG_LEAD
#define TP_PNG_LEAD 256
#endif
constexpr int kLeadBits = TP_PNG_LEAD;
// a lane's tokens for one subsequence (<= kSubBits + one symbol of bits: at most one
// token per 1.5 bits) wait in a per-lane staging area until the round's offsets are known
constexpr int kStageTokens = kSubBits + 64;
static_assert(kStageBytesPerUnit == 32 * kStageTokens * 4, "staging layout");
constexpr int kInflateWarps = 4;

struct SegResult {
  int64_t exit;  // first symbol boundary >= end, or the bit after the end-of-block code
  int ntok;
  int nout;
  int stop;      // 0: reached `end`; 1: end of block; 2: invalid code / overrun
};

// Decode from `from` (taken as a symbol boundary) until the position reaches `end`, an
// end-of-block code or an invalid code.  out != nullptr: write the tokens (literal packs
// are flushed at the segment's end, so counts depend only on the segment).
__device__ SegResult decode_seg(const uint32_t* w, int64_t from, int64_t end, int64_t in_bits,
                                const uint16_t* lt, const uint8_t* dt, uint32_t* out,
                                int out_cap = 1 << 30) {
  SegResult r;
  r.ntok = 0;
  r.nout = 0;
  r.stop = 0;
  Bits br;
  br.init(w, from);
  uint32_t pack = 0;
  int pc = 0;
  const int64_t wlim = (in_bits >> 5) + 12;  // past the stream (and its padding) by now
  // bits left before `end` (a segment is at most a few thousand bits): one subtract per
  // code instead of recomputing the reader's 64-bit position
  int left = static_cast<int>(min(end - from, static_cast<int64_t>(1) << 30));
  while (true) {
    if (left <= 0) break;
    br.refill();
    if (br.wi > wlim) { r.stop = 2; break; }
    uint32_t e = lt[br.peek(kLitRoot)];
    if (e & 0x8000u) {
      const int sub = (e >> 12) & 7;
      if (sub == 7) { r.stop = 2; break; }
      e = lt[(e & 0xFFFu) + (br.peek(kLitRoot + sub) >> kLitRoot)];
      if (e & 0x8000u) { r.stop = 2; break; }
    }
    const int cl = (e >> 11) & 15;
    br.drop(cl);
    left -= cl;
    const int sym = static_cast<int>(e & 511u);
    if (sym < 256) {
      pack |= static_cast<uint32_t>(sym) << (8 * pc);
      ++r.nout;
      if (++pc == 3) {
        if (out && r.ntok < out_cap) out[r.ntok] = (3u << 24) | pack;
        ++r.ntok;
        pc = 0;
        pack = 0;
      }
      continue;
    }
    if (sym == 256) { r.stop = 1; break; }
    if (sym > 285) { r.stop = 2; break; }
    int base, extra;
    length_base(sym - 257, base, extra);
    const int len = base + static_cast<int>(br.peek(extra));
    br.drop(extra);
    br.refill();
    const int n0 = br.n;
    const int ds = decode_dist(br, dt);
    if (ds < 0 || ds > 29) { r.stop = 2; break; }
    int dbase, dextra;
    dist_base(ds, dbase, dextra);
    const int dist = dbase + static_cast<int>(br.peek(dextra));
    br.drop(dextra);
    left -= extra + (n0 - br.n);
    if (pc) {
      if (out && r.ntok < out_cap) out[r.ntok] = (static_cast<uint32_t>(pc) << 24) | pack;
      ++r.ntok;
      pc = 0;
      pack = 0;
    }
    if (out && r.ntok < out_cap)
      out[r.ntok] = kTokMatch | (static_cast<uint32_t>(len - 3) << 16) | static_cast<uint32_t>(dist - 1);
    ++r.ntok;
    r.nout += len;
  }
  if (pc && r.stop != 2) {
    if (out && r.ntok < out_cap) out[r.ntok] = (static_cast<uint32_t>(pc) << 24) | pack;
    ++r.ntok;
  }
  if (r.ntok > out_cap) r.stop = 2;  // more tokens than the staging holds
  r.exit = br.pos();
  return r;
}

struct __align__(16) WarpTables {
  uint16_t lit[kLitCap];
  uint8_t dist[kDistBytes];
  uint8_t lens[320];   // code lengths of the block being set up
  uint8_t pre[128];    // code-length code
  uint16_t sorted[288];  // long literal/length codes in canonical order (build_lit)
};

__global__ void __launch_bounds__(32 * kInflateWarps)
    k_png_inflate(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc, int n,
                  PUnit* __restrict__ units, int U, uint32_t* __restrict__ toks,
                  uint32_t* __restrict__ stage, const int32_t* __restrict__ img_status, int* sched,
                  int round) {
  __shared__ WarpTables wt_all[kInflateWarps];
  const int lane = threadIdx.x & 31;
  WarpTables& wt = wt_all[threadIdx.x >> 5];
  // a resident wave of warps takes the units in order from a per-round counter (the units'
  // decode times differ; one warp per unit left a partial last wave)
  int* next_unit = sched + 1 + round;
  for (int it = 0;; ++it) {
  int u;
  if (TP_PNG_INFLATE_DYN) {
    int v = 0;
    if (lane == 0) v = atomicAdd(next_unit, 1);
    u = __shfl_sync(0xffffffffu, v, 0);
  } else {
    if (it > 0) break;
    u = blockIdx.x * kInflateWarps + (threadIdx.x >> 5);
  }
  if (u >= U) break;
  PUnit& me = units[u];
  if (!me.dirty) continue;
  const int k = unit_image(desc, n, u);
  const PDesc& d = desc[k];
  if (img_status[k] != kImgOk) continue;
  const int64_t start = me.start;
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
  const uint32_t* w = reinterpret_cast<const uint32_t*>(payload + d.in_off);
  uint32_t* tk = toks + d.tok_off + (start >> 1);
  const int64_t cap = last ? d.in_bits / 2 + 256 - (start >> 1) : (stop >> 1) - (start >> 1);
  int64_t ntok = 0, out = 0, cur = start, end = start;
  int status = kUnitOk, fin = 0;
  bool stored_start = me.stored != 0;
  const unsigned below = (1u << lane) - 1u;
  int nfix = 0, nround = 0;  // diagnostics (PUnit::fixups / rounds)
  uint32_t* warp_stage = stage + static_cast<int64_t>(u) * 32 * kStageTokens;
  uint32_t* my_stage = warp_stage + lane * kStageTokens;
  while (true) {
    // ---- block boundary at `cur` (lane 0 reads the header; the state is broadcast)
    int btype = 0, bfinal = 0, action = 0;  // action: 0 data, 1 stored done, 2 stop, 3 error
    int64_t h = cur;
    if (lane == 0) {
      Bits br;
      br.init(w, cur);
      if (stored_start) {
        btype = 0;
        end = cur;
      } else if (cur + 3 > in_bits) {
        action = 3;
        status = kUnitOverrun;
      } else {
        const uint32_t hdr = br.peek(3);
        btype = static_cast<int>(hdr >> 1);
        bfinal = static_cast<int>(hdr & 1);
        end = btype == 0 ? (cur + 3 + 7) & ~int64_t(7) : cur;
        if (!last && end >= stop) action = 2;
        else br.drop(3);
      }
      if (action == 0 && btype == 0) {  // stored
        if (!stored_start) br.drop(br.n & 7);
        const int64_t q = br.pos();
        br.refill();
        const uint32_t v32 = static_cast<uint32_t>(br.buf);
        const uint32_t len = v32 & 0xFFFF, nlen = v32 >> 16;
        const int64_t next = q + 32 + 8 * static_cast<int64_t>(len);
        if ((len ^ nlen) != 0xFFFF) {
          action = 3;
          status = kUnitBadStored;
        } else if (next > in_bits) {
          action = 3;
          status = kUnitOverrun;
        } else {
          if (len) {
            if (ntok >= cap) {
              action = 3;
              status = kUnitTokens;
            } else {
              tk[ntok++] = kTokStored | static_cast<uint32_t>((q + 32) >> 3);
              out += len;
            }
          }
          if (action == 0) {
            action = 1;
            h = next;
            if (next == in_bits - 32) bfinal = 1;  // only the final block meets the trailer
          }
        }
      } else if (action == 0 && (btype == 1 || btype == 2)) {
        bool ok;
        if (btype == 1) {
          for (int i = 0; i < 144; ++i) wt.lens[i] = 8;
          for (int i = 144; i < 256; ++i) wt.lens[i] = 9;
          for (int i = 256; i < 280; ++i) wt.lens[i] = 7;
          for (int i = 280; i < 288; ++i) wt.lens[i] = 8;
          for (int i = 0; i < 32; ++i) wt.lens[288 + i] = 5;
          ok = build_lit(wt.lens, 288, wt.lit, wt.sorted) && build_dist(wt.lens + 288, 32, wt.dist);
        } else {
          int hlit, hdist;
          ok = read_dynamic_lengths(br, wt.lens, wt.pre, hlit, hdist, in_bits) &&
               build_lit(wt.lens, hlit, wt.lit, wt.sorted) && build_dist(wt.lens + hlit, hdist, wt.dist);
        }
        if (!ok) {
          action = 3;
          status = kUnitBadCode;
        }
        h = br.pos();
      } else if (action == 0) {
        action = 3;
        status = kUnitBadCode;
      }
    }
    stored_start = false;
    action = __shfl_sync(0xffffffffu, action, 0);
    status = __shfl_sync(0xffffffffu, status, 0);
    bfinal = __shfl_sync(0xffffffffu, bfinal, 0);
    h = __shfl_sync(0xffffffffu, h, 0);
    end = __shfl_sync(0xffffffffu, end, 0);
    ntok = __shfl_sync(0xffffffffu, ntok, 0);
    out = __shfl_sync(0xffffffffu, out, 0);
    if (action >= 2) break;
    if (action == 1) {  // stored block done
      cur = h;
      if (bfinal) {
        fin = 1;
        break;
      }
      continue;
    }
    __syncwarp();  // tables visible to every lane
    // ---- the block's data, in rounds of 32 subsequences
    bool eob = false;
    while (true) {
      const int64_t nom = h + static_cast<int64_t>(lane) * kSubBits, nom_end = nom + kSubBits;
      int64_t entry;
      SegResult r;
      if (lane == 0) {
        entry = h;
        r = decode_seg(w, h, nom_end, in_bits, wt.lit, wt.dist, my_stage, kStageTokens);
      } else {
        const SegResult lead = decode_seg(w, max(h, nom - kLeadBits), nom, in_bits, wt.lit,
                                          wt.dist, nullptr);
        if (lead.stop == 0) {
          entry = lead.exit;
          r = decode_seg(w, entry, nom_end, in_bits, wt.lit, wt.dist, my_stage, kStageTokens);
        } else {  // the speculative path stopped in the lead-in
          entry = -1;
          r = lead;
          r.stop = 2;
        }
      }
      // fix-up: the lowest lane whose entry is not its predecessor's exit decodes again
      while (true) {
        const int64_t pexit = __shfl_up_sync(0xffffffffu, r.exit, 1);
        const unsigned stops = __ballot_sync(0xffffffffu, r.stop != 0);
        const bool bad = lane > 0 && !(stops & below) && entry != pexit;
        const unsigned mb = __ballot_sync(0xffffffffu, bad);
        if (!mb) break;
        ++nfix;
        if (lane == __ffs(mb) - 1) {
          entry = pexit;
          r = decode_seg(w, entry, nom_end, in_bits, wt.lit, wt.dist, my_stage, kStageTokens);
        }
      }
      ++nround;
      const unsigned stops = __ballot_sync(0xffffffffu, r.stop != 0);
      const int J = stops ? __ffs(stops) - 1 : 31;  // last lane of the round
      const bool in_round = lane <= J;
      const int jstop = __shfl_sync(0xffffffffu, r.stop, J);
      if (jstop == 2) {
        status = kUnitBadCode;
        break;
      }
      // token offsets of the round's lanes
      int incl = in_round ? r.ntok : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int rtok = __shfl_sync(0xffffffffu, incl, 31);
      int rout = in_round ? r.nout : 0;
      for (int o = 16; o > 0; o >>= 1) rout += __shfl_xor_sync(0xffffffffu, rout, o);
      if (ntok + rtok > cap) {
        status = kUnitTokens;
        end = h;
        break;
      }
      // the round's tokens, lane by lane, from the staging areas (coalesced copies)
      __syncwarp();
      for (int j = 0; j <= J; ++j) {
        const int nj = __shfl_sync(0xffffffffu, r.ntok, j);
        const int bj = __shfl_sync(0xffffffffu, incl - r.ntok, j);
        const uint32_t* src = warp_stage + j * kStageTokens;
        for (int i = lane; i < nj; i += 32) tk[ntok + bj + i] = src[i];
      }
      ntok += rtok;
      out += rout;
      h = __shfl_sync(0xffffffffu, r.exit, J);
      if (jstop == 1) {
        eob = true;
        break;
      }
    }
    if (status != kUnitOk) break;
    cur = h;
    if (eob && bfinal) {
      fin = 1;
      break;
    }
    __syncwarp();  // the next header rebuilds the tables
  }
  if (lane == 0) {
    me.end = (last || status == kUnitTokens || fin) ? (status == kUnitTokens ? end : cur) : end;
    me.ntok = static_cast<int32_t>(ntok);
    me.out_len = out;
    me.status = status;
    me.final_ = fin;
    me.dirty = 0;
    me.fixups = nfix;
    me.rounds = nround;
  }
  __syncwarp();  // the next unit's header rebuilds this warp's tables
  }  // units
}

// ---------------------------------------------------------------------------
// chain: one warp per image (lane 0 walks; the units are few)

__global__ void k_png_chain(const PDesc* __restrict__ desc, int n, PUnit* __restrict__ units,
                            int32_t* __restrict__ img_status, int round) {
  const int k = blockIdx.x;
  if (k >= n || threadIdx.x != 0) return;
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const bool last_round = round == kRounds - 1;
  const int u0 = d.unit_base, u1 = d.unit_base + d.n_units;
  // after round 0, only images with re-decoded units walk again (the first unit's `redo`
  // carries that mark from round to round)
  if (round > 0 && units[u0].redo == 0) return;
  units[u0].redo = 0;
  auto next_valid = [&](int u) {
    int v = u + 1;
    while (v < u1 && units[v].start < 0) ++v;
    return v;
  };
  // pass 1: every unit must end where the next start is.  A start the preceding unit's
  // decode passed is not a block start (a finder false positive): it is dropped and the
  // preceding unit decodes again next round.  The walk goes on past such a pair, taking
  // the next start as true until shown otherwise, so all the false starts of an image are
  // dropped in one round and their re-decodes run in parallel.  (Taking a false start
  // for true can at worst drop a true start after it: a longer unit, not a wrong one.)
  bool redo = false;
  bool validated = true;  // u's start is where its predecessor's decode ended (or bit 16)
  int prev = -1;          // the valid unit before u
  for (int u = u0; u < u1;) {
    PUnit& cu = units[u];
    const int v = next_valid(u);
    if (cu.dirty) {  // its end is not known yet: the next start cannot be judged now
      redo = true;
      validated = false;
      prev = u;
      u = v;
      continue;
    }
    if (cu.status != kUnitOk && !(cu.status == kUnitTokens && v < u1 && cu.end > units[v].start)) {
      if (validated) {  // a true block start that does not decode: a corrupt stream
        img_status[k] = kImgInflate;
        return;
      }
      // an unconfirmed start that does not decode is almost surely a false one: drop it
      // now (the unit before decodes on over its range), so runs of false starts -- the
      // raw data of stored blocks of flat images -- go in one round
      cu.start = -1;
      cu.dirty = 0;
      if (prev >= 0) units[prev].dirty = 1;
      redo = true;
      u = v;
      continue;
    }
    if (v >= u1) break;
    if (cu.final_ && cu.status == kUnitOk) {  // a header past the end of the final block
      units[v].start = -1;
      units[v].dirty = 0;
      continue;  // the same unit against its next successor
    }
    if (cu.end != units[v].start) {  // (or a token overflow past the next start)
      units[v].start = -1;
      units[v].dirty = 0;
      cu.dirty = 1;
      redo = true;
      validated = false;
      prev = u;
      u = next_valid(v);
      continue;
    }
    validated = true;
    prev = u;
    u = v;
  }
  if (redo) {
    units[u0].redo = 1;
    if (last_round) img_status[k] = kImgChain;
    return;
  }
  // pass 2: the chain is whole; inflated offsets, the final block, the length
  int64_t off = 0;
  int u = u0;  // unit 0 always starts at a real block
  while (true) {
    PUnit& cu = units[u];
    if (cu.status != kUnitOk) {
      img_status[k] = kImgInflate;
      return;
    }
    cu.out_off = off;
    off += cu.out_len;
    const int v = next_valid(u);
    if (v >= u1) {
      if (!cu.final_) {
        img_status[k] = kImgNotFinal;
        return;
      }
      units[u0].final_end = cu.end;
      break;
    }
    u = v;
  }
  if (off != d.raw_len) img_status[k] = kImgLength;
}

// ---------------------------------------------------------------------------
// expand: one warp per unit, tokens -> u16 bytes (>= 256: window markers).  The
// positions of marker bytes go to the unit's list (a warp-aggregated append: the warp
// walks its unit's tokens in order, so a register counter is the list's length).

#ifndef TP_PNG_EXPAND_MINB  // resident expand CTAs per SM: 6 (<= 40 registers) holds the
#define TP_PNG_EXPAND_MINB 6  // 6,000 unit warps of 64 1080p PNGs in one wave (5: 5,920)
#endif
__global__ void __launch_bounds__(256, TP_PNG_EXPAND_MINB)
    k_png_expand(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc,
                             int n, PUnit* __restrict__ units, int U,
                             const uint32_t* __restrict__ toks, uint16_t* __restrict__ T,
                             uint32_t* __restrict__ M, int32_t* __restrict__ img_status) {
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
  uint32_t* list = M + d.raw_off + ws;
  const unsigned lt_mask = (1u << lane) - 1u;
  int nmark = 0;
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
        for (int j0 = 0; j0 < ln; j0 += 32) {
          const int j = j0 + lane;
          bool mk = false;
          if (j < ln) {
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
            mk = v >= 256;
          }
          const unsigned mm = __ballot_sync(0xffffffffu, mk);
          if (mk) list[nmark + __popc(mm & lt_mask)] = static_cast<uint32_t>(dst + j);
          nmark += __popc(mm);
        }
      }
      __syncwarp();
    }
    cur += total;
  }
  if (lane == 0) units[u].nmark = nmark;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(img_status + k, kImgDistance);
}

// ---------------------------------------------------------------------------
// final: every byte of T into the row layout of R (markers too, as garbage: `window`
// rewrites them); one CTA per row of the batch, eight bytes per thread

__device__ __forceinline__ int row_image(const PDesc* __restrict__ desc, int n, int g) {
  int lo = 0, hi = n;  // largest k with row_base <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (desc[mid].row_base <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// R byte of inflated byte p (image-relative) of image d
__device__ __forceinline__ uint8_t* r_byte(const PDesc& d, uint8_t* r, uint32_t p) {
  const uint32_t stride = static_cast<uint32_t>(d.width) * d.bpp + 1;
  const uint32_t y = p / stride, x = p - y * stride;
  return x == 0 ? r + y : r + r_filter_bytes(d.height) + static_cast<int64_t>(y) * d.r_stride + (x - 1);
}

__global__ void k_png_final(const PDesc* __restrict__ desc, int n, const uint16_t* __restrict__ T,
                            uint8_t* __restrict__ R, const int32_t* __restrict__ img_status) {
  const int g = blockIdx.x;
  const int k = row_image(desc, n, g);
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const int y = g - d.row_base;
  const int64_t rowbytes = static_cast<int64_t>(d.width) * d.bpp;
  const uint16_t* t = T + d.raw_off + static_cast<int64_t>(y) * (rowbytes + 1);
  uint8_t* r = R + d.r_off;
  if (threadIdx.x == 0) r[y] = static_cast<uint8_t>(t[0]);
  uint8_t* row = r + r_filter_bytes(d.height) + static_cast<int64_t>(y) * d.r_stride;
  for (int64_t x = 8 * static_cast<int64_t>(threadIdx.x); x < rowbytes; x += 8 * blockDim.x) {
    uint32_t b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = x + j < rowbytes ? (t[1 + x + j] & 255u) : 0u;
    uint2 v;
    v.x = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
    v.y = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
    *reinterpret_cast<uint2*>(row + x) = v;  // r_stride is a multiple of 16
  }
}

// window: one CTA per image, units in order: each unit's marker bytes read the window
// before the unit, whose bytes are final by then (earlier units' markers resolved)
__global__ void k_png_window(const PDesc* __restrict__ desc, int n, const PUnit* __restrict__ units,
                             const uint16_t* __restrict__ T, const uint32_t* __restrict__ M,
                             uint8_t* __restrict__ R, const int32_t* __restrict__ img_status) {
  const int k = blockIdx.x;
  const PDesc& d = desc[k];
  if (d.n_units == 0 || img_status[k] != kImgOk) return;
  const uint16_t* t = T + d.raw_off;
  uint8_t* r = R + d.r_off;
  for (int u = d.unit_base; u < d.unit_base + d.n_units; ++u) {
    const int cnt = (units[u].start < 0 || units[u].out_len == 0) ? 0 : units[u].nmark;
    if (!cnt) continue;  // uniform across the CTA
    const int64_t os = units[u].out_off, wb = os - kWindow;
    const uint32_t* list = M + d.raw_off + os;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t p = list[i];
      const uint32_t src = static_cast<uint32_t>(wb + (t[p] - 256));
      *r_byte(d, r, p) = *r_byte(d, r, src);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Adler-32 (RFC 1950 §8) of the inflated bytes, checked when the stream holds the four
// trailer bytes after the final block.  Pillow's zlib verifies the trailer whenever it
// is in the data it was fed (a wrong one raises "broken data stream"), and says nothing
// when the stream ends before it (tests/test_gpu_png.py, bad payloads).  For n bytes,
// a = 1 + sum d_i and b = n + sum (n - i) d_i (mod 65521): both are plain sums, so any
// part of the stream can be summed anywhere and added up.

__device__ __forceinline__ int blk_image(const PDesc* __restrict__ desc, int n, int g) {
  int lo = 0, hi = n;  // largest k with blk_base <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (desc[mid].blk_base <= g) lo = mid; else hi = mid;
  }
  return lo;
}

constexpr uint32_t kAdlerMod = 65521;
constexpr int kAdlerThreads = 256;

__device__ __forceinline__ bool adler_trailer(const PDesc& d, const PUnit* units, int64_t* at) {
  const int64_t fin = units[d.unit_base].final_end;
  *at = (fin + 7) >> 3;  // trailer bytes, big-endian
  return *at + 4 <= (d.in_bits >> 3);
}

// One CTA per unfilter row block (128 scanlines) of an image, warp per row, lanes over
// 16-byte chunks: sum d_i and sum (n - i) d_i (mod 65521) of the block's inflated bytes
// (filter bytes included, i their index in the stream), added into the image's sums.
__global__ void __launch_bounds__(kAdlerThreads)
    k_png_adler_rows(const PDesc* __restrict__ desc, int n, const PUnit* __restrict__ units,
                     const uint8_t* __restrict__ R, const int32_t* __restrict__ img_status,
                     unsigned long long* __restrict__ acc, int n_blocks) {
  __shared__ unsigned long long red[2][kAdlerThreads / 32];
  const int g = blockIdx.x;
  if (g >= n_blocks) return;
  const int k = blk_image(desc, n, g);
  const PDesc& d = desc[k];
  int64_t at;
  if (d.n_units == 0 || img_status[k] != kImgOk || !adler_trailer(d, units, &at)) return;
  const int64_t len = d.raw_len;
  const int64_t rowbytes = static_cast<int64_t>(d.width) * d.bpp, stride = rowbytes + 1;
  const int H = d.height;
  const int y0 = (g - d.blk_base) * kUnfilterRows, y1 = min(H, y0 + kUnfilterRows);
  const uint8_t* fb = R + d.r_off;
  const uint8_t* rows = fb + r_filter_bytes(H);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t a = 0, b = 0;
  for (int y = y0 + warp; y < y1; y += kAdlerThreads / 32) {
    const int64_t i0 = static_cast<int64_t>(y) * stride;
    uint64_t la = 0, lb = 0;
    if (lane == 0) {
      la = fb[y];
      lb = static_cast<uint64_t>(len - i0) * fb[y];
    }
    const uint8_t* row = rows + static_cast<int64_t>(y) * d.r_stride;
    for (int64_t x = 16 * static_cast<int64_t>(lane); x < rowbytes; x += 16 * 32) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + x);
      uint32_t wv[4] = {v.x, v.y, v.z, v.w};
      if (x + 16 > rowbytes) {  // the row's last chunk: bytes past the row are padding
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t keep = rowbytes - (x + 4 * q);  // bytes of word q inside the row
          wv[q] = keep >= 4 ? wv[q] : keep <= 0 ? 0u : wv[q] & ((1u << (8 * keep)) - 1u);
        }
      }
      // byte j of the chunk weighs wt0 - j: sum (wt0 - j) d_j = wt0 * S - T with S = sum d_j
      // and T = sum j d_j, both from four byte dot products (dp4a) each
      const uint64_t wt0 = static_cast<uint64_t>(len - (i0 + 1 + x));  // weight of byte x
      uint32_t S = 0, T = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        S = __dp4a(wv[q], 0x01010101u, S);
        T = __dp4a(wv[q], 0x03020100u + 0x04040404u * q, T);
      }
      la += S;
      lb += wt0 * S - T;
    }
    a += la;
    b += lb % kAdlerMod;
  }
  a %= kAdlerMod;
  b %= kAdlerMod;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    red[0][warp] = a;
    red[1][warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t A = 0, B = 0;
    for (int w = 0; w < kAdlerThreads / 32; ++w) {
      A += red[0][w];
      B += red[1][w];
    }
    atomicAdd(acc + 2 * k, A % kAdlerMod);
    atomicAdd(acc + 2 * k + 1, B % kAdlerMod);
  }
}

__global__ void k_png_adler_check(const uint8_t* __restrict__ payload, const PDesc* __restrict__ desc,
                                  int n, const PUnit* __restrict__ units,
                                  const unsigned long long* __restrict__ acc,
                                  int32_t* __restrict__ img_status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const PDesc& d = desc[k];
  int64_t at;
  if (d.n_units == 0 || img_status[k] != kImgOk || !adler_trailer(d, units, &at)) return;
  const uint64_t A = (1 + acc[2 * k]) % kAdlerMod;
  const uint64_t B = (static_cast<uint64_t>(d.raw_len) % kAdlerMod + acc[2 * k + 1]) % kAdlerMod;
  const uint8_t* z = payload + d.in_off + at;
  const uint32_t want = (uint32_t(z[0]) << 24) | (uint32_t(z[1]) << 16) | (uint32_t(z[2]) << 8) | z[3];
  if (((B << 16) | A) != want) atomicOr(img_status + k, kImgAdler);
}

// ---------------------------------------------------------------------------
// unfilter (PNG §9.2) + L/P -> RGB: one CTA per image, thread = scanline



#ifndef TP_PNG_UNFILTER_SPLIT  // 1: one code path per filter type; 0: all predictors, selected
#define TP_PNG_UNFILTER_SPLIT 1
#endif
// chunk of one scanline per wavefront step: NW 32-bit words (TP_PNG_CHUNK bytes)
#ifndef TP_PNG_CHUNK
#define TP_PNG_CHUNK 16
#endif
constexpr int kChunkWords = TP_PNG_CHUNK / 4;
template <int NW> struct ChunkVec;
template <> struct ChunkVec<4> {
  using T = uint4;
  __device__ __forceinline__ static uint32_t w(const T& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  __device__ __forceinline__ static T make(const uint32_t* a) { return make_uint4(a[0], a[1], a[2], a[3]); }
};
template <> struct ChunkVec<2> {
  using T = uint2;
  __device__ __forceinline__ static uint32_t w(const T& v, int i) { return i == 0 ? v.x : v.y; }
  __device__ __forceinline__ static T make(const uint32_t* a) { return make_uint2(a[0], a[1]); }
};
struct Words8 {  // 32-byte chunk
  uint4 a, b;
};
template <> struct ChunkVec<8> {
  using T = Words8;
  __device__ __forceinline__ static uint32_t w(const T& v, int i) {
    return ChunkVec<4>::w(i < 4 ? v.a : v.b, i & 3);
  }
  __device__ __forceinline__ static T make(const uint32_t* a) {
    return Words8{make_uint4(a[0], a[1], a[2], a[3]), make_uint4(a[4], a[5], a[6], a[7])};
  }
};
// L2-coherent chunk loads / stores (the block-to-block row handoff)
__device__ __forceinline__ uint4 chunk_ldcg(const uint4* p) { return __ldcg(p); }
__device__ __forceinline__ uint2 chunk_ldcg(const uint2* p) { return __ldcg(p); }
__device__ __forceinline__ Words8 chunk_ldcg(const Words8* p) {
  return Words8{__ldcg(&p->a), __ldcg(&p->b)};
}
__device__ __forceinline__ void chunk_stcg(uint4* p, const uint4& v) { __stcg(p, v); }
__device__ __forceinline__ void chunk_stcg(uint2* p, const uint2& v) { __stcg(p, v); }
__device__ __forceinline__ void chunk_stcg(Words8* p, const Words8& v) {
  __stcg(&p->a, v.a);
  __stcg(&p->b, v.b);
}
__device__ __forceinline__ void chunk_stcs(uint4* p, const uint4& v) { __stcs(p, v); }
__device__ __forceinline__ void chunk_stcs(uint2* p, const uint2& v) { __stcs(p, v); }
__device__ __forceinline__ void chunk_stcs(Words8* p, const Words8& v) {
  __stcs(&p->a, v.a);
  __stcs(&p->b, v.b);
}
using CV = ChunkVec<kChunkWords>;
using Chunk = CV::T;
constexpr int kCh = 4 * kChunkWords;

__device__ __forceinline__ uint32_t byte_at(const Chunk& v, int j) {  // j: compile-time
  return (CV::w(v, j >> 2) >> (8 * (j & 3))) & 255u;
}

__device__ __forceinline__ uint32_t pack4(const uint32_t* b) {
  return b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
}


// One row block (kUnfilterRows consecutive scanlines of one image) per work item, thread
// = scanline: at step t thread y reconstructs chunk t - y of its row, whose prior-row bytes
// thread y - 1 reconstructed at step t - 1 (shared-memory exchange, double-buffered).  The
// block's first row reads its prior row from the previous block, which a CTA that claimed
// it earlier is producing: its last row is written back in place in R chunk by chunk and
// published through a progress counter (release: threadfence, then the counter; acquire:
// the counter, then an L2 load).  CTAs are persistent and claim the blocks in order, so a
// block only ever waits for a block that is already running: no deadlock, and an image's
// blocks run as a pipeline over several SMs (a 1080p image is 9 blocks).
constexpr int kPriorBatch = 8;
#ifndef TP_PNG_ACQREL  // 1: ld.acquire / st.release on the progress counters instead of fences
#define TP_PNG_ACQREL 1
#endif
#ifndef TP_PNG_RELEASE_BATCH
#define TP_PNG_RELEASE_BATCH 1
#endif

template <int BPP>
__device__ void unfilter_block(const PDesc& d, int blk, uint8_t* __restrict__ r,
                               uint8_t* __restrict__ o, const uint8_t* pal,
                               Chunk (*xch)[kUnfilterRows], Chunk* pbuf,
                               int* __restrict__ progress, int item, bool& bad_filter,
                               bool& bad_pal) {
  const int tid = threadIdx.x;
  const int W = d.width, H = d.height;
  const bool is_p = d.ctype == 3;
  const int64_t rowbytes = static_cast<int64_t>(W) * BPP, S = d.r_stride;
  const int nch = static_cast<int>((rowbytes + kCh - 1) / kCh);
  const uint8_t* fbytes = r;
  uint8_t* rows_base = r + r_filter_bytes(H);
  const int g0 = blk * kUnfilterRows;
  const int rows = min(kUnfilterRows, H - g0);
  const bool last_blk = g0 + rows >= H;
  const Chunk zero = Chunk();
  const int y = g0 + tid;
  const bool has_row = tid < rows;
  uint8_t* row = rows_base + static_cast<int64_t>(y) * S;
  const uint32_t ft = has_row ? fbytes[y] : 0u;
  if (ft > 4) bad_filter = true;
  const uint32_t m1 = 0u - (ft == 1), m2 = 0u - (ft == 2), m3 = 0u - (ft == 3), m4 = 0u - (ft == 4);
  const uint8_t* prior = y > 0 ? row - S : nullptr;  // (thread 0) the previous block's last row
  const volatile int* prior_progress = progress + item - 1;
  Chunk up_prev = zero, rec_prev = zero, fnext = zero;
  // own row: plain (L1-cached) loads -- 8 chunks per line; only this thread ever writes
  // it, after reading
  if (has_row) fnext = *reinterpret_cast<const Chunk*>(row);
  uint8_t* orow = o + static_cast<int64_t>(y) * W * 3;
  const bool oal = (reinterpret_cast<uintptr_t>(orow) & (kCh - 1)) == 0;
  const int steps = nch + rows - 1;
  for (int t = 0; t < steps; ++t) {
    const int i = t - tid;
    if (has_row && i >= 0 && i < nch) {
      const Chunk f = fnext;
      if (i + 1 < nch) fnext = reinterpret_cast<const Chunk*>(row)[i + 1];
      Chunk up = zero;
      if (tid == 0) {
        if (prior) {
          // the previous block's last row, kPriorBatch chunks at a time: one wait and one
          // L2 round trip per batch instead of per step (the block lags a few steps more)
          if (i % kPriorBatch == 0) {
            const int need = min(i + kPriorBatch, nch);
#if TP_PNG_ACQREL
            // acquire load: the chunks written before the counter are visible after it
            for (;;) {
              int v;
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(prior_progress) : "memory");
              if (v >= need) break;
              __nanosleep(32);
            }
#else
            while (*prior_progress < need) __nanosleep(32);
            __threadfence();  // acquire: the chunks were written before the counter
#endif
#pragma unroll
            for (int q = 0; q < kPriorBatch; ++q)
              if (i + q < nch) pbuf[q] = chunk_ldcg(reinterpret_cast<const Chunk*>(prior) + i + q);
          }
          up = pbuf[i % kPriorBatch];
        }
      } else {
        up = xch[(t - 1) & 1][tid - 1];
      }
      const int64_t x0 = kCh * static_cast<int64_t>(i);
      // one path per filter type (TP_PNG_UNFILTER_SPLIT): a warp runs the paths of the
      // types its 32 rows use -- photo-like PNGs mix mostly Sub and Up, whose paths are a
      // few operations per byte (Up: four byte-wise adds per chunk) -- instead of every
      // predictor for every byte
      uint32_t rb[kCh];
      Chunk rec;
#if TP_PNG_UNFILTER_SPLIT
      auto prev_a = [&](int j) -> uint32_t {  // recon[x - bpp] for j < BPP
        return x0 ? byte_at(rec_prev, kCh + j - BPP) : 0u;
      };
      auto prev_c = [&](int j) -> uint32_t {
        return x0 ? byte_at(up_prev, kCh + j - BPP) : 0u;
      };
      if (ft == 2) {
        uint32_t rw[kChunkWords];
#pragma unroll
        for (int q = 0; q < kChunkWords; ++q) rw[q] = __vadd4(CV::w(f, q), CV::w(up, q));
        rec = CV::make(rw);
#pragma unroll
        for (int j = 0; j < kCh; ++j) rb[j] = byte_at(rec, j);
      } else {
        if (ft == 1) {
#pragma unroll
          for (int j = 0; j < kCh; ++j)
            rb[j] = (byte_at(f, j) + (j >= BPP ? rb[j - BPP] : prev_a(j))) & 255u;
        } else if (ft == 3) {
#pragma unroll
          for (int j = 0; j < kCh; ++j) {
            const uint32_t a = j >= BPP ? rb[j - BPP] : prev_a(j);
            rb[j] = (byte_at(f, j) + ((a + byte_at(up, j)) >> 1)) & 255u;
          }
        } else if (ft == 4) {
#pragma unroll
          for (int j = 0; j < kCh; ++j) {
            const uint32_t a = j >= BPP ? rb[j - BPP] : prev_a(j);
            const uint32_t c = j >= BPP ? byte_at(up, j - BPP) : prev_c(j);
            const uint32_t b = byte_at(up, j);
            const int pp = static_cast<int>(a + b) - static_cast<int>(c);
            const int pa = abs(pp - static_cast<int>(a)), pb = abs(pp - static_cast<int>(b)),
                      pc = abs(pp - static_cast<int>(c));
            rb[j] = (byte_at(f, j) + ((pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c))) & 255u;
          }
        } else {  // None (and > 4, flagged above: any bytes will do)
#pragma unroll
          for (int j = 0; j < kCh; ++j) rb[j] = byte_at(f, j);
        }
        uint32_t rw[kChunkWords];
#pragma unroll
        for (int q = 0; q < kChunkWords; ++q) rw[q] = pack4(rb + 4 * q);
        rec = CV::make(rw);
      }
      (void)m1;
      (void)m2;
      (void)m3;
      (void)m4;
#else
#pragma unroll
      for (int j = 0; j < kCh; ++j) {
        uint32_t a, c;
        if (j >= BPP) {
          a = rb[j - BPP];
          c = byte_at(up, j - BPP);
        } else {
          a = x0 ? byte_at(rec_prev, kCh + j - BPP) : 0u;
          c = x0 ? byte_at(up_prev, kCh + j - BPP) : 0u;
        }
        const uint32_t b = byte_at(up, j);
        const int pp = static_cast<int>(a + b) - static_cast<int>(c);
        const int pa = abs(pp - static_cast<int>(a)), pb = abs(pp - static_cast<int>(b)),
                  pc = abs(pp - static_cast<int>(c));
        const uint32_t pae = (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
        // branch-free: neighbouring rows (lanes) use different filter types
        const uint32_t pred = (a & m1) | (b & m2) | (((a + b) >> 1) & m3) | (pae & m4);
        rb[j] = (byte_at(f, j) + pred) & 255u;
      }
      {
        uint32_t rw[kChunkWords];
#pragma unroll
        for (int q = 0; q < kChunkWords; ++q) rw[q] = pack4(rb + 4 * q);
        rec = CV::make(rw);
      }
#endif
      const int nb = static_cast<int>(rowbytes - x0 < kCh ? rowbytes - x0 : kCh);
      if (BPP == 3) {
        uint8_t* dst = orow + x0;
        if (oal && nb == kCh) {
          chunk_stcs(reinterpret_cast<Chunk*>(dst), rec);
        } else {
#pragma unroll
          for (int j = 0; j < kCh; ++j)
            if (j < nb) dst[j] = static_cast<uint8_t>(rb[j]);
        }
      } else {
        uint32_t px[3 * kCh];
#pragma unroll
        for (int j = 0; j < kCh; ++j) {
          const uint32_t v = rb[j];
          if (is_p) {
            if (j < nb && static_cast<int>(v) >= d.pal_n) bad_pal = true;
            px[3 * j] = pal[3 * v];
            px[3 * j + 1] = pal[3 * v + 1];
            px[3 * j + 2] = pal[3 * v + 2];
          } else {
            px[3 * j] = px[3 * j + 1] = px[3 * j + 2] = v;
          }
        }
        uint8_t* dst = orow + 3 * x0;
        if (oal && nb == kCh) {
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            uint32_t pw[kChunkWords];
#pragma unroll
            for (int e = 0; e < kChunkWords; ++e) pw[e] = pack4(px + q * kCh + 4 * e);
            chunk_stcs(reinterpret_cast<Chunk*>(dst) + q, CV::make(pw));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 3 * kCh; ++j)
            if (j < 3 * nb) dst[j] = static_cast<uint8_t>(px[j]);
        }
      }
      if (tid == rows - 1 && !last_blk) {  // the next block's first row reads it
        chunk_stcg(reinterpret_cast<Chunk*>(row) + i, rec);
#if TP_PNG_RELEASE_BATCH
        // published once per kPriorBatch chunks (the reader waits for whole batches): a
        // fence per chunk held this warp -- and through the step barrier the whole CTA --
        // for a memory-barrier round trip every step
        if ((i + 1) % kPriorBatch == 0 || i + 1 == nch) {
#if TP_PNG_ACQREL
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(progress + item), "r"(i + 1) : "memory");
#else
          __threadfence();  // release: the chunks before the counter
          atomicExch(progress + item, i + 1);
#endif
        }
#else
        __threadfence();  // release: the chunk before the counter
        atomicExch(progress + item, i + 1);
#endif
      }
      xch[t & 1][tid] = rec;
      up_prev = up;
      rec_prev = rec;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kUnfilterRows)
    k_png_unfilter(const PDesc* __restrict__ desc, int n, uint8_t* __restrict__ R,
                   uint8_t* __restrict__ out, int32_t* __restrict__ img_status,
                   int* __restrict__ progress, int n_items) {
  __shared__ Chunk xch[2][kUnfilterRows];
  __shared__ Chunk pbuf[kPriorBatch];
  __shared__ uint8_t pal[768];
  __shared__ int cur;
  int* claim = progress + n_items;
  while (true) {
    __syncthreads();  // the previous item's readers of `cur` and `pal` are done
    if (threadIdx.x == 0) cur = atomicAdd(claim, 1);
    __syncthreads();
    const int item = cur;
    if (item >= n_items) break;
    const int k = blk_image(desc, n, item);
    const PDesc& d = desc[k];
    // Skip only on what earlier kernels decided: the flags this kernel sets (filter,
    // palette) appear while the image's blocks run, and a block must never skip while a
    // later block of its image waits for it.
    if (d.n_units == 0 || (img_status[k] & ~(kImgFilter | kImgPalette)) != kImgOk) continue;
    if (d.ctype == 3)
      for (int i = threadIdx.x; i < 768; i += blockDim.x) pal[i] = d.pal[i];
    __syncthreads();
    bool bad_filter = false, bad_pal = false;
    if (d.bpp == 3)
      unfilter_block<3>(d, item - d.blk_base, R + d.r_off, out + d.out_off, pal, xch, pbuf,
                        progress, item, bad_filter, bad_pal);
    else
      unfilter_block<1>(d, item - d.blk_base, R + d.r_off, out + d.out_off, pal, xch, pbuf,
                        progress, item, bad_filter, bad_pal);
    if (bad_filter) atomicOr(img_status + k, kImgFilter);
    if (bad_pal) atomicOr(img_status + k, kImgPalette);
  }
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
  uint32_t* stage = reinterpret_cast<uint32_t*>(work + totals[11]);
  cudaMemsetAsync(d_status, 0, sizeof(int32_t) * n, s);
  // TP_PNG_DEBUG_SYNC=1: synchronise after every kernel and name the one that failed
  static const bool debug_sync = std::getenv("TP_PNG_DEBUG_SYNC") != nullptr;
  auto dbg = [&](const char* what) -> int {
    if (!debug_sync) return TP_OK;
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return tp::set_error(TP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return TP_OK;
  };
#define TP_PNG_DBG(name) \
  do {                   \
    const int rc_ = dbg(name); \
    if (rc_ != TP_OK) return rc_; \
  } while (0)
  if (U > 0) {
    // finder warps per unit: split the scans while the units alone leave the GPU short of
    // warps (small batches: latency-bound), one per unit when they fill it (64 1080p
    // PNGs, 6,000 units: the extra scanning then costs more than it hides)
    const int sms = std::max(1, tp::device_sm_count());
    const int parts = std::max(1, std::min(kFindParts, (sms * 48) / std::max(U, 1)));
    int* sched = reinterpret_cast<int*>(work + totals[13]);  // (the unfilter's progress area)
    k_png_find_init<<<(std::max(U, kSchedInts) + 255) / 256, 256, 0, s>>>(stage, U, sched);
    TP_PNG_DBG("k_png_find_init");
    const int64_t find_warps = static_cast<int64_t>(U) * parts;
    int64_t find_ctas = (find_warps + kFindThreads / 32 - 1) / (kFindThreads / 32);
    if (TP_PNG_FIND_DYN) {  // one resident wave: the warps take the items in turn
      static int find_occ = 0;
      if (find_occ == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&find_occ, k_png_find, kFindThreads, 0);
      find_ctas = std::min<int64_t>(find_ctas, static_cast<int64_t>(std::max(find_occ, 1)) * sms);
    }
    k_png_find<<<static_cast<int>(find_ctas), kFindThreads, 0, s>>>(d_payload, desc, n, units, U,
                                                                    stage, parts, sched);
                 TP_PNG_DBG("k_png_find");
    k_png_find_select<<<(U + 255) / 256, 256, 0, s>>>(units, stage, U, parts,
                                                      static_cast<int>(totals[15]));
                                                      TP_PNG_DBG("k_png_find_select");
    int64_t inflate_ctas = (U + kInflateWarps - 1) / kInflateWarps;
    if (TP_PNG_INFLATE_DYN) {
      static int inflate_occ = 0;
      if (inflate_occ == 0)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&inflate_occ, k_png_inflate, 32 * kInflateWarps, 0);
      inflate_ctas = std::min<int64_t>(inflate_ctas, static_cast<int64_t>(std::max(inflate_occ, 1)) * sms);
    }
    for (int r = 0; r < kRounds; ++r) {
      k_png_inflate<<<static_cast<int>(inflate_ctas), 32 * kInflateWarps, 0, s>>>(
          d_payload, desc, n, units, U, toks, stage, d_status, sched, r);
          TP_PNG_DBG("k_png_inflate");
      k_png_chain<<<n, 32, 0, s>>>(desc, n, units, d_status, r);
      TP_PNG_DBG("k_png_chain");
    }
    uint32_t* M = reinterpret_cast<uint32_t*>(work + totals[9]);
    k_png_expand<<<(U + 7) / 8, 256, 0, s>>>(d_payload, desc, n, units, U, toks, T, M, d_status);
    TP_PNG_DBG("k_png_expand");
    if (totals[10] > 0)
      k_png_final<<<static_cast<int>(totals[10]), 256, 0, s>>>(desc, n, T, R, d_status);
      TP_PNG_DBG("k_png_final");
    k_png_window<<<n, 1024, 0, s>>>(desc, n, units, T, M, R, d_status);
    TP_PNG_DBG("k_png_window");
    if (totals[12] > 0) {
      unsigned long long* acc = reinterpret_cast<unsigned long long*>(work + totals[14]);
      cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 2 * n, s);
      k_png_adler_rows<<<static_cast<int>(totals[12]), kAdlerThreads, 0, s>>>(
          desc, n, units, R, d_status, acc, static_cast<int>(totals[12]));
          TP_PNG_DBG("k_png_adler_rows");
      k_png_adler_check<<<(n + 255) / 256, 256, 0, s>>>(d_payload, desc, n, units, acc, d_status);
      TP_PNG_DBG("k_png_adler_check");
    }
    const int n_items = static_cast<int>(totals[12]);
    if (n_items > 0) {
      int* progress = reinterpret_cast<int*>(work + totals[13]);
      cudaMemsetAsync(progress, 0, sizeof(int) * (n_items + 1), s);
      const int sms = std::max(1, tp::device_sm_count());
      k_png_unfilter<<<std::min(n_items, sms * 8), kUnfilterRows, 0, s>>>(
          desc, n, R, d_out, d_status, progress, n_items);
          TP_PNG_DBG("k_png_unfilter");
    }
  }
  return tp::check_launch("tp_png_decode");
}
