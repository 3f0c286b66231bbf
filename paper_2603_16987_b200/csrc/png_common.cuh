// Device PNG decoder (K8): shared layouts (host describe <-> device kernels).
#pragma once

#include <stdint.h>

namespace tp {
namespace png {

// Block-finder chunk: unit u of an image starts at the first deflate block header found
// in bits [u * kUnitBits, (u + 1) * kUnitBits) of its zlib stream (unit 0 at bit 16,
// right after the two-byte zlib header).  One warp inflates one unit.  The finder scans
// from the unit's start to the first header, so its work is about half a block per
// unit: units a few blocks long (zlib's blocks are 16-32K symbols, ~12-24 KB of a
// photo-like PNG) keep the scan to a fraction of the stream; the warp decodes each block
// 32 subsequences at a time.
constexpr int64_t kUnitBits = 8 * 49152;
constexpr int kWindow = 32768;  // deflate's back-reference window

// Unit states (PUnit::status): 0 ok; the rest send the image to the host decoder.
enum : int32_t {
  kUnitOk = 0,
  kUnitBadCode = 1,      // invalid / over-subscribed / incomplete code, bad symbol
  kUnitOverrun = 2,      // read past the stream, or tokens past the unit's capacity
  kUnitBadStored = 3,    // stored block LEN / NLEN mismatch
  kUnitBadDistance = 4,  // back reference before the image start
  kUnitTokens = 5,       // tokens past the unit's capacity (its decode passed the next
                         // start, or the stream spends < 2 bits per token)
};

// Image states (d_status): 0 ok; nonzero: decode this one on the host (Pillow).  The
// chain kernel sets one of the first four; the later kernels OR in the flags.
enum : int32_t {
  kImgOk = 0,
  kImgInflate = 1,     // a unit failed (see kUnit*)
  kImgChain = 2,       // units do not chain after kRounds rounds
  kImgLength = 3,      // inflated length differs from height * (1 + rowbytes)
  kImgNotFinal = 4,    // the stream ends without a final block
  kImgDistance = 16,   // a back reference before the image start
  kImgFilter = 32,     // filter type > 4
  kImgPalette = 64,    // palette index beyond the PLTE entries
  kImgAdler = 128,     // Adler-32 trailer present and wrong (Pillow's zlib raises)
};

// Inflate rounds: a header the finder accepted that is not a real block start is caught
// when the preceding unit's decode passes it; that unit is then re-decoded up to the next
// start in the following round.
constexpr int kRounds = 6;  // later rounds cost a few microseconds when nothing is dirty

// Per image, written by tp_png_describe and uploaded with the compressed bytes.
struct __align__(16) PDesc {
  int64_t in_off;     // zlib stream (header included) in the payload, 4-byte aligned
  int64_t in_bits;    // bits of the zlib stream (deflate data starts at bit 16)
  int64_t raw_off;    // inflated scanlines: offset in the T (u16) / R (u8) workspaces
  int64_t raw_len;    // height * (1 + width * bpp)
  int64_t out_off;    // RGB HWC uint8 in the output buffer
  int64_t tok_off;    // token workspace (u32) of this image: in_bits / 2 + slack
  int32_t width, height;
  int32_t bpp;        // bytes per pixel of the scanlines: 1 (L, P) or 3 (RGB)
  int32_t ctype;      // PNG colour type: 0 (L), 2 (RGB), 3 (P)
  int32_t unit_base;  // first unit of this image
  int32_t n_units;
  int32_t pal_n;      // PLTE entries (P)
  int32_t row_base;   // first row of this image in the batch's row numbering
  int32_t blk_base;   // first unfilter row block of this image (kUnfilterRows rows each)
  int32_t pad3_;
  int64_t r_off;      // R workspace: filter bytes (align16(height)), then the rows
  int64_t r_stride;   // R row stride: rowbytes rounded up to 16 (rows 16-byte aligned)
  uint8_t pal[768];   // PLTE (P)
};

// Per unit (workspace), filled by the finder and the inflate kernel.
// Unit starts and ends are canonical block positions: the header bit of a dynamic or
// fixed block, but for a stored block the byte boundary of its LEN field (the header bits
// and zero padding before it can begin at several bit positions that all look alike).
struct __align__(16) PUnit {
  int64_t start;    // first bit (relative to the zlib stream); -1: no header found
  int64_t end;      // bit after the unit's last block
  int64_t out_len;  // inflated bytes
  int64_t out_off;  // first inflated byte (relative to raw_off), by the chain scan
  int32_t ntok;     // tokens written
  int32_t status;   // kUnit*
  int32_t final_;   // the unit ended with the BFINAL block
  int32_t dirty;    // (re)decode in the next inflate round
  int32_t stored;   // start is the LEN field of a stored block (its header not read)
  int32_t nmark;    // bytes of this unit that are window markers (listed by expand)
  int32_t fixups;   // diagnostics: lane re-decodes in the inflate's rounds
  int32_t rounds;   // diagnostics: inflate rounds
  int64_t final_end;  // (an image's first unit) bit after the final block, by the chain
  int64_t redo;       // (an image's first unit) the chain dropped a start this round
};

// Unfilter work item: a block of consecutive scanlines of one image, one thread each.
#ifndef TP_PNG_UNFILTER_ROWS  // rows per unfilter block (= threads per unfilter CTA)
#define TP_PNG_UNFILTER_ROWS 128
#endif
constexpr int kUnfilterRows = TP_PNG_UNFILTER_ROWS;

// tp_png_describe's totals[16]: [0] units, [1] tokens, [2] raw bytes (T entries),
// [3..6] byte offsets of units / tokens / T / R, [7] workspace bytes, [8] R bytes,
// [9] marker lists' byte offset (u32 image-relative positions; unit u's list starts at
// the index of its first byte, raw_off + out_off), [10] rows in the batch, [11] byte
// offset of the inflate warps' token staging (kStageBytesPerUnit per unit), [12] unfilter
// row blocks in the batch, [13] byte offset of their progress counters (int32 each, plus
// one claim counter), [14] byte offset of the Adler-32 sums (2 x u64 per image), [15]
// test hooks set by the caller (bit 0: false finder starts, see k_png_find_select)
constexpr int kTotals = 16;
#ifndef TP_PNG_SUB
#define TP_PNG_SUB 512
#endif
constexpr int kSubBits = TP_PNG_SUB;  // bits per lane per inflate round
constexpr int64_t kStageBytesPerUnit = 32 * (kSubBits + 64) * 4;

// R (inflated scanlines) per image: the filter-type bytes, then each row's rowbytes
// data bytes at a 16-byte aligned stride (vector loads and stores in the unfilter)
__host__ __device__ inline int64_t r_filter_bytes(int64_t h) { return (h + 15) / 16 * 16; }

// Token (u32), what the inflate kernel writes and the expand kernel turns into bytes:
//   type 0 (bits 31..30 = 00): 1-3 literals, count in bits 25..24, bytes in 7..0, 15..8, 23..16
//   type 1 (01): match, length - 3 in bits 23..16, distance - 1 in bits 15..0
//   type 2 (10): stored block, byte offset of its data in the zlib stream in bits 29..0;
//                LEN is the 16-bit word 4 bytes before the data
constexpr uint32_t kTokMatch = 1u << 30, kTokStored = 2u << 30;

}  // namespace png
}  // namespace tp
