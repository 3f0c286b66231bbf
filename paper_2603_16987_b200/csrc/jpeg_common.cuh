// Device JPEG decoder: shared layouts (host describe <-> device kernels).
#pragma once

#include <stdint.h>

namespace tp {
namespace jpeg {

constexpr int kMaxComps = 3;
constexpr int kMaxBlocksPerMcu = 6;  // 4:2:0: Y0 Y1 Y2 Y3 Cb Cr
constexpr int kFastBits = 11;  // lookahead: 99.4% of the symbols of a corpus-like JPEG

// One Huffman table, decode-ready (T.81 C.2 canonical codes).
struct __align__(16) JHuff {
  uint16_t fast[1 << kFastBits];  // next kFastBits bits -> (len << 8) | symbol; 0: longer code
  int32_t maxcode[18];            // largest code of length l, -1 when none
  int32_t valoff[18];             // symbol index of code c of length l: valoff[l] + c
  uint8_t vals[256];
};

// Per image: everything the kernels need; written by tp_jpeg_describe on the host and
// uploaded with the compressed bytes.
struct __align__(16) JDesc {
  int64_t raw_off;     // entropy-coded bytes (stuffed, with RST markers) in the payload
  int64_t clean_off;   // workspace: unstuffed bytes, restart intervals back to back
  int64_t seg_off;     // workspace: int32 seg_start[n_seg + 1], int32 sub_prefix[n_seg + 1]
  int64_t slot_base;   // first subsequence slot of this image
  int64_t coef_off;    // workspace: int16 coefficients [n_blocks][64] (natural order)
  int64_t block_base;  // global index of this image's first block (IDCT grid)
  int64_t row_base;    // global index of this image's first output row (colour grid)
  int64_t out_off;     // RGB HWC uint8 in the output buffer
  int64_t plane_off[kMaxComps];  // workspace: uint8 component planes
  int64_t chunk_base;  // first unstuff chunk (32 KB of entropy-coded bytes) of this image
  int32_t raw_len;
  int32_t n_slots;     // slots reserved (an upper bound)
  int32_t n_seg;       // restart intervals
  int32_t ri;          // MCUs per restart interval
  int32_t width, height, ncomp, mcux, mcuy, bmcu, hmax, vmax;
  int32_t n_blocks;
  int32_t n_chunks;
  int32_t plane_w[kMaxComps], plane_h[kMaxComps];  // block-padded
  int32_t ds_w[kMaxComps], ds_h[kMaxComps];        // real (downsampled) samples
  int32_t comp_h[kMaxComps], comp_v[kMaxComps];
  int32_t comp_td[kMaxComps], comp_ta[kMaxComps], comp_tq[kMaxComps];
  int8_t slot_comp[kMaxBlocksPerMcu], slot_bh[kMaxBlocksPerMcu], slot_bv[kMaxBlocksPerMcu];
  int8_t pad_[2];
  // natural order, per component, as libjpeg's ISLOW_MULT_TYPE (short) holds them:
  // (int16) quantval, sign-extended
  alignas(16) int32_t quant[kMaxComps][64];
  JHuff dc[2], ac[2];
};

}  // namespace jpeg
}  // namespace tp
