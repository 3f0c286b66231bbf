// K7 host side: JPEG marker parsing and per-image device descriptors.
//
// The reference decodes every payload with Pillow (imgproc.py:213-229), i.e. with the
// libjpeg-turbo Pillow bundles.  This file restates the marker syntax of ITU-T T.81
// Annex B and libjpeg's table derivation (jdhuff.c jpeg_make_d_derived_tbl) so the
// device decoder (jpeg.cu) can run the entropy decode, IDCT, upsampling and colour
// conversion; it decides which payloads the device takes (baseline Huffman, 8-bit,
// 1 or 3 components, 4:4:4 / 4:2:2 / 4:2:0, one interleaved scan) and leaves the rest
// (TP_JPEG_UNSUPPORTED) to the host decoder, exactly as the reference would decode them.
// Host code only.

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "jpeg_common.cuh"
#include "tileprep.h"
#include "tp_common.cuh"

namespace {

using tp::jpeg::JDesc;
using tp::jpeg::JHuff;

int status(TpJpegInfo* info, int code, const char* fmt, ...) {
  info->status = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(info->message, sizeof(info->message), fmt, ap);
  va_end(ap);
  return TP_OK;
}

const int kZigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                         12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                         35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                         58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// jdhuff.c jpeg_make_d_derived_tbl: canonical codes, maxcode / valoffset, 9-bit lookahead
bool build_huff(const uint8_t* bits, const uint8_t* vals, bool is_dc, JHuff* t) {
  int huffsize[257];
  unsigned huffcode[257];
  int p = 0;
  for (int l = 1; l <= 16; ++l)
    for (int i = 0; i < bits[l - 1]; ++i) {
      if (p >= 256) return false;
      huffsize[p++] = l;
    }
  huffsize[p] = 0;
  const int numsymbols = p;
  unsigned code = 0;
  int si = huffsize[0];
  p = 0;
  while (huffsize[p]) {
    while (huffsize[p] == si) huffcode[p++] = code++;
    if (code >= (1u << si)) return false;  // JERR_BAD_HUFF_TABLE
    code <<= 1;
    ++si;
  }
  p = 0;
  for (int l = 1; l <= 16; ++l) {
    if (bits[l - 1]) {
      t->valoff[l] = p - static_cast<int>(huffcode[p]);
      p += bits[l - 1];
      t->maxcode[l] = static_cast<int32_t>(huffcode[p - 1]);
    } else {
      t->maxcode[l] = -1;
      t->valoff[l] = 0;
    }
  }
  t->maxcode[0] = -1;
  t->valoff[0] = 0;
  t->maxcode[17] = 0x7FFFFFFF;
  t->valoff[17] = 0;
  memset(t->fast, 0, sizeof(t->fast));
  for (p = 0; p < numsymbols; ++p) {
    const int l = huffsize[p];
    if (l > tp::jpeg::kFastBits) break;
    const unsigned look = huffcode[p] << (tp::jpeg::kFastBits - l);
    for (unsigned c = 0; c < (1u << (tp::jpeg::kFastBits - l)); ++c)
      t->fast[look + c] = static_cast<uint16_t>((l << 8) | vals[p]);
  }
  memset(t->vals, 0, sizeof(t->vals));
  for (p = 0; p < numsymbols; ++p) {
    if (is_dc && vals[p] > 11) return false;  // DC categories beyond 8-bit baseline
    t->vals[p] = vals[p];
  }
  return true;
}

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace

extern "C" {

TP_API int tp_jpeg_parse(const uint8_t* d, int64_t n, TpJpegInfo* info) {
  if (!d || !info || n < 0) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_jpeg_parse: null");
  memset(info, 0, sizeof(*info));
  if (n < 4 || d[0] != 0xFF || d[1] != 0xD8) return status(info, TP_JPEG_CORRUPT, "no SOI");
  int64_t pos = 2;
  bool jfif = false, sof = false;
  int adobe = -1;
  while (pos < n) {
    if (d[pos] != 0xFF) return status(info, TP_JPEG_CORRUPT, "expected a marker at %lld",
                                      static_cast<long long>(pos));
    while (pos < n && d[pos] == 0xFF) ++pos;
    if (pos >= n) break;
    const int m = d[pos++];
    if (m == 0xD8 || (m >= 0xD0 && m <= 0xD7) || m == 0x01) continue;
    if (m == 0xD9) return status(info, TP_JPEG_CORRUPT, "EOI before SOS");
    if (pos + 2 > n) break;
    const int len = (d[pos] << 8) | d[pos + 1];
    if (len < 2 || pos + len > n) return status(info, TP_JPEG_CORRUPT, "bad segment length");
    const uint8_t* s = d + pos + 2;
    const int sl = len - 2;
    if (m == 0xC0 || m == 0xC1) {
      if (sl < 6) return status(info, TP_JPEG_CORRUPT, "short SOF");
      if (s[0] != 8) return status(info, TP_JPEG_UNSUPPORTED, "%d-bit samples", s[0]);
      info->height = (s[1] << 8) | s[2];
      info->width = (s[3] << 8) | s[4];
      info->ncomp = s[5];
      if (info->ncomp != 1 && info->ncomp != 3)
        return status(info, TP_JPEG_UNSUPPORTED, "%d components", info->ncomp);
      if (sl < 6 + 3 * info->ncomp) return status(info, TP_JPEG_CORRUPT, "short SOF");
      if (info->width < 1 || info->height < 1)
        return status(info, TP_JPEG_UNSUPPORTED, "zero-size frame (DNL)");
      // block / MCU indices stay below 2^22 (the kernels' float-reciprocal divisions)
      if (static_cast<int64_t>(info->width) * info->height > (int64_t(1) << 27))
        return status(info, TP_JPEG_UNSUPPORTED, "more than 2^27 pixels");
      for (int c = 0; c < info->ncomp; ++c) {
        info->comp_id[c] = s[6 + 3 * c];
        info->comp_h[c] = s[7 + 3 * c] >> 4;
        info->comp_v[c] = s[7 + 3 * c] & 15;
        info->comp_tq[c] = s[8 + 3 * c];
        if (info->comp_tq[c] > 3) return status(info, TP_JPEG_CORRUPT, "bad quant table id");
      }
      sof = true;
    } else if (m >= 0xC2 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC) {
      return status(info, TP_JPEG_UNSUPPORTED, "SOF%d (not baseline Huffman)", m - 0xC0);
    } else if (m == 0xDB) {
      int p = 0;
      while (p < sl) {
        const int pq = s[p] >> 4, tq = s[p] & 15;
        ++p;
        if (tq > 3 || p + (pq ? 128 : 64) > sl) return status(info, TP_JPEG_CORRUPT, "bad DQT");
        for (int i = 0; i < 64; ++i) {
          const int v = pq ? (s[p + 2 * i] << 8) | s[p + 2 * i + 1] : s[p + i];
          info->qt[tq][kZigzag[i]] = static_cast<uint16_t>(v);
        }
        p += pq ? 128 : 64;
        info->qt_mask |= 1 << tq;
      }
    } else if (m == 0xC4) {
      int p = 0;
      while (p < sl) {
        const int tc = s[p] >> 4, th = s[p] & 15;
        if (p + 17 > sl) return status(info, TP_JPEG_CORRUPT, "bad DHT");
        int cnt = 0;
        for (int i = 0; i < 16; ++i) cnt += s[p + 1 + i];
        if (cnt > 256 || p + 17 + cnt > sl) return status(info, TP_JPEG_CORRUPT, "bad DHT");
        if (th > 1 || tc > 1)
          return status(info, TP_JPEG_UNSUPPORTED, "Huffman table class %d id %d", tc, th);
        uint8_t* bits = tc ? info->ac_bits[th] : info->dc_bits[th];
        uint8_t* vals = tc ? info->ac_vals[th] : info->dc_vals[th];
        memcpy(bits, s + p + 1, 16);
        memset(vals, 0, 256);
        memcpy(vals, s + p + 17, cnt);
        (tc ? info->ac_mask : info->dc_mask) |= 1 << th;
        p += 17 + cnt;
      }
    } else if (m == 0xDD) {
      if (sl < 2) return status(info, TP_JPEG_CORRUPT, "bad DRI");
      info->restart_interval = (s[0] << 8) | s[1];
    } else if (m == 0xE0 && sl >= 5 && memcmp(s, "JFIF\0", 5) == 0) {
      jfif = true;
    } else if (m == 0xEE && sl >= 12 && memcmp(s, "Adobe", 5) == 0) {
      adobe = s[11];
    } else if (m == 0xDA) {
      if (!sof) return status(info, TP_JPEG_CORRUPT, "SOS before SOF");
      const int ns = sl > 0 ? s[0] : 0;
      if (sl < 1 + 2 * ns + 3) return status(info, TP_JPEG_CORRUPT, "short SOS");
      if (ns != info->ncomp)
        return status(info, TP_JPEG_UNSUPPORTED, "multi-scan sequential JPEG");
      for (int c = 0; c < ns; ++c) {
        if (s[1 + 2 * c] != info->comp_id[c])
          return status(info, TP_JPEG_UNSUPPORTED, "scan component order differs from the frame");
        info->comp_td[c] = s[2 + 2 * c] >> 4;
        info->comp_ta[c] = s[2 + 2 * c] & 15;
        if (info->comp_td[c] > 1 || info->comp_ta[c] > 1)
          return status(info, TP_JPEG_UNSUPPORTED, "Huffman table id > 1");
      }
      if (s[1 + 2 * ns] != 0 || s[2 + 2 * ns] != 63 || s[3 + 2 * ns] != 0)
        return status(info, TP_JPEG_UNSUPPORTED, "spectral selection / approximation");
      info->scan_off = pos + len;
      int64_t end = n - 2;
      while (end >= info->scan_off && !(d[end] == 0xFF && d[end + 1] == 0xD9)) --end;
      if (end < info->scan_off) return status(info, TP_JPEG_CORRUPT, "no EOI after the scan");
      info->scan_len = end - info->scan_off;
      for (int c = 0; c < info->ncomp; ++c) {
        if (!(info->qt_mask >> info->comp_tq[c] & 1) || !(info->dc_mask >> info->comp_td[c] & 1) ||
            !(info->ac_mask >> info->comp_ta[c] & 1))
          return status(info, TP_JPEG_CORRUPT, "missing table");
      }
      if (info->ncomp == 1) {
        if (info->comp_h[0] != 1 || info->comp_v[0] != 1)
          return status(info, TP_JPEG_UNSUPPORTED, "subsampled single-component scan");
      } else {
        // jdapimin.c default_decompress_parms: JFIF -> YCbCr; Adobe transform 1 -> YCbCr,
        // 0 -> RGB; neither: component ids 'R','G','B' -> RGB, else YCbCr
        if (!jfif && adobe >= 0 && adobe != 1)
          return status(info, TP_JPEG_UNSUPPORTED, "Adobe transform %d colour space", adobe);
        if (!jfif && adobe < 0 && info->comp_id[0] == 82 && info->comp_id[1] == 71 &&
            info->comp_id[2] == 66)
          return status(info, TP_JPEG_UNSUPPORTED, "RGB colour space");
        const bool chroma11 = info->comp_h[1] == 1 && info->comp_v[1] == 1 &&
                              info->comp_h[2] == 1 && info->comp_v[2] == 1;
        const int yh = info->comp_h[0], yv = info->comp_v[0];
        if (!chroma11 || !((yh == 1 && yv == 1) || (yh == 2 && yv == 1) || (yh == 2 && yv == 2)))
          return status(info, TP_JPEG_UNSUPPORTED, "sampling factors other than 4:4:4 / 4:2:2 / 4:2:0");
      }
      return status(info, TP_JPEG_OK, "ok");
    }
    pos += len;
  }
  return status(info, TP_JPEG_CORRUPT, "no SOS");
}

TP_API int64_t tp_jpeg_desc_bytes(void) { return static_cast<int64_t>(sizeof(JDesc)); }

// Workspace: [header 4 KB: step counters] [per slot: exit int64 | blocks | err | bstart |
// lastproc | changed] [per image: clean bytes | seg table | coefficients | planes]
TP_API int64_t tp_jpeg_describe(const TpJpegInfo* infos, int32_t n, const int64_t* raw_off,
                                const int64_t* out_off, int32_t sub_bits, void* desc_out,
                                int64_t* totals) {
  if (n < 0 || (n > 0 && (!infos || !raw_off || !out_off || !desc_out)) || !totals ||
      sub_bits < 64 || (sub_bits & 31))
    return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_jpeg_describe: bad arguments");
  JDesc* descs = static_cast<JDesc*>(desc_out);
  int64_t slots = 0, blocks = 0, rows = 0, chunks = 0;
  constexpr int64_t kChunk = 32768;  // jpeg.cu
  for (int k = 0; k < n; ++k) {
    const TpJpegInfo& in = infos[k];
    JDesc& j = descs[k];
    memset(&j, 0, sizeof(j));
    j.slot_base = slots;  // bases stay monotone across skipped images (kernel binary searches)
    j.block_base = blocks;
    j.row_base = rows;
    j.chunk_base = chunks;
    if (in.status != TP_JPEG_OK) continue;  // decoded on the host
    if (raw_off[k] & 3)
      return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "raw_off[%d] not 4-byte aligned", k);
    j.raw_off = raw_off[k];
    j.raw_len = static_cast<int32_t>(in.scan_len);
    j.width = in.width;
    j.height = in.height;
    j.ncomp = in.ncomp;
    int hmax = 1, vmax = 1;
    for (int c = 0; c < in.ncomp; ++c) {
      hmax = hmax > in.comp_h[c] ? hmax : in.comp_h[c];
      vmax = vmax > in.comp_v[c] ? vmax : in.comp_v[c];
    }
    j.hmax = hmax;
    j.vmax = vmax;
    if (in.ncomp == 1) {
      j.mcux = (in.width + 7) / 8;
      j.mcuy = (in.height + 7) / 8;
      j.bmcu = 1;
      j.slot_comp[0] = 0;
    } else {
      j.mcux = (in.width + 8 * hmax - 1) / (8 * hmax);
      j.mcuy = (in.height + 8 * vmax - 1) / (8 * vmax);
      int b = 0;
      for (int c = 0; c < in.ncomp; ++c)
        for (int bv = 0; bv < in.comp_v[c]; ++bv)
          for (int bh = 0; bh < in.comp_h[c]; ++bh) {
            j.slot_comp[b] = static_cast<int8_t>(c);
            j.slot_bh[b] = static_cast<int8_t>(bh);
            j.slot_bv[b] = static_cast<int8_t>(bv);
            ++b;
          }
      j.bmcu = b;
    }
    const int64_t n_mcu = static_cast<int64_t>(j.mcux) * j.mcuy;
    j.ri = in.restart_interval > 0 ? in.restart_interval : static_cast<int32_t>(n_mcu);
    j.n_seg = static_cast<int32_t>((n_mcu + j.ri - 1) / j.ri);
    j.n_blocks = static_cast<int32_t>(n_mcu * j.bmcu);
    j.n_slots = static_cast<int32_t>((8 * static_cast<int64_t>(in.scan_len) + sub_bits - 1) / sub_bits +
                                     j.n_seg);
    for (int c = 0; c < in.ncomp; ++c) {
      const int hc = in.ncomp == 1 ? 1 : in.comp_h[c], vc = in.ncomp == 1 ? 1 : in.comp_v[c];
      j.comp_h[c] = in.comp_h[c];
      j.comp_v[c] = in.comp_v[c];
      j.comp_td[c] = in.comp_td[c];
      j.comp_ta[c] = in.comp_ta[c];
      j.comp_tq[c] = in.comp_tq[c];
      j.plane_w[c] = j.mcux * hc * 8;
      j.plane_h[c] = j.mcuy * vc * 8;
      j.ds_w[c] = static_cast<int32_t>((static_cast<int64_t>(in.width) * in.comp_h[c] + hmax - 1) / hmax);
      j.ds_h[c] = static_cast<int32_t>((static_cast<int64_t>(in.height) * in.comp_v[c] + vmax - 1) / vmax);
      for (int i = 0; i < 64; ++i) j.quant[c][i] = static_cast<int16_t>(in.qt[in.comp_tq[c]][i]);
    }
    for (int t = 0; t < 2; ++t) {
      if ((in.dc_mask >> t & 1) && !build_huff(in.dc_bits[t], in.dc_vals[t], true, &j.dc[t]))
        return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "image %d: bad DC Huffman table", k);
      if ((in.ac_mask >> t & 1) && !build_huff(in.ac_bits[t], in.ac_vals[t], false, &j.ac[t]))
        return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "image %d: bad AC Huffman table", k);
    }
    j.out_off = out_off[k];
    j.n_chunks = static_cast<int32_t>((in.scan_len + kChunk - 1) / kChunk);
    chunks += j.n_chunks;
    slots += j.n_slots;
    blocks += j.n_blocks;
    rows += j.height;
  }
  // workspace layout (zeroed by tp_jpeg_decode: the counters and the coefficients)
  int64_t w = 4096;                         // step counters
  w += 2 * align_up(8 * slots, 256);        // exit, entry
  w += align_up(16 * slots, 256);           // DC sums / predictors
  w += 5 * align_up(4 * slots, 256);        // blocks, err, errpos, bstart, claim
  w += align_up(8 * 7 * slots, 256);        // checkpoint states (jpeg.cu kCkpts = 7)
  w += align_up(16 * 7 * slots, 256);       // checkpoint accumulators
  totals[6] = w;                            // unstuff chunk counts
  w = align_up(w + 8 * chunks, 256);
  totals[3] = w;
  for (int k = 0; k < n; ++k) {
    JDesc& j = descs[k];
    if (infos[k].status != TP_JPEG_OK) continue;
    j.coef_off = w;
    w = align_up(w + 128 * static_cast<int64_t>(j.n_blocks), 256);
  }
  totals[4] = w;
  for (int k = 0; k < n; ++k) {
    JDesc& j = descs[k];
    if (infos[k].status != TP_JPEG_OK) continue;
    j.clean_off = w;
    w = align_up(w + j.raw_len + 64, 256);
    j.seg_off = w;
    w = align_up(w + 8 * (static_cast<int64_t>(j.n_seg) + 1), 256);
    for (int c = 0; c < j.ncomp; ++c) {
      j.plane_off[c] = w;
      // + 64: the colour kernel reads a row's neighbour byte one past the plane's last row
      w = align_up(w + static_cast<int64_t>(j.plane_w[c]) * j.plane_h[c] + 64, 256);
    }
  }
  totals[0] = slots;
  totals[1] = blocks;
  totals[2] = rows;
  totals[5] = chunks;
  return w;
}

}  // extern "C"
