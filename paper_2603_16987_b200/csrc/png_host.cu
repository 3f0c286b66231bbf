// K8 host side: PNG chunk parsing and per-image device descriptors.
//
// The reference decodes every payload with Pillow (imgproc.py:213-229).  For the PNGs
// the device decoder takes -- 8-bit greyscale (mode "L"), RGB and palette ("P")
// images, non-interlaced, one run of IDAT chunks, a zlib stream without a preset
// dictionary -- the pixels are Pillow's by construction (PNG is lossless).  What this
// file must get exactly right is *which* payloads those are: everything Pillow would
// treat specially (chunk checksums it verifies, chunk handlers that can raise, modes the
// reference rejects or converts differently) is TP_PNG_UNSUPPORTED and is decoded on the
// host by Pillow itself, exactly as the reference does.  The rules follow
// PIL/PngImagePlugin.py (Pillow 12.2): CRCs are checked for every chunk before the first
// IDAT (ChunkStream.crc) and for no chunk after it; IDAT data is read until the first
// non-IDAT chunk (load_read).  Host code only.

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "png_common.cuh"
#include "tileprep.h"
#include "tp_common.cuh"

namespace {

using tp::png::PDesc;

int status(TpPngInfo* info, int code, const char* fmt, ...) {
  info->status = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(info->message, sizeof(info->message), fmt, ap);
  va_end(ap);
  return TP_OK;
}

uint32_t be32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}

// CRC-32 (ISO 3309 / PNG Annex D), table-driven
struct Crc {
  uint32_t t[256];
  Crc() {
    for (uint32_t n = 0; n < 256; ++n) {
      uint32_t c = n;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[n] = c;
    }
  }
  uint32_t operator()(const uint8_t* p, int64_t n) const {
    uint32_t c = 0xFFFFFFFFu;
    for (int64_t i = 0; i < n; ++i) c = t[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
  }
};
const Crc& crc() {
  static const Crc c;
  return c;
}

bool is_cid(const uint8_t* t) {  // PngImagePlugin.is_cid: rb"\w\w\w\w"
  for (int i = 0; i < 4; ++i) {
    const uint8_t c = t[i];
    const bool w = (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9') ||
                   c == '_';
    if (!w) return false;
  }
  return true;
}

bool type_is(const uint8_t* t, const char* s) { return std::memcmp(t, s, 4) == 0; }

}  // namespace

extern "C" {

TP_API int tp_png_parse(const uint8_t* data, int64_t len, TpPngInfo* info, int64_t* idat_off,
                        int64_t* idat_len, int32_t idat_cap) {
  if (!data || !info || len < 0 || idat_cap < 0) {
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_png_parse: invalid argument");
  }
  std::memset(info, 0, sizeof(*info));
  static const uint8_t kSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1A, '\n'};
  if (len < 8 || std::memcmp(data, kSig, 8) != 0)
    return status(info, TP_PNG_UNSUPPORTED, "not a PNG signature");
  int64_t pos = 8;
  bool have_ihdr = false, in_idat = false, after_idat = false;
  int bit_depth = 0, ctype = -1;
  while (true) {
    if (pos + 8 > len) {
      if (after_idat) break;  // load_end: a short read ends the chunk walk quietly
      return status(info, TP_PNG_UNSUPPORTED, "truncated chunk header at %lld", (long long)pos);
    }
    const uint32_t clen = be32(data + pos);
    const uint8_t* ct = data + pos + 4;
    const int64_t body = pos + 8;
    if (!is_cid(ct)) {
      if (after_idat) break;  // SyntaxError inside load_end is caught
      return status(info, TP_PNG_UNSUPPORTED, "invalid chunk type at %lld", (long long)pos);
    }
    if (type_is(ct, "IDAT")) {
      if (!have_ihdr) return status(info, TP_PNG_UNSUPPORTED, "IDAT before IHDR");
      if (after_idat) return status(info, TP_PNG_UNSUPPORTED, "second IDAT run");
      in_idat = true;
      // load_read: IDAT CRCs are skipped; the data may be cut short (the decode then
      // runs out of input and the host decoder reports the truncation)
      const int64_t avail = len - body < 0 ? 0 : len - body;
      const int64_t take = int64_t(clen) < avail ? int64_t(clen) : avail;
      if (info->n_idat < idat_cap) {
        idat_off[info->n_idat] = body;
        idat_len[info->n_idat] = take;
      }
      ++info->n_idat;
      info->zlib_len += take;
      if (int64_t(clen) + 12 > len - pos) {  // truncated inside the IDAT run
        after_idat = true;
        break;
      }
      pos = body + clen + 4;
      continue;
    }
    if (in_idat) {
      in_idat = false;
      after_idat = true;
    }
    if (after_idat) {
      // load_end: chunks after the image data are parsed leniently; only IEND and chunk
      // types without a Pillow handler are known to be harmless here
      if (type_is(ct, "IEND")) break;
      const bool handled = type_is(ct, "IHDR") || type_is(ct, "PLTE") || type_is(ct, "tRNS") ||
                           type_is(ct, "gAMA") || type_is(ct, "cHRM") || type_is(ct, "sRGB") ||
                           type_is(ct, "pHYs") || type_is(ct, "tEXt") || type_is(ct, "zTXt") ||
                           type_is(ct, "iTXt") || type_is(ct, "eXIf") || type_is(ct, "acTL") ||
                           type_is(ct, "fcTL") || type_is(ct, "fdAT") || type_is(ct, "iCCP");
      if (handled) return status(info, TP_PNG_UNSUPPORTED, "chunk with a handler after IDAT");
      if (int64_t(clen) + 12 > len - pos)  // _safe_read raises OSError in load_end
        return status(info, TP_PNG_UNSUPPORTED, "truncated chunk after IDAT");
      pos = body + clen + 4;
      continue;
    }
    // before the first IDAT: Pillow reads the body and verifies the CRC
    if (int64_t(clen) + 12 > len - pos)
      return status(info, TP_PNG_UNSUPPORTED, "truncated chunk at %lld", (long long)pos);
    const uint32_t want = be32(data + body + clen);
    if (crc()(data + pos + 4, int64_t(clen) + 4) != want)
      return status(info, TP_PNG_UNSUPPORTED, "chunk CRC mismatch at %lld", (long long)pos);
    const uint8_t* s = data + body;
    if (!have_ihdr) {
      if (!type_is(ct, "IHDR") || clen != 13)
        return status(info, TP_PNG_UNSUPPORTED, "first chunk is not a 13-byte IHDR");
      have_ihdr = true;
      info->width = int32_t(be32(s));
      info->height = int32_t(be32(s + 4));
      bit_depth = s[8];
      ctype = s[9];
      info->bit_depth = bit_depth;
      info->color_type = ctype;
      info->interlace = s[12];
      if (s[10] != 0 || s[11] != 0)
        return status(info, TP_PNG_UNSUPPORTED, "compression / filter method");
      if (bit_depth != 8 || (ctype != 0 && ctype != 2 && ctype != 3))
        return status(info, TP_PNG_UNSUPPORTED, "bit depth %d colour type %d", bit_depth, ctype);
      if (s[12] != 0) return status(info, TP_PNG_UNSUPPORTED, "interlaced");
      const int64_t w = be32(s), h = be32(s + 4);
      // K1's planner domain, and below Pillow's decompression-bomb warning threshold
      if (w < 1 || h < 1 || w > 65536 || h > 65536 || w * h > 89478485)
        return status(info, TP_PNG_UNSUPPORTED, "size %lldx%lld", (long long)w, (long long)h);
    } else if (type_is(ct, "PLTE")) {
      if (clen % 3 != 0 || clen == 0 || clen > 768)
        return status(info, TP_PNG_UNSUPPORTED, "PLTE length %u", clen);
      if (ctype == 3) {
        info->pal_n = int32_t(clen / 3);
        std::memcpy(info->pal, s, clen);
      }
    } else if (type_is(ct, "tRNS")) {
      // convert("RGB") ignores the transparency of L / RGB / P images; only the lengths
      // Pillow's handler indexes must be there
      if ((ctype == 0 && clen < 2) || (ctype == 2 && clen < 6))
        return status(info, TP_PNG_UNSUPPORTED, "short tRNS");
    } else if (type_is(ct, "gAMA")) {
      if (clen < 4) return status(info, TP_PNG_UNSUPPORTED, "short gAMA");
    } else if (type_is(ct, "cHRM")) {
      if (clen % 4 != 0) return status(info, TP_PNG_UNSUPPORTED, "cHRM length");
    } else if (type_is(ct, "sRGB")) {
      if (clen < 1) return status(info, TP_PNG_UNSUPPORTED, "short sRGB");
    } else if (type_is(ct, "pHYs")) {
      if (clen < 9) return status(info, TP_PNG_UNSUPPORTED, "short pHYs");
    } else if (type_is(ct, "tEXt")) {
      if (clen > (1u << 20)) return status(info, TP_PNG_UNSUPPORTED, "large tEXt");
    } else if (type_is(ct, "IHDR") || type_is(ct, "IEND") || type_is(ct, "zTXt") ||
               type_is(ct, "iTXt") || type_is(ct, "eXIf") || type_is(ct, "acTL") ||
               type_is(ct, "fcTL") || type_is(ct, "fdAT") || type_is(ct, "iCCP")) {
      return status(info, TP_PNG_UNSUPPORTED, "chunk left to Pillow");
    }
    // any other type has no Pillow handler: skipped (CRC checked above)
    pos = body + clen + 4;
  }
  if (!have_ihdr || info->n_idat == 0) return status(info, TP_PNG_UNSUPPORTED, "no image data");
  if (ctype == 3 && info->pal_n == 0) return status(info, TP_PNG_UNSUPPORTED, "P without PLTE");
  // zlib header (RFC 1950): deflate, window <= 32K, no preset dictionary
  if (info->zlib_len < 8) return status(info, TP_PNG_UNSUPPORTED, "short zlib stream");
  {
    uint8_t hdr[2];
    int got = 0;
    for (int i = 0; i < info->n_idat && i < idat_cap && got < 2; ++i)
      for (int64_t j = 0; j < idat_len[i] && got < 2; ++j) hdr[got++] = data[idat_off[i] + j];
    if (got < 2 && info->n_idat <= idat_cap) return status(info, TP_PNG_UNSUPPORTED, "short zlib");
    if (got == 2) {
      const int cmf = hdr[0], flg = hdr[1];
      if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20))
        return status(info, TP_PNG_UNSUPPORTED, "zlib header %02x %02x", cmf, flg);
    }
  }
  info->status = TP_PNG_OK;
  return TP_OK;
}

TP_API int64_t tp_png_desc_bytes(void) { return static_cast<int64_t>(sizeof(PDesc)); }

TP_API int64_t tp_png_describe(const TpPngInfo* infos, int32_t n, const int64_t* in_off,
                               const int64_t* out_off, void* desc, int64_t* totals) {
  if (n < 0 || (n > 0 && (!infos || !in_off || !out_off || !desc || !totals))) {
    return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_png_describe: invalid argument");
  }
  PDesc* d = static_cast<PDesc*>(desc);
  int64_t units = 0, toks = 0, raw = 0, rbytes = 0, rows = 0, blks = 0;
  for (int k = 0; k < n; ++k) {
    const TpPngInfo& in = infos[k];
    PDesc& o = d[k];
    std::memset(&o, 0, sizeof(o));
    o.out_off = out_off[k];
    o.width = in.width;
    o.height = in.height;
    o.ctype = in.color_type;
    o.bpp = in.color_type == 2 ? 3 : 1;
    o.pal_n = in.pal_n;
    std::memcpy(o.pal, in.pal, sizeof(o.pal));
    o.unit_base = static_cast<int32_t>(units);
    o.row_base = static_cast<int32_t>(rows);
    o.blk_base = static_cast<int32_t>(blks);
    if (in.status != TP_PNG_OK || in_off[k] < 0) {
      o.n_units = 0;  // not a device image
      continue;
    }
    if (in_off[k] % 16 != 0)
      return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_png_describe: in_off[%d] not 16-byte aligned", k);
    o.in_off = in_off[k];
    o.in_bits = in.zlib_len * 8;
    const int64_t rowbytes = static_cast<int64_t>(in.width) * o.bpp;
    o.raw_len = static_cast<int64_t>(in.height) * (1 + rowbytes);
    o.raw_off = raw;
    raw += (o.raw_len + 255) / 256 * 256;
    o.r_stride = (rowbytes + 15) / 16 * 16;
    o.r_off = rbytes;
    rbytes += (tp::png::r_filter_bytes(in.height) + in.height * o.r_stride + 64 + 255) / 256 * 256;
    rows += in.height;
    blks += (in.height + tp::png::kUnfilterRows - 1) / tp::png::kUnfilterRows;
    o.tok_off = toks;
    toks += o.in_bits / 2 + 256;
    o.n_units = static_cast<int32_t>((o.in_bits + tp::png::kUnitBits - 1) / tp::png::kUnitBits);
    units += o.n_units;
  }
  if (rows > (int64_t(1) << 31) - 1)
    return -tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_png_describe: too many rows in one batch");
  auto al = [](int64_t v) { return (v + 255) / 256 * 256; };
  const int64_t units_at = 0;
  const int64_t tok_at = al(units_at + units * static_cast<int64_t>(sizeof(tp::png::PUnit)));
  const int64_t t_at = al(tok_at + toks * 4);
  const int64_t r_at = al(t_at + raw * 2);
  const int64_t m_at = al(r_at + rbytes);
  const int64_t stage_at = al(m_at + raw * 4);
  const int64_t prog_at = al(stage_at + units * tp::png::kStageBytesPerUnit);
  const int64_t adler_at = al(prog_at + (blks + 1) * 4);
  const int64_t end = al(adler_at + static_cast<int64_t>(n) * 16);
  for (int i = 0; i < tp::png::kTotals; ++i) totals[i] = 0;
  totals[0] = units;
  totals[1] = toks;
  totals[2] = raw;
  totals[3] = units_at;
  totals[4] = tok_at;
  totals[5] = t_at;
  totals[6] = r_at;
  totals[7] = end;
  totals[8] = rbytes;
  totals[9] = m_at;
  totals[10] = rows;
  totals[11] = stage_at;
  totals[12] = blks;
  totals[13] = prog_at;
  totals[14] = adler_at;
  return end;
}

}  // extern "C"
