/*
 * tileprep.h — C-ABI of the B200-native VLM input-preprocessing path.
 *
 * The reference (vlmfp, /root/reference/pkg/src/vlmfp) is pure Python and has no
 * FFI; its drop-in boundary is the Python call signatures re-exported at
 * vlmfp/__init__.py:99-139.  Each entry point below replaces the arithmetic core
 * of one of those calls; the Python mirror in paper_2603_16987_b200/ keeps the
 * reference signatures and binds these symbols with ctypes.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; every pointer named d_* is DEVICE memory,
 *     every other pointer is host memory read before the call returns;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - calls are asynchronous on `stream` and never allocate: the caller passes
 *     every output and workspace buffer;
 *   - return TP_OK (0) or a TP_ERR_* code; tp_last_error() gives the message
 *     (thread-local).  Argument errors map to the reference's ValueError.
 */
#ifndef TILEPREP_H_
#define TILEPREP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define TP_API __attribute__((visibility("default")))
#else
#define TP_API
#endif

#define TP_ABI_VERSION 1

/* return codes */
#define TP_OK 0
#define TP_ERR_INVALID_ARGUMENT 1 /* -> ValueError (imgproc.py:106-114, :363-366, :458-459) */
#define TP_ERR_CUDA 2             /* CUDA runtime failure / no device             */
#define TP_ERR_UNSUPPORTED 3      /* outside the exactness domain documented below */

/* element types of normalized output (dtypes.py:13-16) */
#define TP_DTYPE_NONE 0 /* no normalized output (uint8 side output only)   */
#define TP_DTYPE_F32 1  /* "float32"                                       */
#define TP_DTYPE_BF16 2 /* "float16-wide" == ml_dtypes.bfloat16 (dtypes.py:19) */

/* layouts of normalized output */
#define TP_LAYOUT_NCHW 0 /* [tiles, C, E, E]: vision-encoder input layout      */
#define TP_LAYOUT_NHWC 1 /* [tiles, E, E, C]: the reference ImageBuffer layout */

/* per-sequence error flags written by tp_expand */
#define TP_EXPAND_ERR_MARKER_COUNT 1 /* -> ExpansionError        (tokenizer.py:300-302) */
#define TP_EXPAND_ERR_NO_ASSISTANT 2 /* -> MalformedSequenceError (tokenizer.py:318-322) */
#define TP_EXPAND_ERR_OVERFLOW 4     /* output length exceeds int32 / capacity          */

/* plan record: 6 x int32 per image, the TilePlan field order (imgproc.py:64-81) */
#define TP_PLAN_ROWS 0
#define TP_PLAN_COLS 1
#define TP_PLAN_TILE_EDGE 2
#define TP_PLAN_THUMB 3
#define TP_PLAN_RESIZED_W 4
#define TP_PLAN_RESIZED_H 5
#define TP_PLAN_FIELDS 6

/* Largest image edge / max_tiles for which the integer planner is proven equal
 * to the reference's float-log planner. */
#define TP_MAX_EDGE 65536
#define TP_MAX_TILES_LIMIT 1024

TP_API int tp_abi_version(void);
TP_API const char* tp_last_error(void);
/* number of SMs of the current device (0 when no device) */
TP_API int tp_device_sm_count(void);

/* K1 — tile-grid planner, one warp per image.
 * Replaces select_tile_plan (imgproc.py:266-292) for a batch.
 *   d_wh       [n][2]  (width, height) per image, each in [1, TP_MAX_EDGE]
 *   d_plan     [n][6]  TilePlan records (TP_PLAN_*)
 *   d_n_img    [n]     plan.n_images (tiles + thumbnail), feeds tp_expand counts
 *   d_tile_off [n+1]   exclusive prefix sum of n_images (output tile offsets)
 * An invalid width/height writes rows=cols=0 and is reported through the
 * returned d_tile_off[n] == -1 (host wrappers check before use). */
TP_API int tp_plan(const int32_t* d_wh, int32_t n, int32_t tile_edge, int32_t max_tiles,
            int32_t* d_plan, int32_t* d_n_img, int32_t* d_tile_off, void* stream);

/* tp_plan with flags.  TP_PLAN_AFTER_KERNEL: the last operation on `stream` is a kernel
 * launch (e.g. the previous batch's tp_tile), not a copy or an event wait, so K1 may be
 * launched as its programmatic dependent (K1 waits for that kernel before writing; d_wh
 * must have been written before that kernel). */
#define TP_PLAN_AFTER_KERNEL 1
TP_API int tp_plan_ex(const int32_t* d_wh, int32_t n, int32_t tile_edge, int32_t max_tiles,
                      int32_t* d_plan, int32_t* d_n_img, int32_t* d_tile_off, int32_t flags,
                      void* stream);

/* K0 — normalize lookup table: lut[c][v] = ((float)v / 255.f - mean[c]) / std[c]
 * in IEEE fp32 (true divides), optionally rounded to bf16 RNE.
 * Replaces the arithmetic of _normalize_array (imgproc.py:471-478).
 *   mean, std  host float[channels] (already rounded to fp32 like
 *              np.asarray(cfg.mean[:c], dtype=np.float32), imgproc.py:473-474)
 *   d_lut      [channels][256] of float or bf16 */
TP_API int tp_build_lut(int32_t channels, const float* mean, const float* std, int32_t dtype,
                 void* d_lut, void* stream);

/* K0 with the affine form: the same table, followed by per-channel fp32 constants
 * (a[c], b[c]) such that  fma((float)v, a[c], b[c])  rounds (bf16 RNE, or fp32 as is)
 * to exactly lut[c][v] for all 256 values v.  The constants are searched and verified
 * exhaustively on the host (IEEE fp32, the same arithmetic as the device table);
 * *affine_ok (host, nullable) says whether such constants were found.  With the
 * flag TP_TILE_NORM_AFFINE, tp_tile_ex normalizes with one fma per value instead
 * of a table lookup -- identical results, no shared-memory gather.
 *   d_lut  tp_lut_bytes(channels, dtype) bytes: [channels][256] table, then at byte
 *          offset tp_lut_table_bytes(channels, dtype): float a[4], float b[4] */
TP_API int64_t tp_lut_table_bytes(int32_t channels, int32_t dtype);
TP_API int64_t tp_lut_bytes(int32_t channels, int32_t dtype);
TP_API int tp_build_norm(int32_t channels, const float* mean, const float* std, int32_t dtype,
                         void* d_lut, int32_t* affine_ok, void* stream);

/* K2 — fused resample + crop + thumbnail + normalize + layout/cast.
 * Replaces tile_image/_tile_fused (imgproc.py:373-412, :449-465) followed by
 * normalize_tiles (imgproc.py:496-513), for a batch of images.
 *   d_src       packed HWC uint8 images; image k starts at d_src + d_src_off[k]
 *   d_wh        [n][2]
 *   channels    1 or 3 (ImageBuffer invariant, imgproc.py:46-47)
 *   d_plan, d_tile_off   from tp_plan (or uploaded TilePlans)
 *   d_lut       from tp_build_lut (ignored when dtype == TP_DTYPE_NONE)
 *   d_out       [tiles][C][E][E] (NCHW) or [tiles][E][E][C] (NHWC) of dtype
 *   d_out_u8    nullable; [tiles][E][E][C] uint8 tiles (the deferred-normalize
 *               payload, imgproc.py:581-585)
 *   out_capacity tiles the output buffers hold; tiles beyond it are not written
 *               (the host compares d_tile_off[n] against it)
 * uint8 tiles are bit-exact with the reference; normalized values are the LUT
 * entry of that uint8 value, hence also bit-exact. */
TP_API int tp_tile(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh, int32_t n,
            int32_t channels, const int32_t* d_plan, const int32_t* d_tile_off,
            int32_t tile_edge, const void* d_lut, int32_t dtype, int32_t layout, void* d_out,
            uint8_t* d_out_u8, int64_t out_capacity, void* stream);

/* tp_tile with an explicit algorithm:
 *   TP_TILE_ALGO_AUTO / _FAST: fp32 2-tap arithmetic with a proven error window,
 *       exact fp64 recomputation of the values inside the window (bit-exact);
 *   TP_TILE_ALGO_EXACT: every value in fp64 in the reference order (the
 *       straightforward kernel, kept as an on-device cross-check). */
#define TP_TILE_ALGO_AUTO 0
#define TP_TILE_ALGO_FAST 1
#define TP_TILE_ALGO_EXACT 2
/* or-ed into algo: d_lut comes from tp_build_norm with *affine_ok == 1 (fast path,
 * normalized outputs without uint8 tiles) */
#define TP_TILE_NORM_AFFINE 256
/* or-ed into algo: the immediately preceding operation on `stream` is the tp_plan
 * that produced d_plan / d_tile_off, so K2 may be launched as its programmatic
 * dependent (its launch and prologue overlap K1).  Without the flag K2 is a plain
 * launch: a programmatic launch could start before a preceding copy had landed. */
#define TP_TILE_AFTER_PLAN 512
TP_API int tp_tile_ex(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                      int32_t n, int32_t channels, const int32_t* d_plan,
                      const int32_t* d_tile_off, int32_t tile_edge, const void* d_lut,
                      int32_t dtype, int32_t layout, void* d_out, uint8_t* d_out_u8,
                      int64_t out_capacity, int32_t algo, void* stream);

/* K1 + K2 in one launch for small batches (n <= TP_PLAN_TILE_MAX_IMAGES; batch-1
 * latency): every CTA of the K2 grid plans the batch with K1's rule itself, CTA 0
 * writes d_plan / d_n_img / d_tile_off exactly as tp_plan would, and the tiles are
 * written as by tp_tile_ex.  Fast algorithm only (AUTO / FAST, optionally
 * TP_TILE_NORM_AFFINE); TP_ERR_UNSUPPORTED for larger batches. */
#define TP_PLAN_TILE_MAX_IMAGES 4
TP_API int tp_plan_tile(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                        int32_t n, int32_t channels, int32_t tile_edge, int32_t max_tiles,
                        int32_t* d_plan, int32_t* d_n_img, int32_t* d_tile_off,
                        const void* d_lut, int32_t dtype, int32_t layout, void* d_out,
                        uint8_t* d_out_u8, int64_t out_capacity, int32_t algo, void* stream);

/* Touched-row staging.  K2 reads only the source rows its 2-tap stencil touches
 * (tiles: H -> rows*E, thumbnail: H -> E), so an uploader can send just those rows.
 *   tp_plan_host     K1's exact planner on the host for one image (plan[6])
 *   tp_touched_rows  row map of one image: row_map[0] = n touched rows,
 *                    row_map[1 + y] = compact index of source row y or -1 (h + 1 ints);
 *                    returns n (or a negative error code)
 *   tp_touched_cols  the same for columns (tiles: W -> cols*E, thumbnail: W -> E):
 *                    col_map[0] = n touched columns, col_map[1 + x] = index or -1
 *   tp_tile_rows     tp_tile_ex over images whose pixel blocks hold only the touched
 *                    rows, each holding only the touched columns (compact order, rows
 *                    of n_cols*channels bytes): d_row_map holds, per image, the row map
 *                    (h + 1 ints) followed by the column map (w + 1 ints);
 *                    d_row_map_off[k] is the int32 index of image k's maps.  Fast
 *                    algorithm only.  Same output as tp_tile_ex on the full images. */
TP_API int tp_plan_host(int32_t width, int32_t height, int32_t tile_edge, int32_t max_tiles,
                        int32_t* plan);
TP_API int64_t tp_touched_rows(int32_t width, int32_t height, const int32_t* plan,
                               int32_t* row_map);
TP_API int64_t tp_touched_cols(int32_t width, int32_t height, const int32_t* plan,
                               int32_t* col_map);
TP_API int tp_tile_rows(const uint8_t* d_src, const int64_t* d_src_off, const int32_t* d_wh,
                        int32_t n, int32_t channels, const int32_t* d_plan,
                        const int32_t* d_tile_off, int32_t tile_edge, const void* d_lut,
                        int32_t dtype, int32_t layout, void* d_out, uint8_t* d_out_u8,
                        int64_t out_capacity, int32_t algo, const int32_t* d_row_map,
                        const int64_t* d_row_map_off, void* stream);

/* Host staging packer (replaces transfer.pack's per-buffer copies, transfer.py:211-233,
 * for image batches).  Copies n HWC uint8 images from caller memory into one payload
 * (normally page-locked, then uploaded with one H2D copy), on a persistent pool of
 * host threads (`threads` <= 0: all of them; tp_host_threads() reports the count).
 *   src[k], src_stride[k]  image k: wh[k][1] rows of wh[k][0]*channels bytes, row y at
 *                          src[k] + y * src_stride[k]
 *   dst + dst_off[k]       image k's block in the payload
 *   row_map                nullable: image k copies only the rows y with
 *                          row_map[row_map_off[k] + 1 + y] = i >= 0, to row i of its
 *                          block (the tp_touched_rows layout read by tp_tile_rows);
 *                          columns are copied whole.
 * Host memory only; no CUDA calls. */
TP_API int32_t tp_host_threads(void);
TP_API int tp_stage_pack(int32_t n, const uint8_t* const* src, const int64_t* src_stride,
                         const int32_t* wh, int32_t channels, const int32_t* row_map,
                         const int64_t* row_map_off, uint8_t* dst, const int64_t* dst_off,
                         int32_t threads);

/* K7 — device JPEG decode (replaces the PIL decode of
 * decode_image / _decode_pass, imgproc.py:213-260, for baseline JPEGs).  Bit-exact with
 * Pillow's libjpeg-turbo (JDCT_ISLOW, fancy upsampling, jdcolor.c YCbCr->RGB).
 * Host side:
 *   tp_jpeg_parse     markers up to SOS of one payload (host memory); info->status says
 *                     whether the device decoder takes it (baseline Huffman 8-bit, 1 or 3
 *                     components, Y sampling 1x1 / 2x1 / 2x2 with 1x1 chroma, JFIF /
 *                     YCbCr, one interleaved scan, restart markers allowed).  Anything else
 *                     (progressive, arithmetic, 12-bit, CMYK, 4:4:0, ...) is
 *                     TP_JPEG_UNSUPPORTED: decode it on the host, as the reference does.
 *   tp_jpeg_describe  per-image device descriptors (tp_jpeg_desc_bytes() each) for a
 *                     batch: image k's entropy-coded bytes sit at raw_off[k] of the payload
 *                     (4-byte aligned), its RGB HWC output at out_off[k] of d_out; returns
 *                     the workspace bytes tp_jpeg_decode needs (< 0: error code)
 * Device side:
 *   tp_jpeg_decode    unstuff -> parallel Huffman decode (self-synchronizing
 *                     subsequences of sub_bits bits) -> DC prediction -> ISLOW IDCT ->
 *                     fancy upsampling + colour conversion into d_out.  d_status[k] = 0,
 *                     or nonzero when image k's entropy data is not a clean baseline
 *                     stream (corrupt / truncated, misnumbered restart markers, a block
 *                     outside the range where libjpeg-turbo's 16-bit SIMD IDCT is exact):
 *                     decode that one on the host. */
#define TP_JPEG_OK 0
#define TP_JPEG_UNSUPPORTED 1
#define TP_JPEG_CORRUPT 2
typedef struct {
  int32_t status;
  int32_t width, height, ncomp;
  int32_t comp_id[3], comp_h[3], comp_v[3], comp_tq[3], comp_td[3], comp_ta[3];
  int32_t restart_interval;
  int32_t qt_mask, dc_mask, ac_mask;
  int64_t scan_off, scan_len; /* entropy-coded bytes: payload[scan_off, scan_off + scan_len) */
  uint16_t qt[4][64];         /* natural order */
  uint8_t dc_bits[2][16], dc_vals[2][256], ac_bits[2][16], ac_vals[2][256];
  char message[96];
} TpJpegInfo;
TP_API int tp_jpeg_parse(const uint8_t* data, int64_t len, TpJpegInfo* info);
TP_API int64_t tp_jpeg_desc_bytes(void);
TP_API int64_t tp_jpeg_describe(const TpJpegInfo* infos, int32_t n, const int64_t* raw_off,
                                const int64_t* out_off, int32_t sub_bits, void* desc,
                                int64_t* totals /* [8]: slots, blocks, rows, zeroed range, chunks, counts */);
TP_API int tp_jpeg_decode(const uint8_t* d_payload, const void* d_desc, int32_t n,
                          const int64_t* totals, int32_t sub_bits, void* d_work,
                          int64_t work_bytes, uint8_t* d_out, int32_t* d_status,
                          void* stream);

/* K8 — device PNG decode (replaces the PIL decode of
 * decode_image / _decode_pass, imgproc.py:213-260, for 8-bit L / RGB / P PNGs).  PNG is
 * lossless, so the pixels are Pillow's by construction; what must match is which
 * payloads the device takes.
 * Host side:
 *   tp_png_parse      chunk walk of one payload (host memory) with Pillow's rules
 *                     (PngImagePlugin: CRCs before the first IDAT, handlers that can
 *                     raise); info->status TP_PNG_OK: 8-bit non-interlaced colour type 0,
 *                     2 or 3, one IDAT run, zlib without preset dictionary.  The first
 *                     idat_cap IDAT chunks' data extents go to idat_off / idat_len
 *                     (info->n_idat counts all of them).  Anything else is
 *                     TP_PNG_UNSUPPORTED: decode it on the host, as the reference does.
 *   tp_png_describe   per-image descriptors (tp_png_desc_bytes() each): image k's zlib
 *                     stream (its IDAT data back to back) at in_off[k] of the payload
 *                     (16-byte aligned, 64 readable bytes after it), RGB HWC output at
 *                     out_off[k]; returns the workspace bytes tp_png_decode needs.
 * Device side:
 *   tp_png_decode     block finder (deflate block headers at unit boundaries) ->
 *                     parallel inflate of the units to tokens -> chain check + unit
 *                     offsets -> token expansion with window markers -> window
 *                     propagation -> marker resolution -> unfilter (Sub/Up/Average/Paeth
 *                     wavefront) + L/P -> RGB.  d_status[k] = 0, or nonzero when image k
 *                     must be decoded on the host (corrupt, truncated, or a stream the
 *                     finder could not chain). */
#define TP_PNG_OK 0
#define TP_PNG_UNSUPPORTED 1
typedef struct {
  int32_t status;
  int32_t width, height, bit_depth, color_type, interlace;
  int32_t pal_n;   /* PLTE entries (colour type 3) */
  int32_t n_idat; /* IDAT chunks in the (first) IDAT run */
  int64_t zlib_len; /* bytes of IDAT data */
  uint8_t pal[768];
  char message[96];
} TpPngInfo;
TP_API int tp_png_parse(const uint8_t* data, int64_t len, TpPngInfo* info, int64_t* idat_off,
                        int64_t* idat_len, int32_t idat_cap);
TP_API int64_t tp_png_desc_bytes(void);
TP_API int64_t tp_png_describe(const TpPngInfo* infos, int32_t n, const int64_t* in_off,
                               const int64_t* out_off, void* desc,
                               int64_t* totals /* [16]: workspace layout (csrc/png_common.cuh) */);
TP_API int tp_png_decode(const uint8_t* d_payload, const void* d_desc, int32_t n,
                         const int64_t* totals, void* d_work, int64_t work_bytes, uint8_t* d_out,
                         int32_t* d_status, void* stream);

/* K2 variant for resize_bilinear / _resize_array (imgproc.py:352-367): one
 * full-frame half-pixel bilinear resize, uint8 HWC -> uint8 HWC. */
TP_API int tp_resize(const uint8_t* d_src, int32_t width, int32_t height, int32_t channels,
              int32_t out_w, int32_t out_h, uint8_t* d_dst, void* stream);

/* K4 — LUT normalize of uint8 HWC pixels (normalize / normalize_tiles,
 * imgproc.py:481-513, and the deferred-normalize completion step run past the
 * transfer boundary, bench.py:405-409).
 *   n_images x pixels_per_image pixels of `channels` bytes each;
 *   layout NHWC keeps the reference layout, NCHW writes [n][C][pixels]. */
TP_API int tp_normalize(const uint8_t* d_src, int64_t n_images, int64_t pixels_per_image,
                 int32_t channels, const void* d_lut, int32_t dtype, int32_t layout,
                 void* d_out, void* stream);

/* K3 — image-placeholder expansion + supervision mask for a batch of ragged
 * prompts.  Replaces expand_image_placeholders (tokenizer.py:294-315),
 * _first_assistant (:318-322) and build_supervision_mask (:410-418).
 *   d_ids [seq_off[n_seq]], d_seq_off [n_seq+1]: input ids per sequence
 *   d_counts [count_off[n_seq]], d_count_off [n_seq+1]: tile count per marker
 *   tokens_per_tile, marker/ctx/asst ids (SpecialIds, tokenizer.py:43-51)
 *   with_mask: 1 = build_supervision_mask law, 0 = all-false mask
 *   d_out_ids [out_capacity], d_out_off [n_seq+1] (exclusive prefix of lengths)
 *   d_spans [count_off[n_seq]][2] (start, length) relative to the sequence
 *   d_first_asst [n_seq], d_mask [out_capacity] (uint8 0/1), d_err [n_seq]
 *   d_work: workspace of tp_expand_workspace_bytes(n_seq) bytes */
TP_API int64_t tp_expand_workspace_bytes(int32_t n_seq);
TP_API int tp_expand(const int32_t* d_ids, const int32_t* d_seq_off, int32_t n_seq,
              const int32_t* d_counts, const int32_t* d_count_off, int32_t tokens_per_tile,
              int32_t marker_id, int32_t ctx_id, int32_t asst_id, int32_t with_mask,
              int32_t* d_out_ids, int64_t out_capacity, int32_t* d_out_off, int32_t* d_spans,
              int32_t* d_first_asst, uint8_t* d_mask, int32_t* d_err, void* d_work,
              void* stream);

/* K3b — supervision mask of an already expanded sequence with a given first
 * assistant index t (build_supervision_mask, tokenizer.py:410-418):
 * mask[i] = i >= t && ids[i] != asst_id.  t outside [0, n] -> TP_ERR_INVALID_ARGUMENT
 * (the reference raises MalformedSequenceError). */
TP_API int tp_supervision_mask(const int32_t* d_ids, int64_t n, int64_t first_asst,
                               int32_t asst_id, uint8_t* d_mask, void* stream);

/* K6 — greedy longest-match tokenizer, batched (replaces tokenize, tokenizer.py:135-158).
 * The vocabulary is an open-addressing hash table built on the HOST by tp_vocab_build
 * into a caller buffer of tp_vocab_table_bytes(n_tokens) bytes; the caller copies it
 * to the device.  Tokens are 1..16 bytes (longer: TP_ERR_UNSUPPORTED); byte_ids[256]
 * holds the byte-fallback token of each byte value, -1 when the vocabulary has none.
 *   tok_bytes / tok_off[n+1] / tok_id   the non-byte tokens (UTF-8), their ids
 * tp_tokenize: texts are concatenated UTF-8 bytes, text t = d_text[off[t] .. off[t+1]).
 *   d_out_ids  capacity total_bytes (a text of B bytes gives at most B ids)
 *   d_out_off  [n+1] exclusive prefix of the id counts (text t's ids at
 *              d_out_ids[out_off[t] .. out_off[t+1]])
 *   d_err      [n]: 0, or 0x100 | byte for a byte with neither a token nor a fallback
 *              (the reference raises DataError there; that text gets 0 ids)
 *   d_workspace tp_tokenize_workspace_bytes(total_bytes, n) bytes */
TP_API int64_t tp_vocab_table_bytes(int32_t n_tokens);
TP_API int tp_vocab_build(const uint8_t* tok_bytes, const int32_t* tok_off, const int32_t* tok_id,
                          int32_t n_tokens, const int32_t* byte_ids, void* host_table,
                          int64_t table_bytes);
TP_API int64_t tp_tokenize_workspace_bytes(int64_t total_bytes, int32_t n_texts);
TP_API int tp_tokenize(const void* d_vocab, const uint8_t* d_text, const int64_t* d_text_off,
                       int32_t n_texts, int64_t total_bytes, int32_t* d_out_ids,
                       int32_t* d_out_off, int32_t* d_err, void* d_workspace,
                       int64_t workspace_bytes, void* stream);

/* pixel_unshuffle (tokenred.py:80-103): [h][w][d] patch grid of elem_bytes-sized
 * elements -> [h/r][w/r][d*r*r], output cell (i, j) = input cells (i*r+a, j*r+b) with
 * a outer, b inner.  A pure permutation (bit-exact for any element type). */
TP_API int tp_pixel_unshuffle(const void* d_in, int32_t h, int32_t w, int64_t d,
                              int32_t elem_bytes, int32_t r, void* d_out, void* stream);

/* Synthetic HWC uint8 images generated on device (bench/test inputs).
 * kind 0: uniform bytes  v = byte(q & 3) of mix32(key(seed, k) ^ (q >> 2) * golden)
 * kind 1: smooth ramp    v = triangle wave of (3x + 2y + 40c + 17k) with period 510
 * d_off[k] must be a multiple of 4.  The CPU twin lives in oracle/ (tests only). */
TP_API int tp_synth(uint8_t* d_dst, const int64_t* d_off, const int32_t* d_wh, int32_t n,
             int32_t channels, uint64_t seed, int32_t kind, int64_t max_image_bytes,
             void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TILEPREP_H_ */
