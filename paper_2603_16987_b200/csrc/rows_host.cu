// Host-side helpers for touched-row staging (tp_plan_host, tp_touched_rows).
//
// K2's 2-tap stencil reads only the source rows y0(j), y1(j) of its output rows (tiles:
// H -> rows*E, thumbnail: H -> E; imgproc.py:298-306), so an uploader that knows the
// plan can send just those rows. tp_touched_rows builds the row map K2 reads them
// through (tp_tile_rows). The arithmetic is the device's: K1's exact integer planner
// (plan_core.cuh, restated scalar here) and the fp64 axis taps with no contraction
// (this file is compiled with -ffp-contract=off; x86-64 has no fused multiply-add by
// default either), so the marked rows are exactly the rows K2 stages.

#include <cmath>
#include <cstdint>

#include "tileprep.h"
#include "tp_common.cuh"

namespace {

struct HostCand {
  uint32_t big = 1, small = 1;
  int32_t rows = 0, cols = 0;
};

HostCand host_cand(uint32_t w, uint32_t h, int r, int c) {
  const uint32_t a = w * static_cast<uint32_t>(r), b = h * static_cast<uint32_t>(c);
  HostCand k;
  k.big = a > b ? a : b;
  k.small = a > b ? b : a;
  k.rows = r;
  k.cols = c;
  return k;
}

// strict "a precedes b" in the reference key order (ratio, tiles, rows): K1's rule
bool host_precedes(const HostCand& a, const HostCand& b) {
  if (b.rows == 0) return a.rows != 0;
  if (a.rows == 0) return false;
  const uint64_t lhs = static_cast<uint64_t>(a.big) * b.small;
  const uint64_t rhs = static_cast<uint64_t>(b.big) * a.small;
  if (lhs != rhs) return lhs < rhs;
  const int ta = a.rows * a.cols, tb = b.rows * b.cols;
  if (ta != tb) return ta < tb;
  return a.rows < b.rows;
}

// the device's axis_tap (tp_common.cuh): pos = (i + 0.5) * (src / out) - 0.5, clipped
void mark_axis(int src, int out, int32_t* map) {
  const double scale = static_cast<double>(src) / static_cast<double>(out);
  for (int i = 0; i < out; ++i) {
    double pos = (static_cast<double>(i) + 0.5) * scale;
    pos = pos - 0.5;
    pos = std::fmin(std::fmax(pos, 0.0), static_cast<double>(src - 1));
    int i0 = static_cast<int>(std::floor(pos));
    if (i0 > src - 1) i0 = src - 1;
    const int i1 = i0 + 1 < src ? i0 + 1 : src - 1;
    map[i0] = 1;
    map[i1] = 1;
  }
}

}  // namespace

extern "C" int tp_plan_host(int32_t width, int32_t height, int32_t tile_edge, int32_t max_tiles,
                            int32_t* plan) {
  if (!plan) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_plan_host: null plan");
  if (width < 1 || height < 1 || width > TP_MAX_EDGE || height > TP_MAX_EDGE)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "image size %dx%d outside [1, %d]", width,
                         height, TP_MAX_EDGE);
  if (tile_edge < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tile_edge must be positive");
  if (max_tiles < 1 || max_tiles > TP_MAX_TILES_LIMIT)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "max_tiles %d outside [1, %d]", max_tiles,
                         TP_MAX_TILES_LIMIT);
  const uint32_t w = static_cast<uint32_t>(width), h = static_cast<uint32_t>(height);
  HostCand best;
  for (int r = 1; r <= max_tiles; ++r) {
    const int cmax = max_tiles / r;
    int c0 = static_cast<int>((w * static_cast<uint32_t>(r)) / h);
    c0 = c0 < 1 ? 1 : (c0 > cmax ? cmax : c0);
    const int c1 = c0 + 1 < cmax ? c0 + 1 : cmax;
    const HostCand k0 = host_cand(w, h, r, c0);
    if (host_precedes(k0, best)) best = k0;
    if (c1 != c0) {
      const HostCand k1 = host_cand(w, h, r, c1);
      if (host_precedes(k1, best)) best = k1;
    }
  }
  const int tiles = best.rows * best.cols;
  plan[TP_PLAN_ROWS] = best.rows;
  plan[TP_PLAN_COLS] = best.cols;
  plan[TP_PLAN_TILE_EDGE] = tile_edge;
  plan[TP_PLAN_THUMB] = tiles > 1 ? 1 : 0;
  plan[TP_PLAN_RESIZED_W] = best.cols * tile_edge;
  plan[TP_PLAN_RESIZED_H] = best.rows * tile_edge;
  return TP_OK;
}

extern "C" int64_t tp_touched_rows(int32_t width, int32_t height, const int32_t* plan,
                                   int32_t* row_map) {
  if (!plan || !row_map || width < 1 || height < 1 || height > TP_MAX_EDGE)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_touched_rows: bad arguments");
  const int E = plan[TP_PLAN_TILE_EDGE], RH = plan[TP_PLAN_RESIZED_H];
  if (E < 1 || RH < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_touched_rows: bad plan");
  int32_t* map = row_map + 1;
  for (int y = 0; y < height; ++y) map[y] = 0;
  mark_axis(height, RH, map);                     // tiles: H -> rows * E
  if (plan[TP_PLAN_THUMB]) mark_axis(height, E, map);  // thumbnail: H -> E
  int32_t n = 0;
  for (int y = 0; y < height; ++y) map[y] = map[y] ? n++ : -1;
  row_map[0] = n;
  return n;
}

extern "C" int64_t tp_touched_cols(int32_t width, int32_t height, const int32_t* plan,
                                   int32_t* col_map) {
  if (!plan || !col_map || width < 1 || height < 1 || width > TP_MAX_EDGE)
    return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_touched_cols: bad arguments");
  const int E = plan[TP_PLAN_TILE_EDGE], RW = plan[TP_PLAN_RESIZED_W];
  if (E < 1 || RW < 1) return tp::set_error(TP_ERR_INVALID_ARGUMENT, "tp_touched_cols: bad plan");
  int32_t* map = col_map + 1;
  for (int x = 0; x < width; ++x) map[x] = 0;
  mark_axis(width, RW, map);                          // tiles: W -> cols * E
  if (plan[TP_PLAN_THUMB]) mark_axis(width, E, map);  // thumbnail: W -> E
  int32_t n = 0;
  for (int x = 0; x < width; ++x) map[x] = map[x] ? n++ : -1;
  col_map[0] = n;
  return n;
}

