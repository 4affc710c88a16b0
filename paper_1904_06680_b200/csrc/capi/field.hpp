// field.hpp -- the obstacle field of one planning tick, split and binned.
//
// The reference hands the planner an ExtrapolatedField: (H+1) rows of N
// anchor-frame points, point j of row h at x_j + h*step_x, y_j + h*step_y
// (src/geometry.cpp:43-61), and tests every point of row h at state h
// (src/geometry.cpp:63-76, src/planner.cpp:138-142). Here the points are
// split into a static part (identical in every row: stored once) and a
// dynamic part (one row per state), and both are binned on a uniform cell
// grid so a collision query visits only the cells within cull > r of the
// vehicle. The collision verdict is an OR over points, so neither the split
// nor the cell order changes it; skipped points fail the reference's own
// bounding-circle prefilter.
//
// `Binned` is the FP64 image (kept on the host for the exact rollouts of the
// certification and the epilogue); the device images (FP32 or FP64) are
// packed from it with the same layout.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "paraplan/geometry.hpp"

namespace ppfield {

struct Binned {
  int Ns = 0, Nd = 0, rows = 0;  // static points, dynamic points per row, rows (H+1)
  int nx = 1, ny = 1;            // cells; ny == 1: x-buckets (small clouds)
  double x0 = 0.0, y0 = 0.0, g = 1.0, cull = 0.0;
  std::vector<double> spts;      // Ns x 2, cell order
  std::vector<double> dpts;      // rows x Nd x 2, per row cell order
  std::vector<int32_t> sst;      // cells + 1
  std::vector<int32_t> dst;      // rows x (cells + 1)
  // Dense static clouds: per cell the tight bounding box of its points as
  // (centre x, centre y, half width, half height); a query skips a cell whose
  // box is separated from the chassis rectangle.
  bool boxes = false;
  std::vector<double> sbox;      // cells x 4 (when boxes)
  // ... and per cell its points in chunks of chunk_size(count) consecutive
  // points, each with its own tight box: chunk j of cell c is box
  // cst[c] + j and covers points sst[c] + j * chunk_size .. (when boxes)
  std::vector<int32_t> cst;      // cells + 1
  std::vector<double> cbox;      // chunks x 4
  // Raw movers of a points field (x, y, step x, step y) x Nd. With
  // `dyn_deferred` the dynamic rows (dpts, dst) are not binned yet: the
  // device bins its own image from these, and bin_dynamic() fills the host
  // image later (overlapped with the device round).
  std::vector<double> dbase;
  bool dyn_deferred = false;
  // Device image only: sentinel points (far away, never inside the chassis)
  // after the static part and after each dynamic row, so the single-part
  // x-bucket scan (kernel kind 3) reads its window's points without a bounds
  // select: a lane reads past its window into later buckets (outside the
  // chassis box) or into the sentinels. Set by the upload (finish_field).
  int pad_s = 0, pad_d = 0;
  int cells() const { return nx * ny; }
  // 0: x-buckets, 1: 2-D cells scanned by column, 2: 2-D cells with boxes
  int mode() const { return boxes ? 2 : (ny > 1 ? 1 : 0); }
  int points() const { return Ns + Nd; }
};

// Points per box chunk of a cell holding `count` points: >= 16, and at most
// 32 chunks per cell (the device keeps a 32-bit chunk mask).
inline int chunk_size(int count) { return count <= 512 ? 16 : (count + 31) / 32; }

// Device image layout: byte offsets of [spts][dpts][sst][dst][sbox][cst]
// [cbox] (16-aligned; the box parts only with boxes).
struct Layout {
  size_t dpts = 0, sst = 0, dst = 0, sbox = 0, cst = 0, cbox = 0, bytes = 0;
};
Layout layout(const Binned& b, size_t elem);

// From a reference field (rows x N points, rows >= 1): a point whose position
// is identical in every row is static.
void from_rows(Binned& b, const double* xy, int rows, int N, double cull);

// From raw anchor-frame points (x, y, heading, speed) x N: the reference's
// extrapolate (src/geometry.cpp:43-61) evaluated for rows 0..rows-1; points
// with a zero step in x and y are static. defer_dynamic: leave the dynamic
// rows unbinned (dyn_deferred) -- see bin_dynamic.
void from_points(Binned& b, const double* pts4, int N, int rows, double T_s, double cull,
                 bool defer_dynamic = false);

// Bins the deferred dynamic rows on the host (no-op when not deferred).
void bin_dynamic(Binned& b);

// Device image in the compute precision (fp64: the binned doubles as-is).
// with_dynamic = false leaves the dynamic parts of the image untouched (the
// device bins them).
void pack(const Binned& b, bool fp64, void* out, bool with_dynamic = true);

// The chassis rectangle in the body frame: -rear < x < front, |y| < half_width.
struct Box {
  double front = 0.0, rear = 0.0, half_width = 0.0;
};

// Exact collision at state k (the reference's per-point test) over the cells
// covering the world bounding box of `box` at (x, y, phi) + g/8.
bool collides(const Binned& b, const paraplan::ChassisPolytope& ch, const Box& box, int k, double x,
              double y, double phi);

// The full (rows x N) position of point j of row k in the reference's order
// is not needed by anyone: the field is only ever queried by state.

}  // namespace ppfield
