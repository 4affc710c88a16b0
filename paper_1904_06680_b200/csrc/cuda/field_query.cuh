// field_query.cuh -- the binned obstacle field on the device and the collision query
// (src/geometry.cpp:63-76) over the cells under the chassis bounding box.
// Part of the sampler kernels (rollout.cuh).
#pragma once

#include "common.cuh"

namespace ppdev {

// Binned obstacle field (csrc/capi/field.hpp): static points stored once,
// dynamic points once per state row, both in cell order of one uniform grid
// (cell size g, origin bx0/by0); starts[cell] = first point of the cell.
// With ncy == 1 the grid is a row of x-buckets.
template <typename Real>
struct Field {
  const typename Vec2T<Real>::type* spts;
  const typename Vec2T<Real>::type* dpts;
  const int* sst;
  const int* dst;
  const typename Vec2T<Real>::type* sbox;  // per cell: (centre), (half extents)
  const int* cst;                          // per cell: first chunk box
  const typename Vec2T<Real>::type* cbox;  // per chunk: (centre), (half extents)
  int Ns, Nd;
  int dstride;  // points per dynamic row in the image (Nd + sentinels)
  int ncx, ncy;
  int coop;  // RoundArgs::coop
  // kernel kind 3 (one x-bucket part staged in shared memory): 32-bit shared
  // addresses of its points and starts, fixed once per CTA so a step's row
  // base is one IMAD each instead of a generic-to-shared conversion (the byte
  // strides of a state row, 0 for a static part, are the round constants
  // Consts::k3_row_bytes / k3_st_row_bytes)
  uint32_t s_pts, s_st;
};

// ld.shared of a staged field's point / start at a 32-bit shared address
template <typename Real>
__device__ __forceinline__ typename Vec2T<Real>::type lds_point(uint32_t a);
template <>
__device__ __forceinline__ float2 lds_point<float>(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ double2 lds_point<double>(uint32_t a) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_start(uint32_t a) {
  int v;
  asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

template <typename Real>
__device__ __forceinline__ Field<Real> field_at(const RoundArgs& a, const void* base,
                                                const FieldLayout& l) {
  using R2 = typename Vec2T<Real>::type;
  const unsigned char* p = static_cast<const unsigned char*>(base);
  Field<Real> f{reinterpret_cast<const R2*>(p), reinterpret_cast<const R2*>(p + l.dpts),
                reinterpret_cast<const int*>(p + l.sst), reinterpret_cast<const int*>(p + l.dst),
                reinterpret_cast<const R2*>(p + l.sbox), reinterpret_cast<const int*>(p + l.cst),
                reinterpret_cast<const R2*>(p + l.cbox), a.field_ns, a.field_nd,
                a.field_dstride, a.grid_nx, a.grid_ny, a.coop, 0u, 0u};
  return f;
}

// The kind-3 shared addressing of a field staged at `smem`.
template <typename Real>
__device__ __forceinline__ void bind_shared(Field<Real>& f, const unsigned char* smem,
                                            const FieldLayout& l) {
  const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const bool dyn = f.Nd > 0;
  f.s_pts = s0 + static_cast<uint32_t>(dyn ? l.dpts : 0);
  f.s_st = s0 + static_cast<uint32_t>(dyn ? l.dst : l.sst);
}

// Inside-margin of one point against the chassis at (x, y, phi):
// min(r2 - d2, fe - bx, re + bx, hw - by, hw + by) in the reference's own
// expressions (src/geometry.cpp:63-76): > 0 iff the reference reports the
// point inside (each difference has the exact sign of its comparison).
template <typename Real>
__device__ __forceinline__ Real point_margin(const Consts<Real>& K, Real x, Real y, Real c, Real s,
                                             Real kx, Real ky, Real mx, Real my) {
  const Real dx = mx - x, dy = my - y;
  const Real bx = c * dx + s * dy;
  const Real by = -s * dx + c * dy;
  const Real pre = K.r2 - (dx * dx + dy * dy);
  const Real box = fmin(fmin(K.fe - bx, K.re + bx), fmin(K.hw - by, K.hw + by));
  return fmin(pre, box);
}
// FP32: the point in the vehicle frame via the pre-rotated vehicle position
// (kx, ky include the rectangle centre offset), the rectangle tested around
// its centre and no separate circle prefilter (the rectangle lies inside the
// bounding circle; the prefilter can only matter at the rear corners within
// rounding -- a narrow hit, which the marginal flag sends to the exact
// re-ranking).
// The pair (bx, by) = (fma(c, mx, fma(s, my, -kx)), fma(-s, mx, fma(c, my, -ky)))
// in two packed FFMA2 with the point coordinate as the broadcast operand
// (sm_100 FFMA2 Ra.F32 form): bit-identical to the scalar FMAs, half the issue.
template <>
__device__ __forceinline__ float point_margin<float>(const Consts<float>& K, float, float,
                                                     float c, float s, float kx, float ky,
                                                     float mx, float my) {
#if PARAPLAN_FFMA2
  const float2 t = __ffma2_rn(make_float2(my, my), make_float2(s, c), make_float2(-kx, -ky));
  const float2 b = __ffma2_rn(make_float2(mx, mx), make_float2(c, -s), t);
  return fminf(K.bhx - fabsf(b.x), K.hw - fabsf(b.y));
#else
  const float bx = fmaf(c, mx, fmaf(s, my, -kx));
  const float by = fmaf(-s, mx, fmaf(c, my, -ky));
  return fminf(K.bhx - fabsf(bx), K.hw - fabsf(by));
#endif
}

// Collision of the chassis at (x, y, phi) with row h. Only the grid cells
// covering [x - qpad, x + qpad] x [y - qpad, y + qpad] are visited: every
// point outside them is farther than cull > r from the vehicle and fails the
// reference's bounding-circle prefilter (src/geometry.cpp:71). Returns the
// inside-margin max over visited points (the reference reports a collision
// iff it is > 0; a small |margin| marks a verdict rounding could flip).
// A lane stops at its first robust hit (margin >= stop). Warp-synchronous:
// all 32 lanes call it, every loop is warp-uniform.
// Points of one part (static, or the dynamic row of state h) in the cells
// covering the query window; updates the inside-margin `best`.
template <typename Real, int kGrid>
__device__ __forceinline__ void scan_part(const typename Vec2T<Real>::type* pts, const int* st,
                                          int ncy, int cx_lo, int cx_hi, int cy_lo, int cy_hi,
                                          const Consts<Real>& K, Real x, Real y, Real c, Real s,
                                          Real kx, Real ky, Real stop, Real& best) {
  if constexpr (kGrid == 3) {
    // x-buckets of a sentinel-padded part (field.hpp pad_s / pad_d): every
    // lane reads `rounds` consecutive points from its window's first. Points
    // past its window lie in later buckets (outside the chassis box by more
    // than the pad) or are sentinels, so their margins are negative and the
    // max is the window's -- no bounds select, immediate-offset loads
    const int lo = st[cx_lo];
    const int cnt = st[cx_hi + 1] - lo;
    const int rounds = __reduce_max_sync(kFull, cnt);
    const auto* p = pts + lo;
#pragma unroll 4
    for (int j = 0; j < rounds; ++j) {
      const auto m = p[j];
      best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
    }
  } else if constexpr (kGrid == 0) {  // x-buckets: one contiguous range
    const int lo = st[cx_lo];
    const int cnt = st[cx_hi + 1] - lo;
    const int rounds = __reduce_max_sync(kFull, cnt);
#if PARAPLAN_BRANCHLESS_SCAN
    // no per-point branch: a lane past its own range re-reads point 0 of
    // the part (which exists: the part is not empty) and discards it
    for (int j = 0; j < rounds; ++j) {
      const bool in = j < cnt;
      const auto m = pts[in ? lo + j : 0];
      const Real pm = point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y);
      best = in ? fmax(best, pm) : best;
    }
#else
    for (int j = 0; j < rounds; ++j) {
      if (j < cnt) {
        const auto m = pts[lo + j];
        best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
      }
    }
#endif
  } else {  // 2-D cells, one contiguous range per cell column; early exit
    const int ncol = cx_hi - cx_lo + 1;
    const int cols = __reduce_max_sync(kFull, ncol);
    for (int k = 0; k < cols; ++k) {
      const bool has = k < ncol;
      const int cell = (has ? cx_lo + k : cx_lo) * ncy;
      const int lo = st[cell + cy_lo];
      const int cnt = has ? st[cell + cy_hi + 1] - lo : 0;
      // a lane stops at its first robust hit (margin >= stop)
      for (int j = 0; __any_sync(kFull, j < cnt && best < stop); ++j) {
        if (j < cnt && best < stop) {
          const auto m = pts[lo + j];
          best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
        }
      }
    }
  }
}

// Dense static part (grid_mode 2), column by column. A column holding more
// than kDenseCol points in the window is visited cell by cell: a cell whose
// tight point box is separated from the rectangle along the rectangle's own
// axes (by more than the pad) holds no point the reference could report
// inside, and is skipped without reading its points. Sparser columns are
// scanned as one range, as in grid_mode 1.
constexpr int kDenseCol = 16;

// Points per chunk box of a cell holding `count` points (field.hpp
// chunk_size: >= 16, at most 32 chunks per cell).
__device__ __forceinline__ int chunk_size_dev(int count) {
  return count <= 512 ? 16 : (count + 31) / 32;
}

// A box (centre m, half extents e) against the chassis rectangle in the
// rectangle's own frame: > 0 when the box lies inside the rectangle by that
// much (every point of it is a robust hit), < -pad when it is separated from
// it by more than the pad (no point of it can be inside), else in between.
template <typename Real>
__device__ __forceinline__ Real box_margin(const Consts<Real>& K, Real c, Real s, Real ac, Real as,
                                           Real kx, Real ky, typename Vec2T<Real>::type m,
                                           typename Vec2T<Real>::type e) {
  const Real du = fabs(c * m.x + s * m.y - kx), dv = fabs(-s * m.x + c * m.y - ky);
  const Real eu = e.x * ac + e.y * as, ev = e.x * as + e.y * ac;
  // inside margin of the box's farthest extent; separation of its nearest
  const Real inside = fmin(K.bhx - (du + eu), K.hw - (dv + ev));
  const Real apart = fmax(du - eu - K.bhx, dv - ev - K.hw);
  return apart > K.qpad ? -apart : (inside > Real(0) ? inside : Real(0));
}

template <typename Real>
__device__ __forceinline__ void scan_boxed(const Field<Real>& f, int ncy, int cx_lo, int cx_hi,
                                           int cy_lo, int cy_hi, const Consts<Real>& K, Real x,
                                           Real y, Real c, Real s, Real kx, Real ky, Real stop,
                                           Real& best) {
  const auto* pts = f.spts;
  const int* st = f.sst;
  const Real ac = fabs(c), as = fabs(s);
  const int nrow = cy_hi - cy_lo + 1;
  const int ncol = cx_hi - cx_lo + 1;
  const int cols = __reduce_max_sync(kFull, ncol);
  for (int k = 0; k < cols; ++k) {
    const bool has = k < ncol;
    const int cell0 = (has ? cx_lo + k : cx_lo) * ncy + cy_lo;
    const int lo = st[cell0];
    const int n = has ? st[cell0 + nrow] - lo : 0;
    const bool dense = n > kDenseCol;
    // dense columns: cell by cell behind the cell box, then chunk by chunk
    // behind the chunk boxes; a box inside the rectangle is a robust hit
    const int rows = __reduce_max_sync(kFull, dense ? nrow : 0);
    for (int q = 0; q < rows; ++q) {
      int clo = 0, cnt = 0, ch0 = 0, nch = 0;
      if (dense && q < nrow && best < stop) {
        const int cell = cell0 + q;
        clo = st[cell];
        cnt = st[cell + 1] - clo;
        if (cnt > 0) {
          const Real bm = box_margin(K, c, s, ac, as, kx, ky, f.sbox[2 * cell], f.sbox[2 * cell + 1]);
          if (bm > Real(0)) {
            best = fmax(best, bm);
          } else if (bm == Real(0)) {
            ch0 = f.cst[cell];
            nch = f.cst[cell + 1] - ch0;
          }
        }
      }
      const int csz = chunk_size_dev(cnt);
      const int nchunks = __reduce_max_sync(kFull, nch);
      for (int j = 0; j < nchunks; ++j) {
        int at = 0, left = 0;
        if (j < nch && best < stop) {
          const Real bm = box_margin(K, c, s, ac, as, kx, ky, f.cbox[2 * (ch0 + j)],
                                     f.cbox[2 * (ch0 + j) + 1]);
          if (bm > Real(0)) {
            best = fmax(best, bm);
          } else if (bm == Real(0)) {
            at = clo + j * csz;
            left = min(csz, clo + cnt - at);
          }
        }
        if (__any_sync(kFull, left > 0)) {
#pragma unroll 4
          for (int i = 0; i < csz; ++i) {
            if (i < left) {
              const auto m = pts[at + i];
              best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
            }
          }
        }
      }
    }
    // sparse columns: one range
    const int cnt = dense ? 0 : n;
    for (int j = 0; __any_sync(kFull, j < cnt && best < stop); ++j) {
      if (j < cnt && best < stop) {
        const auto m = pts[lo + j];
        best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
      }
    }
  }
}

// Dense static part for ONE query, scanned by the whole warp: lane k takes
// the window cells k, k + 32, ... and applies scan_boxed's per-cell rule
// (a column holding <= kDenseCol points in the window: all its points; else
// the cell box, then the chunk boxes, then the points of straddling chunks).
// The contributions are scan_boxed's without its early exit, so the
// max margin decides the same verdict and the same marginal flag. Returns
// the warp-wide max (every lane). Used when few lanes of a warp still need
// a dense scan (the end of a round), where the lane-serial scan would run
// one long latency chain per lane.
template <typename Real>
__device__ __forceinline__ Real coop_scan_boxed(const Field<Real>& f, int ncy, int cx_lo, int cx_hi,
                                                int cy_lo, int cy_hi, const Consts<Real>& K,
                                                Real x, Real y, Real c, Real s, Real kx, Real ky,
                                                int lane) {
  const auto* pts = f.spts;
  const int* st = f.sst;
  const Real ac = fabs(c), as = fabs(s);
  const int nrow = cy_hi - cy_lo + 1;
  const int ncell = (cx_hi - cx_lo + 1) * nrow;
  Real best = Real(-1e30);
  for (int idx = lane; idx < ncell; idx += 32) {
    const int col = idx / nrow;
    const int cell0 = (cx_lo + col) * ncy + cy_lo;
    const int cell = cell0 + (idx - col * nrow);
    const int clo = st[cell];
    const int cnt = st[cell + 1] - clo;
    if (cnt == 0) continue;
    if (st[cell0 + nrow] - st[cell0] <= kDenseCol) {  // sparse column: its points
      for (int i = 0; i < cnt; ++i) {
        const auto m = pts[clo + i];
        best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
      }
      continue;
    }
    const Real bm = box_margin(K, c, s, ac, as, kx, ky, f.sbox[2 * cell], f.sbox[2 * cell + 1]);
    if (bm > Real(0)) {
      best = fmax(best, bm);
      continue;
    }
    if (bm < Real(0)) continue;
    const int ch0 = f.cst[cell], nch = f.cst[cell + 1] - ch0;
    const int csz = chunk_size_dev(cnt);
    for (int j = 0; j < nch; ++j) {
      const Real cm = box_margin(K, c, s, ac, as, kx, ky, f.cbox[2 * (ch0 + j)],
                                 f.cbox[2 * (ch0 + j) + 1]);
      if (cm > Real(0)) {
        best = fmax(best, cm);
      } else if (cm == Real(0)) {
        const int at = clo + j * csz;
        const int left = min(csz, clo + cnt - at);
        for (int i = 0; i < left; ++i) {
          const auto m = pts[at + i];
          best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
        }
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(kFull, best, off));
  return best;
}

// The points of the window cells (one contiguous range per cell column) for
// ONE query, scanned by the whole warp: column by column, lane k takes the
// points k, k + 32, ... Returns the warp-wide max margin (every lane).
template <typename Real>
__device__ __forceinline__ Real coop_scan_cells(const typename Vec2T<Real>::type* pts,
                                                const int* st, int ncy, int cx_lo, int cx_hi,
                                                int cy_lo, int cy_hi, const Consts<Real>& K,
                                                Real x, Real y, Real c, Real s, Real kx, Real ky,
                                                int lane) {
  Real best = Real(-1e30);
  for (int k = cx_lo; k <= cx_hi; ++k) {
    const int cell = k * ncy;
    const int hi = st[cell + cy_hi + 1];
    for (int j = st[cell + cy_lo] + lane; j < hi; j += 32) {
      const auto m = pts[j];
      best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_xor_sync(kFull, best, off));
  return best;
}

// At most this many live lanes in a warp: the warp scans each of their
// collision windows together (coop_scan_boxed / coop_scan_cells) instead of
// lane by lane. At the end of a round most lanes are idle and the few
// remaining rollouts would otherwise run as long single-lane latency chains.
#ifndef PARAPLAN_COOP_LANES
#define PARAPLAN_COOP_LANES 4
#endif

// Collision of the chassis at (x, y, phi) with the field at state h. Only the
// cells covering the world-frame bounding box of the chassis rectangle (+ a
// pad of an eighth of a cell) are visited: the reference reports a point
// inside only if it lies strictly inside the rectangle (src/geometry.cpp:
// 63-76), so every point outside that box is a miss whatever the rounding.
// Returns the inside-margin max over visited points (the reference reports a
// collision iff it is > 0; a small |margin| marks a verdict rounding could
// flip). Warp-synchronous: all 32 lanes call it, every loop is warp-uniform.
// `live` is false for a lane whose rollout is over (idle at the end of a
// round): it scans nothing, and on 2-D grids a warp with few live lanes
// scans their windows with all 32 lanes (coop_scan_boxed / coop_scan_cells).
template <typename Real, int kGrid>
__device__ __forceinline__ Real collide_margin(const Field<Real>& f, const Consts<Real>& K, int h,
                                               Real x, Real y, Real c, Real s, Real stop,
                                               bool live = true) {
  const int ncx = f.ncx, ncy = f.ncy;
  const Real ac = fabs(c), as = fabs(s);
  const Real top = K.xtop;  // ncx - 1
  // rectangle centre (x, y) + bcx (c, s); half extents bhx |c| + hw |s| (x)
  const Real ox = x + K.bcx * c - K.bx0;
  const Real ex = K.bhx * ac + K.hw * as + K.qpad;
  const int cx_lo = static_cast<int>(fmin(fmax((ox - ex) * K.binv, Real(0)), top));
  const int cx_hi = static_cast<int>(fmin(fmax((ox + ex) * K.binv, Real(0)), top));
  int cy_lo = 0, cy_hi = 0;
  if constexpr (kGrid == 1 || kGrid == 2) {
    const Real ytop = K.ytop;  // ncy - 1
    const Real oy = y + K.bcx * s - K.by0;
    const Real ey = K.bhx * as + K.hw * ac + K.qpad;
    cy_lo = static_cast<int>(fmin(fmax((oy - ey) * K.binv, Real(0)), ytop));
    cy_hi = static_cast<int>(fmin(fmax((oy + ey) * K.binv, Real(0)), ytop));
  }
  const Real kx = c * x + s * y + K.bcx;  // FP32 rotated-frame form only
  const Real ky = -s * x + c * y;
  Real best = Real(-1e30);
  if constexpr (kGrid == 3) {
    // one part (all points static, or all dynamic: the row of state h),
    // sentinel-padded, in shared memory: every lane reads `rounds`
    // consecutive points from its window's first (see scan_part). A lane
    // whose rollout is over scans nothing (its window would only lengthen the
    // warp's point loop)
    const uint32_t st = f.s_st + static_cast<uint32_t>(h) * K.k3_st_row_bytes;
    const uint32_t pr = f.s_pts + static_cast<uint32_t>(h) * K.k3_row_bytes;
    const int lo = lds_start(st + 4u * static_cast<uint32_t>(cx_lo));
    const int cnt = live ? lds_start(st + 4u * static_cast<uint32_t>(cx_hi + 1)) - lo : 0;
    const int rounds = __reduce_max_sync(kFull, cnt);
    constexpr uint32_t kPt = sizeof(typename Vec2T<Real>::type);
    // whole groups of kK3Group points (the padding covers the overrun: a
    // point past a lane's window lies beyond its box in x, or is a sentinel)
    const int groups = (rounds + kK3Group - 1) / kK3Group;
    uint32_t p = pr + static_cast<uint32_t>(lo) * kPt;
#pragma unroll 1
    for (int j = 0; j < groups; ++j, p += kK3Group * kPt) {
#pragma unroll
      for (int u = 0; u < kK3Group; ++u) {
        const auto m = lds_point<Real>(p + static_cast<uint32_t>(u) * kPt);
        best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
      }
    }
    return best;
  }
  const size_t row_cells = static_cast<size_t>(ncx) * ncy + 1;
  if constexpr (kGrid == 1 || kGrid == 2) {
    // few live lanes (the end of a round): the warp scans each live lane's
    // window together, both parts; lanes whose rollout is over scan nothing
    const unsigned want = __ballot_sync(kFull, live);
    if (f.coop && __popc(want) <= PARAPLAN_COOP_LANES) {
      const int lane = static_cast<int>(threadIdx.x & 31u);
      for (unsigned pend = want; pend != 0u; pend &= pend - 1u) {
        const int src = __ffs(pend) - 1;
        const Real qx = __shfl_sync(kFull, x, src), qy = __shfl_sync(kFull, y, src);
        const Real qc = __shfl_sync(kFull, c, src), qs = __shfl_sync(kFull, s, src);
        const Real qkx = __shfl_sync(kFull, kx, src), qky = __shfl_sync(kFull, ky, src);
        const int q0 = __shfl_sync(kFull, cx_lo, src), q1 = __shfl_sync(kFull, cx_hi, src);
        const int r0 = __shfl_sync(kFull, cy_lo, src), r1 = __shfl_sync(kFull, cy_hi, src);
        const int qh = __shfl_sync(kFull, h, src);
        Real m = Real(-1e30);
        if (f.Ns > 0) {
          m = kGrid == 2 ? coop_scan_boxed<Real>(f, ncy, q0, q1, r0, r1, K, qx, qy, qc, qs, qkx,
                                                 qky, lane)
                         : coop_scan_cells<Real>(f.spts, f.sst, ncy, q0, q1, r0, r1, K, qx, qy,
                                                 qc, qs, qkx, qky, lane);
        }
        if (f.Nd > 0) {
          m = fmax(m, coop_scan_cells<Real>(f.dpts + static_cast<size_t>(qh) * f.dstride,
                                            f.dst + static_cast<size_t>(qh) * row_cells, ncy, q0,
                                            q1, r0, r1, K, qx, qy, qc, qs, qkx, qky, lane));
        }
        if (lane == src) best = m;
      }
      return best;
    }
  }
  // lane by lane. part 0: static points; part 1: the dynamic row of state h
  // (one copy of the scan code, warp-uniform part loop)
  const int cl_hi = live ? cx_hi : cx_lo - 1;  // a lane whose rollout is over scans nothing
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    const bool dyn = part == 1;
    if ((dyn ? f.Nd : f.Ns) == 0) continue;
    const auto* pts = dyn ? f.dpts + static_cast<size_t>(h) * f.dstride : f.spts;
    const int* st = dyn ? f.dst + static_cast<size_t>(h) * row_cells : f.sst;
    if constexpr (kGrid == 2) {
      if (!dyn) {
        scan_boxed<Real>(f, ncy, cx_lo, cl_hi, cy_lo, cy_hi, K, x, y, c, s, kx, ky, stop, best);
        continue;
      }
    }
    scan_part<Real, kGrid>(pts, st, ncy, cx_lo, cl_hi, cy_lo, cy_hi, K, x, y, c, s, kx, ky, stop,
                           best);
  }
  return best;
}

}  // namespace ppdev
