// rollout.cuh -- the fused per-control-step sampler kernels (sm_100a).
//
// One lane per candidate. Per candidate a lane
//   1. derives the keyed SplitMix64 stream in closed form and draws
//      theta = center + sigma * N(0,1) (src/rng.cpp:26-58,
//      src/planner.cpp:207-226), in FP64, rounded once to Real,
//   2. rolls the kinematic bicycle over the horizon with the reference's
//      exact check order (src/planner.cpp:66-191): collision vs obstacle row h,
//      inclusive goal box in the goal frame, horizon stop, tanh MLP ->
//      map_controls -> explicit Euler,
//   3. scores the rollout (src/planner.cpp:27-44); lanes reduce to the
//      lexicographically best candidate, ties to the lowest index.
//
// Obstacle rows arrive sorted by x (host, capi.cpp) and are staged once per
// CTA in shared memory. A lane only tests the points of its row whose x lies
// within (r + margin) of its own x, found by binary search: every skipped
// point satisfies |dx| > r, so the reference's bounding-circle prefilter
// (src/geometry.cpp:71, dx^2 + dy^2 >= r^2 -> skip) would have skipped it
// too and the collision verdict is unchanged.
//
// Two schedules:
//   generate_kernel + refill_kernel (theta in registers, [5,2,2] /
//     [5,10,2]): the generator draws theta and the first action of every
//     candidate at full SIMT width into an L2-sized buffer; in the rollout
//     kernel persistent warps claim restart-aligned 32-candidate batches and
//     a lane whose rollout ends loads the next candidate at once, so lanes
//     never idle behind the longest rollout of their warp. Lane bests flush
//     into per-warp, per-restart shared tables, CTAs write per-restart
//     records, the last CTA reduces them.
//   lockstep_kernel (any architecture, theta in a global column per lane):
//     one candidate per lane per tile, 1-restart tiles, last-CTA reduction.
//
// Real = float: throughput path (FMA contraction on). Real = double: parity
// path (rollout_f64.cu is compiled with --fmad=false so each add/mul rounds
// like the reference's -ffp-contract=off build).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "device_api.h"

namespace ppdev {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kBlock = 128;
constexpr int kWarps = kBlock / 32;
#ifndef PARAPLAN_COLL_EXIT
#define PARAPLAN_COLL_EXIT 1
#endif
#ifndef PARAPLAN_REFILL_MINB
#define PARAPLAN_REFILL_MINB 6  // <= 85 registers: 6 CTAs (24 warps) per SM, no spills
#endif

// src/rng.cpp:11-18
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// src/rng.cpp:20-22
__device__ __forceinline__ uint64_t fold(uint64_t h, uint64_t f) {
  return mix64(h ^ (mix64(f) + kGamma + (h << 6) + (h >> 2)));
}
__device__ __forceinline__ double unit53(uint64_t x) {
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}

// Counter-based view of KeyedRng: draw k of key h is mix64(h + (k+1) gamma).
struct Stream {
  uint64_t s;
  __device__ __forceinline__ uint64_t next() {
    s += kGamma;
    return mix64(s);
  }
};

template <typename Real>
struct Vec2T;
template <>
struct Vec2T<float> {
  using type = float2;
};
template <>
struct Vec2T<double> {
  using type = double2;
};

// --------------------------------------------------------------- math ----
template <typename Real>
struct M;

// FP32 sin/cos kernels on [-pi/4, pi/4] (minimax, ~1 ulp; Cephes-style
// coefficients) and the quadrant reduction used by the FP32 rollout.
__device__ __forceinline__ float sin_poly(float r) {
  const float r2 = r * r;
  float p = fmaf(r2, -1.9515295891e-4f, 8.3321608736e-3f);
  p = fmaf(r2, p, -1.6666654611e-1f);
  return fmaf(r * r2, p, r);
}
__device__ __forceinline__ float cos_poly(float r) {
  const float r2 = r * r;
  float p = fmaf(r2, 2.443315711809948e-5f, -1.388731625493765e-3f);
  p = fmaf(r2, p, 4.166664568298827e-2f);
  return fmaf(r2 * r2, p, fmaf(-0.5f, r2, 1.0f));
}
// sincos for the rollout's headings (|x| well below 2^7 * pi/2, where the
// three-part pi/2 products stay exact).
__device__ __forceinline__ void fast_sincosf(float x, float* s, float* c) {
  const float q = rintf(x * 0.636619772367581343f);
  float r = fmaf(-q, 1.5703125f, x);
  r = fmaf(-q, 4.837512969970703125e-4f, r);
  r = fmaf(-q, 7.54978995489188216e-8f, r);
  const float sp = sin_poly(r), cp = cos_poly(r);
  const int qi = static_cast<int>(q);
  const bool swap = (qi & 1) != 0;
  float sv = swap ? cp : sp;
  float cv = swap ? sp : cp;
  sv = (qi & 2) ? -sv : sv;
  cv = ((qi + 1) & 2) ? -cv : cv;
  *s = sv;
  *c = cv;
}

template <>
struct M<float> {
  static __device__ __forceinline__ float th(float x) { return tanhf(x); }
  static __device__ __forceinline__ float tn(float x) { return tanf(x); }
  // tan for |x| <= pi/4 (the steering range when delta_max <= pi/4)
  static __device__ __forceinline__ float tn_small(float x) {
    return sin_poly(x) * __frcp_rn(cos_poly(x));
  }
  static __device__ __forceinline__ void sc(float x, float* s, float* c) {
    fast_sincosf(x, s, c);
  }
  static __device__ __forceinline__ float sq(float x) { return sqrtf(x); }
  static __device__ __forceinline__ float ab(float x) { return fabsf(x); }
  // wrap_angle (src/geometry.cpp:9-13): remainder by 2*pi (two-part
  // Cody-Waite), lower boundary folded onto +pi.
  static __device__ __forceinline__ float wrap(float a) {
    const float n = rintf(a * 0.15915494309189535f);
    float r = fmaf(-n, 6.28318548202514648f, a);
    r = fmaf(-n, -1.7484555314695172e-07f, r);
    return r <= -3.14159274101257324f ? r + 6.28318548202514648f : r;
  }
  static __device__ __forceinline__ float ndiv(float a, double, float inv) { return a * inv; }
};

template <>
struct M<double> {
  static __device__ __forceinline__ double th(double x) { return tanh(x); }
  static __device__ __forceinline__ double tn(double x) { return tan(x); }
  static __device__ __forceinline__ double tn_small(double x) { return tan(x); }
  static __device__ __forceinline__ void sc(double x, double* s, double* c) { sincos(x, s, c); }
  static __device__ __forceinline__ double sq(double x) { return sqrt(x); }
  static __device__ __forceinline__ double ab(double x) { return fabs(x); }
  static __device__ __forceinline__ double wrap(double a) {
    const double r = remainder(a, kTwoPi);  // exact, identical to glibc
    return r <= -kPi ? r + kTwoPi : r;
  }
  // true division, as the reference (src/planner.cpp:117-120, 186-189)
  static __device__ __forceinline__ double ndiv(double a, double d, double) { return a / d; }
};

template <typename Real>
__device__ __forceinline__ Real clampr(Real v, Real lo, Real hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// Round constants live in the kernel parameter bank (RoundArgs::kf / kd).
template <typename Real>
using Consts = ConstsT<Real>;

template <typename Real>
__device__ __forceinline__ const Consts<Real>& consts_of(const RoundArgs& a);
template <>
__device__ __forceinline__ const Consts<float>& consts_of<float>(const RoundArgs& a) {
  return a.kf;
}
template <>
__device__ __forceinline__ const Consts<double>& consts_of<double>(const RoundArgs& a) {
  return a.kd;
}

// ----------------------------------------------------------- networks ----
// [5, H1, 2] forward pass over any weight accessor w(i); layout per layer W
// (out x in, row-major) then b (include/paraplan/policy.hpp:50-53,
// src/policy.cpp:53-80): acc = b, acc += W[o][i] * x[i] ascending, tanh.
template <typename Real, int H1, class W>
__device__ __forceinline__ void mlp_5h2(W&& w, const Real s[5], Real& a0, Real& a1) {
  Real hdn[H1];
#pragma unroll
  for (int o = 0; o < H1; ++o) {
    Real acc = w(5 * H1 + o);
#pragma unroll
    for (int i = 0; i < 5; ++i) acc += w(o * 5 + i) * s[i];
    hdn[o] = M<Real>::th(acc);
  }
  constexpr int off = 6 * H1;
  Real out[2];
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    Real acc = w(off + 2 * H1 + o);
#pragma unroll
    for (int i = 0; i < H1; ++i) acc += w(off + o * H1 + i) * hdn[i];
    out[o] = M<Real>::th(acc);
  }
  a0 = out[0];
  a1 = out[1];
}

// [5, H1, 2], theta in registers.
template <typename Real, int H1>
struct NetReg {
  static constexpr int P = 6 * H1 + (H1 + 1) * 2;
  static constexpr int kP = P;
  static constexpr int kH1 = H1;
  Real w[P];
  __device__ __forceinline__ void set(int i, Real v) { w[i] = v; }
  __device__ __forceinline__ void eval(const Real s[5], Real& a0, Real& a1) const {
    mlp_5h2<Real, H1>([&](int i) { return w[i]; }, s, a0, a1);
  }
};

// [5, A, B, 2], theta in registers (FP32 [5,10,10,2]: 192 parameters, two
// CTAs of 128 threads per SM at <= 255 registers).
template <typename Real, int A, int B>
struct NetReg3 {
  static constexpr int P = 6 * A + (A + 1) * B + (B + 1) * 2;
  static constexpr int kP = P;
  Real w[P];
  __device__ __forceinline__ void set(int i, Real v) { w[i] = v; }
  __device__ __forceinline__ void eval(const Real s[5], Real& a0, Real& a1) const {
    Real h1[A], h2[B];
#pragma unroll
    for (int o = 0; o < A; ++o) {
      Real acc = w[5 * A + o];
#pragma unroll
      for (int i = 0; i < 5; ++i) acc += w[o * 5 + i] * s[i];
      h1[o] = M<Real>::th(acc);
    }
    constexpr int off2 = 6 * A;
#pragma unroll
    for (int o = 0; o < B; ++o) {
      Real acc = w[off2 + A * B + o];
#pragma unroll
      for (int i = 0; i < A; ++i) acc += w[off2 + o * A + i] * h1[i];
      h2[o] = M<Real>::th(acc);
    }
    constexpr int off3 = off2 + (A + 1) * B;
    Real out[2];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      Real acc = w[off3 + 2 * B + o];
#pragma unroll
      for (int i = 0; i < B; ++i) acc += w[off3 + o * B + i] * h2[i];
      out[o] = M<Real>::th(acc);
    }
    a0 = out[0];
    a1 = out[1];
  }
};

// Any architecture (sizes <= 256): theta in a per-lane column of a global
// scratch buffer (coalesced across the warp), activations in local memory.
template <typename Real>
struct NetGlobal {
  static constexpr int kP = 0;
  Real* col;  // element i at col[i * stride]
  int stride;
  const int32_t* sizes;
  int n_layers;
  __device__ __forceinline__ void set(int i, Real v) { col[static_cast<size_t>(i) * stride] = v; }
  __device__ void eval(const Real s[5], Real& a0, Real& a1) const {
    Real buf[2][256];
    for (int i = 0; i < 5; ++i) buf[0][i] = s[i];
    int cur = 0;
    size_t off = 0;
    for (int l = 0; l + 1 < n_layers; ++l) {
      const int nin = sizes[l], nout = sizes[l + 1];
      for (int o = 0; o < nout; ++o) {
        Real acc = col[(off + static_cast<size_t>(nin) * nout + o) * stride];
        for (int i = 0; i < nin; ++i) {
          acc += col[(off + static_cast<size_t>(o) * nin + i) * stride] * buf[cur][i];
        }
        buf[1 - cur][o] = M<Real>::th(acc);
      }
      off += static_cast<size_t>(nin + 1) * nout;
      cur = 1 - cur;
    }
    a0 = buf[cur][0];
    a1 = buf[cur][1];
  }
};

// ------------------------------------------------------------- sample ----
// theta for candidate c of a restart (src/planner.cpp:207-226): c == 0 is the
// centre; otherwise sigma first, then Box-Muller pairs (cos value first). The
// stream is evaluated in FP64, then rounded to Real; `put(i, v)` stores it.
// In injected mode row `c` of the injected matrix is used instead.
template <typename Real, int KP, class Put>
__device__ __forceinline__ void draw_theta(const RoundArgs& a, uint64_t prefix, int64_t c,
                                           int Pdyn, Put&& put) {
  const int P = KP > 0 ? KP : Pdyn;
  const double* center = a.center;
  if (a.injected != nullptr) {
    const double* src = a.injected + c * P;
#pragma unroll
    for (int i = 0; i < P; ++i) put(i, Real(src[i]));
    return;
  }
  if (c == 0) {
#pragma unroll
    for (int i = 0; i < P; ++i) put(i, Real(__ldg(center + i)));
    return;
  }
  Stream g{fold(prefix, static_cast<uint64_t>(c))};
  if constexpr (sizeof(Real) == sizeof(float)) {
    // FP32 path: the integer stream is exact; the Box-Muller transform runs in
    // float (theta agrees with the FP64 draw to a few float ulps, well inside
    // the FP32 parity tolerance; the host regenerates the winner in FP64).
    const float sigma =
        exp10f(static_cast<float>(a.sig_lo + unit53(g.next()) * a.sig_span));
#pragma unroll
    for (int i = 0; i < P; i += 2) {
      // float(1 - unit53) and float(unit53) straight from the integers:
      // 1 - m 2^-53 = (2^53 - m) 2^-53 exactly, and scaling by 2^-53 commutes
      // with rounding to float
      const uint64_t m1 = g.next() >> 11, m2 = g.next() >> 11;
      const float u1 = __ull2float_rn((1ull << 53) - m1) * 0x1.0p-53f;
      const float u2 = __ull2float_rn(m2) * 0x1.0p-53f;
      const float r = sqrtf(-2.0f * logf(u1));
      // sincos(2 pi u2): quarter-turn reduction t = 4 u2 - q is exact
      const float q = rintf(4.0f * u2);
      const float t = fmaf(4.0f, u2, -q) * 1.57079632679489662f;
      const float sp = sin_poly(t), cp = cos_poly(t);
      const int qi = static_cast<int>(q);
      float sn = (qi & 1) ? cp : sp;
      float cs = (qi & 1) ? sp : cp;
      sn = (qi & 2) ? -sn : sn;
      cs = ((qi + 1) & 2) ? -cs : cs;
      put(i, Real(static_cast<float>(__ldg(center + i)) + sigma * (r * cs)));
      if (i + 1 < P) put(i + 1, Real(static_cast<float>(__ldg(center + i + 1)) + sigma * (r * sn)));
    }
  } else {
    const double sigma = pow(10.0, a.sig_lo + unit53(g.next()) * a.sig_span);
#pragma unroll
    for (int i = 0; i < P; i += 2) {
      const double u1 = 1.0 - unit53(g.next());
      const double u2 = unit53(g.next());
      const double r = sqrt(-2.0 * log(u1));
      const double t = kTwoPi * u2;
      double sn, cs;
      sincos(t, &sn, &cs);
      put(i, Real(__ldg(center + i) + sigma * (r * cs)));
      if (i + 1 < P) put(i + 1, Real(__ldg(center + i + 1) + sigma * (r * sn)));
    }
  }
}

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
  int Ns, Nd;
  int ncx, ncy;
};

template <typename Real>
__device__ __forceinline__ Field<Real> field_at(const RoundArgs& a, const void* base,
                                                const FieldLayout& l) {
  using R2 = typename Vec2T<Real>::type;
  const unsigned char* p = static_cast<const unsigned char*>(base);
  return Field<Real>{reinterpret_cast<const R2*>(p), reinterpret_cast<const R2*>(p + l.dpts),
                     reinterpret_cast<const int*>(p + l.sst),
                     reinterpret_cast<const int*>(p + l.dst),
                     reinterpret_cast<const R2*>(p + l.sbox), a.field_ns, a.field_nd, a.grid_nx,
                     a.grid_ny};
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
template <>
__device__ __forceinline__ float point_margin<float>(const Consts<float>& K, float, float,
                                                     float c, float s, float kx, float ky,
                                                     float mx, float my) {
  const float bx = fmaf(c, mx, fmaf(s, my, -kx));
  const float by = fmaf(-s, mx, fmaf(c, my, -ky));
  return fminf(K.bhx - fabsf(bx), K.hw - fabsf(by));
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
  if constexpr (kGrid == 0) {  // x-buckets: the window is one contiguous range
    const int lo = st[cx_lo];
    const int cnt = st[cx_hi + 1] - lo;
    const int rounds = __reduce_max_sync(kFull, cnt);
    for (int j = 0; j < rounds; ++j) {
      if (j < cnt) {
        const auto m = pts[lo + j];
        best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
      }
    }
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

template <typename Real>
__device__ __forceinline__ void scan_boxed(const typename Vec2T<Real>::type* pts, const int* st,
                                           const typename Vec2T<Real>::type* box, int ncy,
                                           int cx_lo, int cx_hi, int cy_lo, int cy_hi,
                                           const Consts<Real>& K, Real x, Real y, Real c, Real s,
                                           Real kx, Real ky, Real stop, Real& best) {
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
    // dense columns: cell by cell behind the box test
    const int rows = __reduce_max_sync(kFull, dense ? nrow : 0);
    for (int q = 0; q < rows; ++q) {
      int clo = 0, cnt = 0;
      if (dense && q < nrow && best < stop) {
        const int cell = cell0 + q;
        clo = st[cell];
        cnt = st[cell + 1] - clo;
        if (cnt > 0) {
          const auto m = box[2 * cell], e = box[2 * cell + 1];
          const Real du = fabs(c * m.x + s * m.y - kx), dv = fabs(-s * m.x + c * m.y - ky);
          if (du > K.bhx + e.x * ac + e.y * as + K.qpad ||
              dv > K.hw + e.x * as + e.y * ac + K.qpad) {
            cnt = 0;
          }
        }
      }
      for (int j = 0; __any_sync(kFull, j < cnt && best < stop); ++j) {
        if (j < cnt && best < stop) {
          const auto m = pts[clo + j];
          best = fmax(best, point_margin<Real>(K, x, y, c, s, kx, ky, m.x, m.y));
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

// Collision of the chassis at (x, y, phi) with the field at state h. Only the
// cells covering the world-frame bounding box of the chassis rectangle (+ a
// pad of an eighth of a cell) are visited: the reference reports a point
// inside only if it lies strictly inside the rectangle (src/geometry.cpp:
// 63-76), so every point outside that box is a miss whatever the rounding.
// Returns the inside-margin max over visited points (the reference reports a
// collision iff it is > 0; a small |margin| marks a verdict rounding could
// flip). Warp-synchronous: all 32 lanes call it, every loop is warp-uniform.
template <typename Real, int kGrid>
__device__ __forceinline__ Real collide_margin(const Field<Real>& f, const Consts<Real>& K, int h,
                                               Real x, Real y, Real c, Real s, Real stop) {
  const int ncx = f.ncx, ncy = f.ncy;
  const Real ac = fabs(c), as = fabs(s);
  const Real top = Real(ncx - 1);
  // rectangle centre (x, y) + bcx (c, s); half extents bhx |c| + hw |s| (x)
  const Real ox = x + K.bcx * c - K.bx0;
  const Real ex = K.bhx * ac + K.hw * as + K.qpad;
  const int cx_lo = static_cast<int>(fmin(fmax((ox - ex) * K.binv, Real(0)), top));
  const int cx_hi = static_cast<int>(fmin(fmax((ox + ex) * K.binv, Real(0)), top));
  int cy_lo = 0, cy_hi = 0;
  if constexpr (kGrid) {
    const Real ytop = Real(ncy - 1);
    const Real oy = y + K.bcx * s - K.by0;
    const Real ey = K.bhx * as + K.hw * ac + K.qpad;
    cy_lo = static_cast<int>(fmin(fmax((oy - ey) * K.binv, Real(0)), ytop));
    cy_hi = static_cast<int>(fmin(fmax((oy + ey) * K.binv, Real(0)), ytop));
  }
  const Real kx = c * x + s * y + K.bcx;  // FP32 rotated-frame form only
  const Real ky = -s * x + c * y;
  Real best = Real(-1e30);
  // part 0: static points; part 1: the dynamic row of state h (one copy of
  // the scan code, warp-uniform part loop)
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    const bool dyn = part == 1;
    if ((dyn ? f.Nd : f.Ns) == 0) continue;
    const auto* pts = dyn ? f.dpts + static_cast<size_t>(h) * f.Nd : f.spts;
    const int* st = dyn ? f.dst + static_cast<size_t>(h) * (ncx * ncy + 1) : f.sst;
    if constexpr (kGrid == 2) {
      if (!dyn) {
        scan_boxed<Real>(pts, st, f.sbox, ncy, cx_lo, cx_hi, cy_lo, cy_hi, K, x, y, c, s, kx, ky,
                         stop, best);
        continue;
      }
    }
    scan_part<Real, kGrid>(pts, st, ncy, cx_lo, cx_hi, cy_lo, cy_hi, K, x, y, c, s, kx, ky, stop,
                           best);
  }
  return best;
}

// One candidate's rollout state (src/planner.cpp:123-125, 130-132).
template <typename Real>
struct Lane {
  Real x, y, phi, v, act, pa0, path, f0, f1, ephi;
  int h;
  bool marg;  // a worse-side collision / goal verdict came within K.dmarg of flipping
  __device__ __forceinline__ void start(const Consts<Real>& K, Real first0, Real first1) {
    x = y = phi = Real(0);
    v = K.v0;
    act = K.act0;
    pa0 = K.pa0;
    path = Real(0);
    f0 = first0;
    f1 = first1;
    h = 0;
    marg = false;
  }
};

// Features of the EV-at-start state: identical for every candidate.
template <typename Real>
__device__ __forceinline__ void start_features(const Consts<Real>& K, Real s[5]) {
  s[0] = M<Real>::ndiv(K.gx - Real(0), K.d_xi, K.inv_xi);
  s[1] = M<Real>::ndiv(K.gy - Real(0), K.d_eta, K.inv_eta);
  s[2] = M<Real>::ndiv(M<Real>::wrap(K.gphi - Real(0)), K.d_phi, K.inv_phi);
  s[3] = M<Real>::ndiv(K.gv - K.v0, K.d_v, K.inv_v);
  s[4] = K.pa0;
}

// One state of the rollout loop (src/planner.cpp:137-183). Returns -1 while
// running, else the class (0 collided, 1 horizon, 2 reached at state h).
// Warp-synchronous and branch-free: the checks and the next state are
// computed for every lane and committed only by the lanes still running,
// so the warp never splits into per-outcome paths.
template <typename Real, int kGrid, class Net>
__device__ __forceinline__ int advance(Lane<Real>& L, const Net& net, const Consts<Real>& K,
                                       const Field<Real>& f, int H) {
  Real sphi, cphi;
  M<Real>::sc(L.phi, &sphi, &cphi);
  L.ephi = M<Real>::wrap(K.gphi - L.phi);
  bool hit = false;
  if (f.Ns + f.Nd > 0) {
    // a lane may stop at a hit whose margin is too large to flip
    const Real cm = collide_margin<Real, kGrid>(f, K, L.h, L.x, L.y, cphi, sphi, K.dmarg);
    hit = cm > Real(0);
    // a narrow hit might be free in exact arithmetic (a better outcome)
    L.marg |= hit & (cm < K.dmarg);
  }
  const Real gdx = K.gx - L.x, gdy = K.gy - L.y;
  // inclusive goal box: eps - |err| >= 0 <=> |err| <= eps, exactly
  const Real gm = fmin(fmin(K.eps_xi - M<Real>::ab(K.gcos * gdx + K.gsin * gdy),
                            K.eps_eta - M<Real>::ab(-K.gsin * gdx + K.gcos * gdy)),
                       fmin(K.eps_phi - M<Real>::ab(L.ephi), K.eps_v - M<Real>::ab(K.gv - L.v)));
  const bool reached = gm >= Real(0);
  // a narrow miss might reach in exact arithmetic (a better outcome)
  L.marg |= !reached & (gm > -K.dmarg);
  const int cls = hit ? 0 : (reached ? 2 : (L.h == H ? 1 : -1));

  Real s[5];
  s[0] = M<Real>::ndiv(gdx, K.d_xi, K.inv_xi);
  s[1] = M<Real>::ndiv(gdy, K.d_eta, K.inv_eta);
  s[2] = M<Real>::ndiv(L.ephi, K.d_phi, K.inv_phi);
  s[3] = M<Real>::ndiv(K.gv - L.v, K.d_v, K.inv_v);
  s[4] = L.pa0;
  Real a0, a1;
  net.eval(s, a0, a1);
  if (L.h == 0) {  // the first action was computed before the loop
    a0 = L.f0;
    a1 = L.f1;
  }
  // map_controls (src/dynamics.cpp:30-43)
  const Real c0 = clampr(a0, Real(-1), Real(1));
  const Real c1 = clampr(a1, Real(-1), Real(1));
  Real delta = clampr(K.dmax * c0, L.act - K.window, L.act + K.window);
  delta = clampr(delta, -K.dmax, K.dmax);
  const Real w = Real(0.5) * (c1 + Real(1));
  const Real u_v = (Real(1) - w) * K.umin + w * K.umax;
  // explicit Euler (src/dynamics.cpp:45-62)
  const Real tan_d = K.tan_small ? M<Real>::tn_small(delta) : M<Real>::tn(delta);
  const Real tb = M<Real>::ndiv(K.l_r * tan_d, K.wb_d, K.inv_wb);
  const Real tv = K.Ts * L.v;
  const Real nx = L.x + tv * (cphi - tb * sphi);
  const Real ny = L.y + tv * (sphi + tb * cphi);
  const Real nphi = L.phi + M<Real>::ndiv(tv * tan_d, K.wb_d, K.inv_wb);
  const Real nv = L.v + K.Ts * u_v;
  const Real dx = nx - L.x, dy = ny - L.y;
  const Real seg = M<Real>::sq(dx * dx + dy * dy);
  if (cls < 0) {
    L.path += seg;
    L.x = nx;
    L.y = ny;
    L.phi = nphi;
    L.v = nv;
    L.act = delta;
    L.pa0 = a0;
    ++L.h;
  }
  return cls;
}

// src/planner.cpp:186-189 at the final state (L.ephi is that state's).
template <typename Real>
__device__ __forceinline__ Real terminal_cost(const Lane<Real>& L, const Consts<Real>& K) {
  return M<Real>::ndiv(M<Real>::ab(K.gx - L.x), K.d_xi, K.inv_xi) +
         M<Real>::ndiv(M<Real>::ab(K.gy - L.y), K.d_eta, K.inv_eta) +
         M<Real>::ndiv(M<Real>::ab(L.ephi), K.d_phi, K.inv_phi) +
         M<Real>::ndiv(M<Real>::ab(K.gv - L.v), K.d_v, K.inv_v);
}

// ---------------------------------------------------------- reduction ----
// Lexicographic (cls, k1, k2) descending, index ascending: a total order, so
// any reduction tree gives the reference's "strict better, lowest index
// wins" result (src/planner.cpp:40-44, 295, 316).
struct Key {
  int cls;
  int idx;
  double k1, k2;
};

__device__ __forceinline__ Key empty_key() { return Key{-1, -1, 0.0, 0.0}; }

__device__ __forceinline__ bool prefer(const Key& a, const Key& b) {
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  if (a.k2 != b.k2) return a.k2 > b.k2;
  return static_cast<unsigned>(a.idx) < static_cast<unsigned>(b.idx);
}

template <typename Real>
__device__ __forceinline__ Key make_key(int cls, int h, Real path, Real term, int idx) {
  Key k;  // src/planner.cpp:27-38
  k.cls = cls;
  k.idx = idx;
  if (cls == 2) {
    k.k1 = -static_cast<double>(h);
    k.k2 = -static_cast<double>(path);
  } else {
    k.k1 = -static_cast<double>(term);
    k.k2 = 0.0;
  }
  return k;
}

__device__ __forceinline__ Key shfl_key(const Key& k, int off) {
  Key o;
  o.cls = __shfl_down_sync(kFull, k.cls, off);
  o.idx = __shfl_down_sync(kFull, k.idx, off);
  o.k1 = __shfl_down_sync(kFull, k.k1, off);
  o.k2 = __shfl_down_sync(kFull, k.k2, off);
  return o;
}

// Warp argmin; result valid in lane 0.
__device__ __forceinline__ Key warp_best(Key k) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Key o = shfl_key(k, off);
    if (prefer(o, k)) k = o;
  }
  return k;
}

// Block argmin; result valid in thread 0. `scratch` holds >= 32 keys.
__device__ __forceinline__ Key block_best(Key k, Key* scratch) {
  k = warp_best(k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = k;
  __syncthreads();
  if (warp == 0) {
    k = lane < static_cast<int>(blockDim.x >> 5) ? scratch[lane] : empty_key();
    k = warp_best(k);
  }
  __syncthreads();
  return k;
}

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v,
                                                        unsigned long long* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < static_cast<int>(blockDim.x >> 5) ? scratch[lane] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  }
  __syncthreads();
  return v;
}

__device__ __forceinline__ Key load_rec_cg(const Rec* src) {
  // written by other CTAs: read through L2 (ld.global.cg), never L1
  return Key{__ldcg(&src->cls), __ldcg(&src->cand), __ldcg(&src->k1), __ldcg(&src->k2)};
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor drains; it waits here (the
// predecessor has completed and its writes are visible) before reading what
// the predecessor wrote. A no-op for an ordinary launch.
__device__ __forceinline__ void wait_prior_grid() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Field of the round, staged whole into shared memory when it fits
// (a.field_smem_bytes > 0), else read through L1/L2. The staging is one TMA
// bulk copy (cp.async.bulk, global -> shared) issued by thread 0 and
// completed on an mbarrier (transaction count = the image size, a multiple
// of 16 bytes, <= 40 KB); every thread waits on the barrier's phase 0.
__device__ __forceinline__ void bulk_stage(unsigned char* dst, const void* src, uint32_t bytes,
                                           uint64_t* mbar) {
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  if (threadIdx.x == 0) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
  }
  __syncthreads();  // the barrier is initialised before anyone polls it
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(bar)
      : "memory");
}

template <typename Real>
__device__ __forceinline__ Field<Real> stage_field(const RoundArgs& a, unsigned char* smem) {
  __shared__ __align__(8) uint64_t stage_bar;
  if (a.field_smem_bytes > 0 && a.n_points > 0) {
    bulk_stage(smem, a.field, static_cast<uint32_t>(a.field_smem_bytes), &stage_bar);
    return field_at<Real>(a, smem, a.lay);
  }
  __syncthreads();
  return field_at<Real>(a, a.field, a.lay);
}

// Compact per-sample key for the near-tie re-ranking (select_kernel):
// cost = terminal cost (cls 0/1) or path length (cls 2); meta = cls | marg<<2
// | t_goal<<8.
template <typename Real>
__device__ __forceinline__ void write_skey(const RoundArgs& a, int64_t slot, int cls,
                                           const Lane<Real>& L, Real term) {
  if (a.skeys == nullptr) return;
  const uint32_t meta = static_cast<uint32_t>(cls) | (L.marg ? 4u : 0u) |
                        (static_cast<uint32_t>(cls == 2 ? L.h : 0) << 8);
  if constexpr (sizeof(Real) == sizeof(float)) {
    static_cast<SKey32*>(a.skeys)[slot] = SKey32{cls == 2 ? L.path : term, meta};
  } else {
    static_cast<SKey*>(a.skeys)[slot] = SKey{cls == 2 ? L.path : term, meta, 0u};
  }
}

// Per-sample debug/parity record.
template <typename Real>
__device__ __forceinline__ void write_sample(const RoundArgs& a, int64_t slot, int cls,
                                             const Lane<Real>& L, Real term) {
  SampleOut& so = a.per_sample[slot];
  so.reached = cls == 2;
  so.t_goal = cls == 2 ? L.h : -1;
  so.collided = cls == 0;
  so.steps = L.h;
  so.path_length = static_cast<double>(L.path);
  so.terminal_cost = static_cast<double>(term);
  so.first_a0 = static_cast<double>(L.f0);
  so.first_a1 = static_cast<double>(L.f1);
}

// Last CTA: per-restart reduction of `n_src` records per restart (laid out
// restart-major), publish the work counters, re-arm the tickets.
// Last-block election over the whole grid (the ticket is re-armed by
// publish_round).
__device__ __forceinline__ bool last_block(const RoundArgs& a) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  const unsigned n_blocks = gridDim.x * gridDim.y;
  if (threadIdx.x == 0) s_last = atomicAdd(&a.counters[1], 1u) == n_blocks - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Per-restart reduction of `n_src` records per restart (restart-major) into
// out[restart].
__device__ __forceinline__ void reduce_recs(const RoundArgs& a, const Rec* recs, int n_src,
                                            Key* red, Rec* out) {
  for (int r = 0; r < a.restart_count; ++r) {
    Key k = empty_key();
    for (int t = threadIdx.x; t < n_src; t += blockDim.x) {
      const Key o = load_rec_cg(recs + static_cast<size_t>(r) * n_src + t);
      if (o.cls >= 0 && (k.cls < 0 || prefer(o, k))) k = o;
    }
    const Key best = block_best(k, red);
    if (threadIdx.x == 0) out[r] = Rec{best.cls, best.idx, best.k1, best.k2};
  }
}

// Publish the work counters and re-arm the tickets (last block only).
__device__ __forceinline__ void publish_round(const RoundArgs& a) {
  if (threadIdx.x == 0) {
    a.exec[2] = atomicExch(&a.exec[0], 0ull);
    a.exec[3] = atomicExch(&a.exec[1], 0ull);
    a.counters[0] = 0;
    a.counters[1] = 0;
    a.counters[2] = 0;  // the window selection that follows counts from zero
  }
}

__device__ __forceinline__ void finish_round(const RoundArgs& a, const Rec* recs, int n_src,
                                             Key* red) {
  if (!last_block(a)) return;
  reduce_recs(a, recs, n_src, red, a.out);
  publish_round(a);
}

// Warp-cooperative flush of the lanes' best keys (flagged by `flush`) into
// the warp's per-restart shared table, one restart at a time.
__device__ __forceinline__ void flush_bests(bool& flush, Key& best, int best_r, Key* table_w,
                                            int lane) {
  unsigned pend = __ballot_sync(kFull, flush);
  while (pend != 0u) {
    const int r0 = __shfl_sync(kFull, best_r, __ffs(pend) - 1);
    const bool mine = flush && best_r == r0;
    const Key k = warp_best(mine ? best : empty_key());
    if (lane == 0 && (table_w[r0].cls < 0 || prefer(k, table_w[r0]))) table_w[r0] = k;
    if (mine) {
      flush = false;
      best = empty_key();
    }
    pend = __ballot_sync(kFull, flush);
  }
}

// --------------------------------------------------- generate kernel ----
// theta (rounded to Real) and the first action of every candidate of the
// round, one thread per candidate at full SIMT width: the FP64 RNG lives here
// and not in the rollout kernel, so the rollout kernel stays register-light.
// Layout: one record of kRecW(P) Reals per candidate, [theta 0..P-1][f0][f1]
// [pad], so a refilling lane loads it with 16-byte vector loads; the flat
// index is s = r * count + local (restart-major).
template <typename Real>
constexpr int rec_width(int P) {
  return ((P + 2) * static_cast<int>(sizeof(Real)) + 15) / 16 * 16 / static_cast<int>(sizeof(Real));
}
template <typename Real>
using Vec16 = typename std::conditional<sizeof(Real) == 4, float4, double2>::type;

template <typename Real, class Net>
__global__ void __launch_bounds__(256) generate_kernel(const RoundArgs a) {
  constexpr int P = Net::P;
  constexpr int W = rec_width<Real>(P);
  constexpr int V = W * static_cast<int>(sizeof(Real)) / 16;
  const Consts<Real>& K = consts_of<Real>(a);
  Real s0[5];
  start_features(K, s0);
  Vec16<Real>* recs = static_cast<Vec16<Real>*>(a.theta_buf);
  const int64_t total = a.count * a.restart_count;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // restart of flat index s (32-bit division when the round is small)
    const int r = total <= 0x7fffffff
                      ? static_cast<int>(static_cast<uint32_t>(s) / static_cast<uint32_t>(a.count))
                      : static_cast<int>(s / a.count);
    const int64_t local = s - static_cast<int64_t>(r) * a.count;
    union {
      Real v[W];
      Vec16<Real> q[V];
    } rec;
    draw_theta<Real, P>(a, __ldg(a.key_prefix + r), a.injected ? local : a.cand_begin + local, P,
                        [&](int i, Real v) { rec.v[i] = v; });
    Net n;
#pragma unroll
    for (int i = 0; i < P; ++i) n.w[i] = rec.v[i];
    n.eval(s0, rec.v[P], rec.v[P + 1]);  // first action (src/planner.cpp:130-132)
#pragma unroll
    for (int i = P + 2; i < W; ++i) rec.v[i] = Real(0);
#pragma unroll
    for (int j = 0; j < V; ++j) recs[s * V + j] = rec.q[j];
  }
}

// ------------------------------------------------------ refill kernel ----
// Resident CTAs per SM the register allocation must allow: [5,2,2] in FP32
// fits 6 (<= 85 registers), wider nets and FP64 need more registers.
template <typename Real, class Net>
constexpr int refill_min_blocks() {
  return sizeof(Real) == 4 ? (Net::kP <= 24 ? PARAPLAN_REFILL_MINB : (Net::kP <= 100 ? 3 : 2))
                           : (Net::kP <= 24 ? 4 : 2);
}

template <typename Real, class Net, int kGrid>
__global__ void __launch_bounds__(kBlock, refill_min_blocks<Real, Net>())
    refill_kernel(const RoundArgs a) {
  constexpr int P = Net::kP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Key table[kWarps][kMaxRestartsPerLaunch];
  __shared__ Key red[32];
  __shared__ unsigned long long red_sum[32];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Consts<Real>& K = consts_of<Real>(a);
  const int H = a.H;
  for (int i = threadIdx.x; i < kWarps * kMaxRestartsPerLaunch; i += blockDim.x) {
    (&table[0][0])[i] = empty_key();
  }
  const Field<Real> f = stage_field<Real>(a, smem_raw);
  wait_prior_grid();  // the generator's theta records

  const int bpr = a.tiles_per_restart;  // 32-candidate batches per restart
  const unsigned total_batches = static_cast<unsigned>(a.n_tiles);
  constexpr int W = rec_width<Real>(P);
  constexpr int V = W * static_cast<int>(sizeof(Real)) / 16;
  const Vec16<Real>* recs = static_cast<const Vec16<Real>*>(a.theta_buf);

  Net net;
#pragma unroll
  for (int i = 0; i < P; ++i) net.w[i] = Real(0);
  Lane<Real> L;
  L.start(K, Real(0), Real(0));  // idle lanes step a valid (discarded) state
  bool active = false;
  int my_r = 0;
  int my_c = 0;  // local candidate index within [0, count)
  Key best = empty_key();
  int best_r = -1;
  int q_head = 32, q_count = 0, q_r = 0, q_c0 = 0;
  // claimed batch range [qb, qe): with several restarts a warp claims runs of
  // consecutive batches, so its lanes rarely cross restarts (each crossing
  // flushes lane bests into the per-restart tables); single batches near the
  // end of the round keep the tail balanced
  unsigned qb = 0, qe = 0;
  const unsigned run = a.restart_count > 1 ? 8u : 1u;
  const unsigned tail = static_cast<unsigned>(gridDim.x) * kWarps * 2u * run;
  bool exhausted = false;
  unsigned long long n_steps = 0, n_states = 0;
  const bool track = a.keys_only == 0;  // lane bests (one restart) or keys only

  for (;;) {
    // -------- hand the warp's current batch to idle lanes --------
    const unsigned need = __ballot_sync(kFull, !active);
    if (need != 0u) {
      if (q_head >= q_count && !exhausted) {
        if (qb >= qe) {
          unsigned b = 0;
          if (lane == 0) {
            const unsigned seen = __ldcg(&a.counters[0]);
            const unsigned k = seen + tail < total_batches ? run : 1u;
            b = atomicAdd(&a.counters[0], k);
            qe = min(b + k, total_batches);
          }
          b = __shfl_sync(kFull, b, 0);
          qe = __shfl_sync(kFull, qe, 0);
          qb = b;
        }
        if (qb >= total_batches) {
          exhausted = true;
        } else {
          q_r = static_cast<int>(qb) / bpr;
          q_c0 = (static_cast<int>(qb) - q_r * bpr) * 32;
          const int64_t left = a.count - q_c0;
          q_count = left < 32 ? static_cast<int>(left) : 32;
          q_head = 0;
          ++qb;
        }
      }
      const int avail = q_count - q_head;
      if (avail > 0) {
        const int rank = __popc(need & ((1u << lane) - 1u));
        if (!active && rank < avail) {
          my_r = q_r;
          my_c = q_c0 + q_head + rank;
          const int64_t sidx = static_cast<int64_t>(my_r) * a.count + my_c;
          // contiguous record: one address, immediate offsets, no extra registers
          const Real* rp = reinterpret_cast<const Real*>(recs + sidx * V);
#pragma unroll
          for (int i = 0; i < P; ++i) net.w[i] = __ldg(rp + i);
          L.start(K, __ldg(rp + P), __ldg(rp + P + 1));
          active = true;
        }
        q_head += __popc(need) < avail ? __popc(need) : avail;
      }
    }
    if (!__any_sync(kFull, active)) break;  // stream exhausted, all lanes done

    // -------- one rollout state per lane --------
    // every lane steps (idle lanes only at the stream tail, results unused)
    const int cls = advance<Real, kGrid>(L, net, K, f, H);
    const bool done = active && cls >= 0;
    // lane bests are per restart: flush the old one before crossing over
    bool flush = track && done && best.cls >= 0 && best_r != my_r;
    if (__any_sync(kFull, flush)) flush_bests(flush, best, best_r, table[warp], lane);
    if (done) {
      const Real term = terminal_cost(L, K);
      if (track) {
        const Key k =
            make_key<Real>(cls, L.h, L.path, term, static_cast<int>(a.cand_begin + my_c));
        if (best.cls < 0 || prefer(k, best)) {
          best = k;
          best_r = my_r;
        }
      }
      n_steps += static_cast<unsigned long long>(L.h);
      n_states += static_cast<unsigned long long>(L.h + 1);
      if (a.per_sample != nullptr) {
        write_sample(a, static_cast<int64_t>(my_r) * a.count + my_c, cls, L, term);
      }
      write_skey(a, static_cast<int64_t>(my_r) * a.count + my_c, cls, L, term);
      active = false;
    }
  }

  // -------- flush lane bests, combine warps, publish CTA records --------
  const unsigned long long steps = block_sum(n_steps, red_sum);
  const unsigned long long states = block_sum(n_states, red_sum);
  if (threadIdx.x == 0) {
    atomicAdd(&a.exec[0], steps);
    atomicAdd(&a.exec[1], states);
  }
  if (!track) return;  // reduce_keys_kernel forms the winners
  bool flush = best.cls >= 0;
  flush_bests(flush, best, best_r, table[warp], lane);
  __syncthreads();
  for (int r = threadIdx.x; r < a.restart_count; r += blockDim.x) {
    Key k = table[0][r];
    for (int w = 1; w < kWarps; ++w) {
      if (table[w][r].cls >= 0 && (k.cls < 0 || prefer(table[w][r], k))) k = table[w][r];
    }
    a.tile_recs[static_cast<size_t>(r) * gridDim.x + blockIdx.x] = Rec{k.cls, k.idx, k.k1, k.k2};
  }
  finish_round(a, a.tile_recs, static_cast<int>(gridDim.x), red);
}

// Per-restart winners from the sample keys (RoundArgs::keys_only): block
// (x, r) reduces chunk x of restart r; the last block reduces the chunks.
// The keys are the rollout's own: (cls, t_goal, FP32 cost) give the same
// (cls, k1, k2) as make_key, and the index is the slot's.
static __global__ void __launch_bounds__(256) reduce_keys_kernel(const RoundArgs a) {
  __shared__ Key red[32];
  wait_prior_grid();  // the rollout's keys
  const int r = blockIdx.y;
  const int64_t chunk = (a.count + gridDim.x - 1) / gridDim.x;
  const int64_t lo = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t hi = lo + chunk < a.count ? lo + chunk : a.count;
  Key k = empty_key(), kf = empty_key();  // best, best not flagged marginal
  for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) {
    const int64_t slot = static_cast<int64_t>(r) * a.count + c;
    double cost;
    uint32_t meta;
    if (a.skey32) {
      const SKey32 q = static_cast<const SKey32*>(a.skeys)[slot];
      cost = static_cast<double>(q.cost);
      meta = q.meta;
    } else {
      const SKey q = static_cast<const SKey*>(a.skeys)[slot];
      cost = q.cost;
      meta = q.meta;
    }
    Key o;
    o.cls = static_cast<int>(meta & 3u);
    o.idx = static_cast<int>(a.cand_begin + c);
    if (o.cls == 2) {
      o.k1 = -static_cast<double>(meta >> 8);
      o.k2 = -cost;
    } else {
      o.k1 = -cost;
      o.k2 = 0.0;
    }
    if (k.cls < 0 || prefer(o, k)) k = o;
    if ((meta & 4u) == 0u && (kf.cls < 0 || prefer(o, kf))) kf = o;
  }
  k = block_best(k, red);
  kf = block_best(kf, red);
  const unsigned n_src = gridDim.x;
  Rec* tiles_free = a.tile_recs + static_cast<size_t>(a.restart_count) * n_src;
  if (threadIdx.x == 0) {
    a.tile_recs[static_cast<size_t>(r) * n_src + blockIdx.x] = Rec{k.cls, k.idx, k.k1, k.k2};
    tiles_free[static_cast<size_t>(r) * n_src + blockIdx.x] = Rec{kf.cls, kf.idx, kf.k1, kf.k2};
  }
  if (!last_block(a)) return;
  reduce_recs(a, a.tile_recs, static_cast<int>(n_src), red, a.out);
  if (a.out_free != nullptr) reduce_recs(a, tiles_free, static_cast<int>(n_src), red, a.out_free);
  publish_round(a);
}

// ---------------------------------------------------- lockstep kernel ----
template <typename Real, class Net>
struct NetFactory;

template <typename Real, int H1>
struct NetFactory<Real, NetReg<Real, H1>> {
  static __device__ __forceinline__ NetReg<Real, H1> make(const RoundArgs&) { return {}; }
};
template <typename Real, int A, int B>
struct NetFactory<Real, NetReg3<Real, A, B>> {
  static __device__ __forceinline__ NetReg3<Real, A, B> make(const RoundArgs&) { return {}; }
};

template <typename Real>
struct Scratch;
template <>
struct Scratch<float> {
  static __device__ __forceinline__ float* ptr(const RoundArgs& a) { return a.theta_scratch; }
};
template <>
struct Scratch<double> {
  static __device__ __forceinline__ double* ptr(const RoundArgs& a) { return a.theta_scratch64; }
};

template <typename Real>
struct NetFactory<Real, NetGlobal<Real>> {
  static __device__ __forceinline__ NetGlobal<Real> make(const RoundArgs& a) {
    NetGlobal<Real> n;
    n.stride = a.grid * a.block;
    n.col = Scratch<Real>::ptr(a) + blockIdx.x * a.block + threadIdx.x;
    n.sizes = a.sizes;
    n.n_layers = a.n_layers;
    return n;
  }
};

template <typename Real, class Net, int kGrid>
__global__ void __launch_bounds__(kBlock) lockstep_kernel(const RoundArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Key red[32];
  __shared__ unsigned long long red_sum[32];
  __shared__ int s_tile;

  const Consts<Real>& K = consts_of<Real>(a);
  const int H = a.H;
  const int P = a.n_params;
  const Field<Real> f = stage_field<Real>(a, smem_raw);
  Real s0[5];
  start_features(K, s0);

  Net net = NetFactory<Real, Net>::make(a);
  unsigned long long n_steps = 0, n_states = 0;
  for (;;) {
    if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(&a.counters[0], 1u));
    __syncthreads();
    const int tile = s_tile;
    __syncthreads();
    if (tile >= a.n_tiles) break;
    const int r = tile / a.tiles_per_restart;
    const int64_t local =
        static_cast<int64_t>(tile - r * a.tiles_per_restart) * blockDim.x + threadIdx.x;
    Key key = empty_key();
    const bool valid = local < a.count;
    const int64_t c = a.cand_begin + (valid ? local : 0);
    draw_theta<Real, Net::kP>(a, __ldg(a.key_prefix + r), a.injected ? (valid ? local : 0) : c,
                              P, [&](int i, Real v) { net.set(i, v); });
    Real f0, f1;
    net.eval(s0, f0, f1);
    Lane<Real> L;
    L.start(K, f0, f1);
    int cls = -1;
    // lanes keep stepping (and discarding) until the whole warp is done
    while (__any_sync(kFull, cls < 0)) {
      const int k = advance<Real, kGrid>(L, net, K, f, H);
      if (cls < 0) cls = k;
    }
    if (valid) {
      const Real term = terminal_cost(L, K);
      key = make_key<Real>(cls, L.h, L.path, term, static_cast<int>(c));
      n_steps += static_cast<unsigned long long>(L.h);
      n_states += static_cast<unsigned long long>(L.h + 1);
      if (a.per_sample != nullptr) {
        write_sample(a, static_cast<int64_t>(r) * a.count + local, cls, L, term);
      }
      write_skey(a, static_cast<int64_t>(r) * a.count + local, cls, L, term);
    }
    const Key best = block_best(key, red);
    // tile records are restart-major: [r][tile within restart]
    if (threadIdx.x == 0) a.tile_recs[tile] = Rec{best.cls, best.idx, best.k1, best.k2};
  }
  const unsigned long long steps = block_sum(n_steps, red_sum);
  const unsigned long long states = block_sum(n_states, red_sum);
  if (threadIdx.x == 0) {
    atomicAdd(&a.exec[0], steps);
    atomicAdd(&a.exec[1], states);
  }
  finish_round(a, a.tile_recs, a.tiles_per_restart, red);
}

// ------------------------------------------------------ select kernel ----
// Near-tie window of every restart: candidates of the winner's class whose
// key lies within (1 + rho) * cost + alpha of the round winner, plus every
// candidate flagged marginal. Indices are appended to a.sel_list.
static __global__ void __launch_bounds__(256) select_kernel(const RoundArgs a) {
  wait_prior_grid();  // the rollout's keys and winners
  const int64_t total = a.count * a.restart_count;
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(s / a.count);
    SelBound bd;
    if (a.sel_bound != nullptr) {  // widened window of a later pass
      bd = a.sel_bound[r];
    } else {  // first pass: around the round winner (its best unflagged candidate)
      const Rec b = (a.out_free != nullptr && a.out_free[r].cls >= 0) ? a.out_free[r] : a.out[r];
      bd.cls = b.cls;
      bd.t_goal = b.cls == 2 ? static_cast<int>(-b.k1) : 0;
      bd.thr = (b.cls == 2 ? -b.k2 : -b.k1) * (1.0 + a.sel_rho) + a.sel_alpha;
    }
    SKey k;
    if (a.skey32) {
      const SKey32 k32 = static_cast<const SKey32*>(a.skeys)[s];
      k.cost = static_cast<double>(k32.cost);
      k.meta = k32.meta;
    } else {
      k = static_cast<const SKey*>(a.skeys)[s];
    }
    const int cls = static_cast<int>(k.meta & 3u);
    bool take = (k.meta & 4u) != 0u && bd.cls >= 0;
    if (cls == bd.cls && k.cost <= bd.thr) {
      take |= cls != 2 || static_cast<int>(k.meta >> 8) == bd.t_goal;
    }
    if (take) {
      const unsigned i = atomicAdd(&a.counters[2], 1u);
      if (i < static_cast<unsigned>(a.sel_cap)) a.sel_list[i] = s;
    }
  }
}

// ------------------------------------------------------ refine kernel ----
// FP64 re-evaluation of the selected candidates (theta redrawn in FP64,
// FP64 field). One lane per candidate, warp-synchronous stepping.
template <class Net64>
struct RefineNet;
template <int H1>
struct RefineNet<NetReg<double, H1>> {
  static __device__ __forceinline__ NetReg<double, H1> make(const RoundArgs&) { return {}; }
};
template <>
struct RefineNet<NetGlobal<double>> {
  static __device__ __forceinline__ NetGlobal<double> make(const RoundArgs& a) {
    NetGlobal<double> n;
    n.stride = gridDim.x * blockDim.x;
    n.col = a.theta_scratch64 + blockIdx.x * blockDim.x + threadIdx.x;
    n.sizes = a.sizes;
    n.n_layers = a.n_layers;
    return n;
  }
};

template <class Net64, int kGrid>
__global__ void __launch_bounds__(128) refine_kernel(const RoundArgs a) {
  const Consts<double>& K = a.kd;
  const unsigned n_sel = min(__ldcg(&a.counters[2]), static_cast<unsigned>(a.sel_cap));
  const Field<double> f = field_at<double>(a, a.field64, a.lay64);
  double s0[5];
  start_features(K, s0);
  Net64 net = RefineNet<Net64>::make(a);
  // warp-uniform bound so every lane of a live warp keeps stepping
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n_sel;
       base += stride) {
    const unsigned i = base + (threadIdx.x & 31u);
    const bool valid = i < n_sel;
    const int64_t s = a.sel_list[valid ? i : base];
    const int r = static_cast<int>(s / a.count);
    const int64_t local = s - static_cast<int64_t>(r) * a.count;
    draw_theta<double, Net64::kP>(a, __ldg(a.key_prefix + r),
                                  a.injected ? local : a.cand_begin + local, a.n_params,
                                  [&](int j, double v) { net.set(j, v); });
    double f0, f1;
    net.eval(s0, f0, f1);
    Lane<double> L;
    L.start(K, f0, f1);
    int cls = -1;
    while (__any_sync(kFull, cls < 0)) {
      const int k = advance<double, kGrid>(L, net, K, f, a.H);
      if (cls < 0) cls = k;
    }
    if (valid) {
      const double term = terminal_cost(L, K);
      const Key k = make_key<double>(cls, L.h, L.path, term, static_cast<int>(a.cand_begin + local));
      a.sel_out[i] = SelRec{k.cls, k.idx, r, 0, k.k1, k.k2};
    }
  }
}

// ------------------------------------------------------------ launch ----
// Register-resident nets use the refill schedule; PARAPLAN_SCHEDULE=lockstep
// forces the lockstep schedule (A/B measurements only).
inline bool force_lockstep() {
  static const bool v = [] {
    const char* e = std::getenv("PARAPLAN_SCHEDULE");
    return e != nullptr && std::strcmp(e, "lockstep") == 0;
  }();
  return v;
}

template <class Net>
bool refill_schedule() {
  return Net::kP > 0 && !force_lockstep();
}

using KernelFn = void (*)(const RoundArgs);

// Launch with programmatic stream serialization when `pdl` (the kernel calls
// wait_prior_grid() before reading its predecessor's output).
inline cudaError_t launch_dependent(KernelFn k, int grid, int block, size_t smem, cudaStream_t st,
                                    bool pdl, const RoundArgs& a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <typename Real, class Net, int kGrid>
KernelFn kernel_of_g() {
  if constexpr (Net::kP > 0) {
    if (refill_schedule<Net>()) return refill_kernel<Real, Net, kGrid>;
  }
  return lockstep_kernel<Real, Net, kGrid>;
}

// grid mode of the field (0 x-buckets, 1 2-D, 2 2-D with cell boxes) -- a
// separate instantiation each, so the small-field kernel stays lean.
template <typename Real, class Net>
KernelFn kernel_of(int mode) {
  return mode == 2 ? kernel_of_g<Real, Net, 2>()
                   : (mode == 1 ? kernel_of_g<Real, Net, 1>() : kernel_of_g<Real, Net, 0>());
}

// Stage 1 of a round: the theta generator (refill schedule only; a no-op
// for the lockstep schedule, which draws theta itself).
template <typename Real, class Net>
int launch_generate_impl(const RoundArgs& a, void* stream) {
  if constexpr (Net::kP > 0) {
    if (refill_schedule<Net>()) {
      const int64_t total = a.count * a.restart_count;
      const int gen_blocks = static_cast<int>((total + 255) / 256);
      generate_kernel<Real, Net><<<gen_blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
      return static_cast<int>(cudaGetLastError());
    }
  }
  return 0;
}

// Stage 2: the rollout. After the generator it is a dependent launch (the
// rollout CTAs stage the field while the generator drains, then wait for its
// records).
template <typename Real, class Net>
int launch_rollout_impl(const RoundArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto k = kernel_of<Real, Net>(a.grid_mode);
  const size_t smem = static_cast<size_t>(a.field_smem_bytes);
  if (smem > 32 * 1024) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  }
  bool after_generate = false;
  if constexpr (Net::kP > 0) after_generate = refill_schedule<Net>();
  cudaError_t e = launch_dependent(k, a.grid, a.block, smem, st, after_generate, a);
  if (e == cudaSuccess && a.keys_only) {
    // about four blocks per SM over all restarts
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>((a.count + 2047) / 2048,
                                                              148 * 4 / a.restart_count));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(per), static_cast<unsigned>(a.restart_count));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, reduce_keys_kernel, a);
  }
  return static_cast<int>(e);
}

// Near-tie window of a finished round (a dependent launch after the rollout).
inline int launch_select_impl(const RoundArgs& a, void* stream) {
  const int64_t total = a.count * a.restart_count;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  return static_cast<int>(
      launch_dependent(select_kernel, blocks, 256, 0, static_cast<cudaStream_t>(stream), true, a));
}

// FP64 re-evaluation of the selected window.
template <class Net64>
int launch_refine_impl(const RoundArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a.grid_mode == 2) {
    refine_kernel<Net64, 2><<<a.refine_grid, 128, 0, st>>>(a);
  } else if (a.grid_mode == 1) {
    refine_kernel<Net64, 1><<<a.refine_grid, 128, 0, st>>>(a);
  } else {
    refine_kernel<Net64, 0><<<a.refine_grid, 128, 0, st>>>(a);
  }
  return static_cast<int>(cudaGetLastError());
}

template <typename Real, class Net>
int shape_impl(int device, int field_bytes, int grid, LaunchShape* out) {
  auto k = kernel_of<Real, Net>(grid);
  const bool refill = refill_schedule<Net>();
  const int smem_bytes = field_bytes;
  out->queue_bytes = 0;
  out->theta_elem = refill ? rec_width<Real>(Net::kP) : 0;  // Reals per candidate record
  int sms = 0, blocks = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return static_cast<int>(e);
  if (smem_bytes > 32 * 1024) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kBlock, smem_bytes);
  if (e != cudaSuccess) return static_cast<int>(e);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  out->block = kBlock;
  out->grid = sms * (blocks > 0 ? blocks : 1);
  out->smem_limit = smem_optin;
  out->refill = refill ? 1 : 0;
  return 0;
}

}  // namespace ppdev
