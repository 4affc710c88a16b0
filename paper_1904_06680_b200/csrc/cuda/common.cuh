// common.cuh -- constants, the keyed SplitMix64 stream (src/rng.cpp), FP32/FP64 math
// helpers of the rollout (accurate sincos/tan/wrap kernels), round constants.
// Part of the sampler kernels (rollout.cuh).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

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
#ifndef PARAPLAN_ACCURATE_TANH
#define PARAPLAN_ACCURATE_TANH 0
#endif
#ifndef PARAPLAN_BRANCHLESS_SCAN
#define PARAPLAN_BRANCHLESS_SCAN 1
#endif
#ifndef PARAPLAN_FAST_SQRT
#define PARAPLAN_FAST_SQRT 1
#endif
#ifndef PARAPLAN_GEN_MINB
// theta generator of the small FP32 net ([5,2,2]): resident CTAs of 256 the
// register cap must allow (6: 40 registers, no spills; measured 2% faster
// than 4 CTAs at C2 once the Box-Muller runs in MUFU); other nets: 1
#define PARAPLAN_GEN_MINB 6
#endif
#ifndef PARAPLAN_GEN_MINB_MID
#define PARAPLAN_GEN_MINB_MID 2  // theta generator of FP32 [5,10,2] (rollout.cuh gen_min_blocks)
#endif
#ifndef PARAPLAN_REFILL_MINB_MID
// FP32 [5,10,2] rollout CTAs/SM (4: 128 registers, 8 B spill; its C2 round
// 0.452 ms at 3 CTAs / 142 registers, 0.433 at 4, 0.52 at 5 with 168 B spills)
#define PARAPLAN_REFILL_MINB_MID 4
#endif
#ifndef PARAPLAN_REFILL_MINB_BIG
// FP32 [5,10,10,2] rollout CTAs/SM (2: 255 registers; 3 spills 344 B and its
// C2 round goes 1.06 -> 1.47 ms)
#define PARAPLAN_REFILL_MINB_BIG 2
#endif
#ifndef PARAPLAN_GEN_MID_MAXP
#define PARAPLAN_GEN_MID_MAXP 96
#endif
#ifndef PARAPLAN_REFILL64_MINB
#define PARAPLAN_REFILL64_MINB 4  // FP64 [5,2,2]/[5,10,2]: <= 128 registers
#endif
// L2 residency of the theta records between the generator and the rollout
// (PARAPLAN_REC_L2=0: default caching): the generator stores them with an
// evict_last policy, the rollout's single read demotes them (evict_first).
#ifndef PARAPLAN_REC_L2
#define PARAPLAN_REC_L2 1
#endif
__device__ __forceinline__ unsigned long long l2_keep_policy() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_drop_policy() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_rec(float4* p, const float4& v, unsigned long long pol) {
#if PARAPLAN_REC_L2
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_rec(double2* p, const double2& v, unsigned long long pol) {
#if PARAPLAN_REC_L2
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
               :: "l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ float4 ld_rec(const float4* p, unsigned long long pol) {
#if PARAPLAN_REC_L2
  float4 v;
  asm("ld.global.L1::evict_first.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
#else
  return __ldcg(p);
#endif
}
__device__ __forceinline__ double2 ld_rec(const double2* p, unsigned long long pol) {
#if PARAPLAN_REC_L2
  double2 v;
  asm("ld.global.L1::evict_first.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
#else
  return __ldcg(p);
#endif
}
#ifndef PARAPLAN_FAST_BOXMULLER
#define PARAPLAN_FAST_BOXMULLER 1  // FP32 generator: MUFU log2 / sqrt in Box-Muller
#endif
#ifndef PARAPLAN_SELECT_BPS
#define PARAPLAN_SELECT_BPS 16  // window select: blocks per SM
#endif
#ifndef PARAPLAN_FAST_FP64
#define PARAPLAN_FAST_FP64 1  // FP64 rollout: branch-free tanh, polynomial tan (|x| <= pi/4)
#endif
#ifndef PARAPLAN_FFMA2
// packed FP32x2 FMAs in the point scan (sm_100 FFMA2): the kind-3 scan body
// drops from 39 to 33 instructions per 4 points, but the C2 rollout measured
// 0.6% slower and C4/C5 unchanged (A/B on B200), so it is off by default
#define PARAPLAN_FFMA2 0
#endif
#ifndef PARAPLAN_REFILL_MINB_2D
// 2-D grid kinds (C4, C5 dense: latency-bound chains of cell / chunk / point
// loads): 8 CTAs/SM at 64 registers despite 180-280 B of spills beat 6 at 80
// (measured on B200: C4 -6.5%, C5 100k -6..7%, C5 10k H=100 -5%, N=1k equal;
// 10 CTAs helped 100k further but cost N=1k 4%)
#define PARAPLAN_REFILL_MINB_2D 8
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
  // tanh(x) = 1 - 2 / (1 + 2^(2x log2 e)): one ex2, one rcp, three FP32 ops
  // (absolute error below ~4e-7 over the whole range, saturating to +-1;
  // libm's tanhf spends ~16 instructions for relative accuracy near 0 that
  // the policy outputs do not need). PARAPLAN_ACCURATE_TANH=1 restores it.
  static __device__ __forceinline__ float th(float x) {
#if PARAPLAN_ACCURATE_TANH
    return tanhf(x);
#else
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
    return fmaf(-2.0f, r, 1.0f);
#endif
  }
  // th of x / (2 log2 e): the prescaled weights' argument (nets.cuh prescale)
  static __device__ __forceinline__ float th_pre(float x) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
    return fmaf(-2.0f, r, 1.0f);
  }
  static __device__ __forceinline__ float tn(float x) { return tanf(x); }
  // tan for |x| <= pi/4 (the steering range when delta_max <= pi/4)
  static __device__ __forceinline__ float tn_small(float x) {
#if PARAPLAN_FAST_SQRT
    float r;  // cos_poly >= 0.7 here: no denormal or zero input
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(cos_poly(x)));
    return sin_poly(x) * r;
#else
    return sin_poly(x) * __frcp_rn(cos_poly(x));
#endif
  }
  static __device__ __forceinline__ void sc(float x, float* s, float* c) {
    fast_sincosf(x, s, c);
  }
  static __device__ __forceinline__ float sq(float x) {
#if PARAPLAN_FAST_SQRT
    float r;  // path segments: ~1 ulp, no slow path for denormals
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return sqrtf(x);
#endif
  }
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
#if PARAPLAN_FAST_FP64
  // tanh(x) = sign(x) (1 - 2 / (exp(2|x|) + 1)): branch-free (libdevice's
  // tanh takes a polynomial path below |x| = 0.55 and an exp path above, and
  // a warp runs both), absolute error a few ulp of 1 (the policy's outputs
  // are clamped actions: absolute accuracy is what propagates). The FP64
  // rollout is certified against the reference's own arithmetic like the
  // FP32 one; its measured error stays ~1e-13.
  static __device__ __forceinline__ double th(double x) {
    const double e = exp(2.0 * fabs(x));
    return copysign(1.0 - 2.0 / (e + 1.0), x);
  }
  // tan on |x| <= pi/4 (the steering range when delta_max <= pi/4): sin / cos
  // of their minimax kernels (fdlibm __kernel_sin / __kernel_cos
  // coefficients), no range reduction
  static __device__ __forceinline__ double tn_small(double x) {
    const double z = x * x;
    const double sp = x + x * z * (-1.66666666666666324348e-01 +
        z * (8.33333333332248946124e-03 + z * (-1.98412698298579493134e-04 +
        z * (2.75573137070700676789e-06 + z * (-2.50507602534068634195e-08 +
        z * 1.58969099521155010221e-10)))));
    const double cp = 1.0 - 0.5 * z + z * z * (4.16666666666666019037e-02 +
        z * (-1.38888888888741095749e-03 + z * (2.48015872894767294178e-05 +
        z * (-2.75573143513906633035e-07 + z * (2.08757232129817482790e-09 +
        z * -1.13596475577881948265e-11)))));
    return sp / cp;
  }
#else
  static __device__ __forceinline__ double th(double x) { return tanh(x); }
  static __device__ __forceinline__ double tn_small(double x) { return tan(x); }
#endif
  static __device__ __forceinline__ double tn(double x) { return tan(x); }
  static __device__ __forceinline__ void sc(double x, double* s, double* c) { sincos(x, s, c); }
  static __device__ __forceinline__ double sq(double x) { return sqrt(x); }
  static __device__ __forceinline__ double ab(double x) { return fabs(x); }
  static __device__ __forceinline__ double wrap(double a) {
    const double r = remainder(a, kTwoPi);  // exact, identical to glibc
    return r <= -kPi ? r + kTwoPi : r;
  }
  // the correctly rounded a / d of the reference (src/planner.cpp:117-120,
  // 186-189) for a constant divisor d with inv = RN(1 / d) (the host's
  // 1.0 / d): Markstein's correction, q = RN(a inv), r = a - q d exactly by
  // FMA, RN(q + r inv) = RN(a / d) (no over/underflow in this range). Three
  // DFMA/DMUL instead of div.rn.f64's iteration and special-case checks; a
  // zero residual keeps q itself (the sign of a zero quotient)
  static __device__ __forceinline__ double ndiv(double a, double d, double inv) {
    const double q = a * inv;
    const double r = fma(-q, d, a);
    return r == 0.0 ? q : fma(r, inv, q);
  }
};

template <typename Real>
__device__ __forceinline__ Real clampr(Real v, Real lo, Real hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}
// FP32: two FMNMX (equal to std::clamp for every non-NaN v when lo <= hi;
// the rollout's inputs are finite)
template <>
__device__ __forceinline__ float clampr<float>(float v, float lo, float hi) {
  return fminf(fmaxf(v, lo), hi);
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

}  // namespace ppdev
