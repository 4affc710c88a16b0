// sample.cuh -- candidate theta from the keyed stream (src/planner.cpp:207-226).
// Part of the sampler kernels (rollout.cuh).
#pragma once

#include "common.cuh"

namespace ppdev {

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
#if PARAPLAN_FAST_BOXMULLER
      // r = sqrt(-2 ln u1) with MUFU lg2 / rsqrt: ~1e-7 relative for r of
      // order 1; near u1 = 1 (r < 0.02, 1.5e-4 of the draws) the absolute
      // error of lg2.approx (2^-22.6) leaves r within ~2e-5 absolute. The
      // FP32 path only (certified; the host regenerates the winner in FP64).
      float l2, rr;
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(u1));
      const float t2 = -1.3862943611198906f * l2;  // -2 ln 2 log2(u1) = -2 ln(u1)
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rr) : "f"(fmaxf(t2, 0.0f)));
      const float r = rr;
#else
      const float r = sqrtf(-2.0f * logf(u1));
#endif
#if PARAPLAN_FAST_BOXMULLER
      // sincos(2 pi u2) = sincos(2 pi (u2 - rint(u2))) (the difference is
      // exact) with MUFU sin/cos on [-pi, pi]: absolute error ~2^-21.4
      float sn, cs;
      __sincosf(6.28318530717958648f * (u2 - rintf(u2)), &sn, &cs);
#else
      // sincos(2 pi u2): quarter-turn reduction t = 4 u2 - q is exact
      const float q = rintf(4.0f * u2);
      const float t = fmaf(4.0f, u2, -q) * 1.57079632679489662f;
      const float sp = sin_poly(t), cp = cos_poly(t);
      const int qi = static_cast<int>(q);
      float sn = (qi & 1) ? cp : sp;
      float cs = (qi & 1) ? sp : cp;
      sn = (qi & 2) ? -sn : sn;
      cs = ((qi + 1) & 2) ? -cs : cs;
#endif
      put(i, Real(__ldg(a.center_f + i) + sigma * (r * cs)));
      if (i + 1 < P) put(i + 1, Real(__ldg(a.center_f + i + 1) + sigma * (r * sn)));
    }
  } else {
    // FP64 path: libdevice's exp10 and sincospi (sin / cos of pi * 2 u2, the
    // product 2 u2 exact) instead of pow(10, .) and sincos(2 pi u2): theta
    // stays within a few ulps of the reference's draw (the host regenerates
    // the returned plan's theta in the reference's own arithmetic), and
    // sincospi needs no multi-part reduction of 2 pi u2
    const double sigma = exp10(a.sig_lo + unit53(g.next()) * a.sig_span);
#pragma unroll
    for (int i = 0; i < P; i += 2) {
      const double u1 = 1.0 - unit53(g.next());
      const double u2 = unit53(g.next());
      const double r = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      put(i, Real(__ldg(center + i) + sigma * (r * cs)));
      if (i + 1 < P) put(i + 1, Real(__ldg(center + i + 1) + sigma * (r * sn)));
    }
  }
}

}  // namespace ppdev
