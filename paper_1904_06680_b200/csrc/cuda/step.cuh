// step.cuh -- one rollout state of one candidate (src/planner.cpp:137-189).
// Part of the sampler kernels (rollout.cuh).
#pragma once

#include "field_query.cuh"
#include "nets.cuh"

namespace ppdev {

// One candidate's rollout state (src/planner.cpp:123-125, 130-132).
template <typename Real>
struct Lane {
  Real x, y, phi, v, act, pa0, path, f0, f1, ephi;
  int h;
  uint32_t mstep;  // earliest state of a verdict within the flag band (meta, kNoStep = none)
  Real mpath;      // FP64: the path up to that state (a flip there reaches with this path)
  __device__ __forceinline__ void start(const Consts<Real>& K, Real first0, Real first1) {
    x = y = phi = Real(0);
    v = K.v0;
    act = K.act0;
    pa0 = K.pa0;
    path = Real(0);
    f0 = first0;
    f1 = first1;
    h = 0;
    mstep = kNoStep;
    mpath = Real(0);
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
                                       const Field<Real>& f, int H, bool live = true) {
  Real sphi, cphi;
  M<Real>::sc(L.phi, &sphi, &cphi);
  L.ephi = M<Real>::wrap(K.gphi - L.phi);
  bool hit = false;
  // the flag band: the base margin plus the drift the state may have
  // accumulated over the path so far, which grows with the state index like
  // the measured relative path error (rho2_fp32's envelope)
  Real band = K.dmarg;
  if (K.dmarg_rel != Real(0)) {
    const Real f = static_cast<Real>(L.h) * Real(1.0 / 150.0);
    band += L.path * fmax(K.dmarg_floor, K.dmarg_rel * fmin(f * f, Real(1)));
  }
  bool narrow = false;
  if (f.Ns + f.Nd > 0) {
    // a lane may stop at a hit whose margin is too large to flip
    const Real cm = collide_margin<Real, kGrid>(f, K, L.h, L.x, L.y, cphi, sphi, band, live);
    hit = cm > Real(0);
    // a narrow hit might be free in exact arithmetic (a better outcome).
    // With several restarts a narrow miss is flagged too: it might be a hit
    // (a worse outcome), so it must not anchor a restart's window, which is
    // built around the restart's best unflagged candidate (flagged ones are
    // always in the window)
    narrow = (cm > (K.flag_miss ? -band : Real(0))) & (cm < band);
  }
  const Real gdx = K.gx - L.x, gdy = K.gy - L.y;
  // inclusive goal box: eps - |err| >= 0 <=> |err| <= eps, exactly
  const Real gm = fmin(fmin(K.eps_xi - M<Real>::ab(K.gcos * gdx + K.gsin * gdy),
                            K.eps_eta - M<Real>::ab(-K.gsin * gdx + K.gcos * gdy)),
                       fmin(K.eps_phi - M<Real>::ab(L.ephi), K.eps_v - M<Real>::ab(K.gv - L.v)));
  const bool reached = gm >= Real(0);
  // a narrow miss might reach in exact arithmetic (a better outcome)
  narrow |= !reached & (gm > -band);
  // state 0 is every candidate's (theta plays no part before the first
  // step): its verdicts cannot order candidates, and the host decides them
  // exactly (host_stops_at_state0), so they are never flags
  narrow &= L.h > 0;
  if constexpr (sizeof(Real) == sizeof(double)) {
    if (narrow && L.mstep == kNoStep) L.mpath = L.path;
  }
  L.mstep = narrow ? min(L.mstep, static_cast<uint32_t>(L.h)) : L.mstep;
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
  // u_v = lerp(umin, umax, (c1 + 1) / 2) (src/dynamics.cpp:40-42); FP32 folds
  // it with T_s into one FMA of the speed update below
  Real u_v = Real(0);
  if constexpr (sizeof(Real) == sizeof(double)) {
    const Real w = Real(0.5) * (c1 + Real(1));
    u_v = (Real(1) - w) * K.umin + w * K.umax;
  }
  // explicit Euler (src/dynamics.cpp:45-62)
  const Real tan_d = K.tan_small ? M<Real>::tn_small(delta) : M<Real>::tn(delta);
  const Real tb = M<Real>::ndiv(K.l_r * tan_d, K.wb_d, K.inv_wb);
  const Real tv = K.Ts * L.v;
  const Real ix = tv * (cphi - tb * sphi);
  const Real iy = tv * (sphi + tb * cphi);
  const Real nx = L.x + ix;
  const Real ny = L.y + iy;
  const Real nphi = L.phi + M<Real>::ndiv(tv * tan_d, K.wb_d, K.inv_wb);
  Real nv;
  if constexpr (sizeof(Real) == sizeof(double)) {
    nv = L.v + K.Ts * u_v;
  } else {
    nv = fmaf(c1, K.ts_uhalf, L.v + K.ts_umid);
  }
  // path segment (src/planner.cpp:177-179): FP64 takes the reference's
  // difference of the rounded positions; FP32 takes the increment itself,
  // since nx - x cancels ~|x| / |dx| float ulps (1e-6 relative per segment at
  // 30 m), which the FP64 difference does not
  Real seg;
  if constexpr (sizeof(Real) == sizeof(double)) {
    const Real dx = nx - L.x, dy = ny - L.y;
    seg = M<Real>::sq(dx * dx + dy * dy);
  } else {
    seg = M<Real>::sq(ix * ix + iy * iy);
  }
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

}  // namespace ppdev
