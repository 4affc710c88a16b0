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
  // state 0 with the first action (first0, first1) still to apply
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

// The verdicts at the lane's state h (src/planner.cpp:137-152): collision
// with field row h, the goal box, the horizon. Returns -1 while running, else
// the class (0 collided, 1 horizon, 2 reached at state h); records the
// earliest flagged state. Branch-free: every lane computes every check.
template <typename Real, int kGrid>
__device__ __forceinline__ int check_state(Lane<Real>& L, const Consts<Real>& K,
                                           const Field<Real>& f, int H, bool live, Real sphi,
                                           Real cphi) {
  bool hit = false;
  // the flag band: the base margin plus the drift the state may have
  // accumulated over the path so far, which grows with the state index like
  // the measured relative path error (rho2_fp32's envelope)
  Real band = K.dmarg;
  if (K.dmarg_rel != Real(0)) {
    const Real q = static_cast<Real>(L.h) * Real(1.0 / 150.0);
    band += L.path * fmax(K.dmarg_floor, K.dmarg_rel * fmin(q * q, Real(1)));
  }
  bool narrow = false;
  if (K.any_pts) {  // f.Ns + f.Nd > 0
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
  return hit ? 0 : (reached ? 2 : (L.h == H ? 1 : -1));
}

// The transition from the lane's state h under action (a0, a1):
// map_controls (src/dynamics.cpp:30-43) and the explicit Euler step
// (src/dynamics.cpp:45-62), with the path segment (src/planner.cpp:177-179).
template <typename Real>
struct Next {
  Real x, y, phi, v, act, seg;
};
template <typename Real>
__device__ __forceinline__ Next<Real> transition(const Lane<Real>& L, const Consts<Real>& K,
                                                 Real a0, Real a1, Real sphi, Real cphi) {
  const Real c0 = clampr(a0, Real(-1), Real(1));
  const Real c1 = clampr(a1, Real(-1), Real(1));
  Real delta = clampr(K.dmax * c0, L.act - K.window, L.act + K.window);
  delta = clampr(delta, -K.dmax, K.dmax);
  const Real tan_d = K.tan_small ? M<Real>::tn_small(delta) : M<Real>::tn(delta);
  const Real tb = M<Real>::ndiv(K.l_r * tan_d, K.wb_d, K.inv_wb);
  const Real tv = K.Ts * L.v;
  const Real ix = tv * (cphi - tb * sphi);
  const Real iy = tv * (sphi + tb * cphi);
  Next<Real> n;
  n.x = L.x + ix;
  n.y = L.y + iy;
  n.phi = L.phi + M<Real>::ndiv(tv * tan_d, K.wb_d, K.inv_wb);
  n.act = delta;
  if constexpr (sizeof(Real) == sizeof(double)) {
    // u_v = lerp(umin, umax, (c1 + 1) / 2) (src/dynamics.cpp:40-42)
    const Real w = Real(0.5) * (c1 + Real(1));
    const Real u_v = (Real(1) - w) * K.umin + w * K.umax;
    n.v = L.v + K.Ts * u_v;
    // the reference's difference of the rounded positions
    const Real dx = n.x - L.x, dy = n.y - L.y;
    n.seg = M<Real>::sq(dx * dx + dy * dy);
  } else {
    // FP32 folds the lerp with T_s into one FMA; the path takes the
    // increment itself, since n.x - x cancels ~|x| / |dx| float ulps (1e-6
    // relative per segment at 30 m), which the FP64 difference does not
    n.v = fmaf(c1, K.ts_uhalf, L.v + K.ts_umid);
    n.seg = M<Real>::sq(ix * ix + iy * iy);
  }
  return n;
}

// Apply a transition: the lane moves to state h + 1 (a0: the action's first
// component, the next state's feature).
template <typename Real>
__device__ __forceinline__ void commit(Lane<Real>& L, const Next<Real>& n, Real a0) {
  L.path += n.seg;
  L.x = n.x;
  L.y = n.y;
  L.phi = n.phi;
  L.v = n.v;
  L.act = n.act;
  L.pa0 = a0;
  ++L.h;
}

// State 1 of every candidate: state 0 under its first action (f0, f1), as
// advance computes it. The refill schedule's generator applies it, so the
// rollout starts at state 1 (the checks of state 0, the same for every
// candidate, run once per rollout thread).
template <typename Real>
__device__ __forceinline__ void first_step(Lane<Real>& L, const Consts<Real>& K) {
  const Next<Real> n = transition(L, K, L.f0, L.f1, Real(0), Real(1));
  commit(L, n, L.f0);
}

// Whether a refill-schedule net's weights are prescaled (nets.cuh prescale):
// FP32 register nets with the fast tanh.
template <typename Real, class Net>
constexpr bool prescaled(bool refill) {
  return refill && sizeof(Real) == sizeof(float) && Net::kP > 0 && !PARAPLAN_ACCURATE_TANH;
}

// One state of the rollout loop (src/planner.cpp:137-183): the checks of
// state h and, independent of them, the MLP and transition to state h + 1,
// committed only by lanes still running (live, and no verdict at h).
// Returns -1 while running, else the class at state h. Warp-synchronous and
// branch-free: the checks and the next state are computed for every lane, so
// the warp never splits into per-outcome paths; a lane with live == false
// (idle, or parked with a finished rollout until the warp's next flush) scans
// no points and keeps its state.
// kFromZero: lanes may be at state 0 (the lockstep schedules), whose action
// is the precomputed first one; otherwise the lanes come from the refill
// schedule's records (state >= 1, prescaled weights where prescaled()).
template <typename Real, int kGrid, class Net, bool kFromZero = true>
__device__ __forceinline__ int advance(Lane<Real>& L, const Net& net, const Consts<Real>& K,
                                       const Field<Real>& f, int H, bool live = true) {
  Real sphi, cphi;
  M<Real>::sc(L.phi, &sphi, &cphi);
  L.ephi = M<Real>::wrap(K.gphi - L.phi);
  const int cls = check_state<Real, kGrid>(L, K, f, H, live, sphi, cphi);
  Real s[5];
  constexpr bool kPre = prescaled<Real, Net>(!kFromZero);
  if constexpr (kPre) {  // the normalisation lives in the weights
    s[0] = K.gx - L.x;
    s[1] = K.gy - L.y;
    s[2] = L.ephi;
    s[3] = K.gv - L.v;
  } else {
    s[0] = M<Real>::ndiv(K.gx - L.x, K.d_xi, K.inv_xi);
    s[1] = M<Real>::ndiv(K.gy - L.y, K.d_eta, K.inv_eta);
    s[2] = M<Real>::ndiv(L.ephi, K.d_phi, K.inv_phi);
    s[3] = M<Real>::ndiv(K.gv - L.v, K.d_v, K.inv_v);
  }
  s[4] = L.pa0;
  Real a0, a1;
  net.template eval<kPre>(s, a0, a1);
  if (kFromZero && L.h == 0) {  // the first action was computed before the loop
    a0 = L.f0;
    a1 = L.f1;
  }
  const Next<Real> n = transition(L, K, a0, a1, sphi, cphi);
  if (live && cls < 0) commit(L, n, a0);  // a parked or idle lane keeps its state
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
