// rollout.cuh -- the fused per-control-step sampler kernel (sm_100a).
//
// One thread per candidate. Per candidate it
//   1. derives the keyed SplitMix64 stream in closed form and draws
//      theta = center + sigma * N(0,1) (src/rng.cpp:26-58,
//      src/planner.cpp:207-226) into registers,
//   2. rolls the kinematic bicycle over the horizon with the reference's
//      exact check order (src/planner.cpp:66-191): collision vs the obstacle
//      row h (field staged once per CTA in shared memory, read as a warp
//      broadcast), inclusive goal box in the goal frame, horizon stop, tanh
//      MLP -> map_controls -> explicit Euler,
//   3. scores the rollout (src/planner.cpp:27-44) and reduces to the
//      lexicographically best candidate, ties to the lowest index.
// CTAs are persistent and pull 1-restart tiles from an atomic ticket; the last
// CTA to finish reduces the tile winners per restart (the ordered merge of
// src/planner.cpp:310-321) and resets the tickets, so a round is ONE launch.
//
// Real = float is the throughput path (FMA contraction on); Real = double is
// the parity path (compiled with --fmad=false so every add/mul rounds like
// the reference's -ffp-contract=off build).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device_api.h"

namespace ppdev {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;

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

template <>
struct M<float> {
  static __device__ __forceinline__ float th(float x) { return tanhf(x); }
  static __device__ __forceinline__ float tn(float x) { return tanf(x); }
  static __device__ __forceinline__ void sc(float x, float* s, float* c) { sincosf(x, s, c); }
  static __device__ __forceinline__ float sq(float x) { return sqrtf(x); }
  static __device__ __forceinline__ float ab(float x) { return fabsf(x); }
  // wrap_angle (src/geometry.cpp:9-13): remainder by 2*pi (Cody-Waite in two
  // parts), lower boundary folded onto +pi.
  static __device__ __forceinline__ float wrap(float a) {
    const float n = rintf(a * 0.15915494309189535f);
    float r = fmaf(-n, 6.28318548202514648f, a);
    r = fmaf(-n, -1.7484555314695172e-07f, r);
    return r <= -3.14159274101257324f ? r + 6.28318548202514648f : r;
  }
  static __device__ __forceinline__ float ndiv(float a, double d, float inv) { return a * inv; }
};

template <>
struct M<double> {
  static __device__ __forceinline__ double th(double x) { return tanh(x); }
  static __device__ __forceinline__ double tn(double x) { return tan(x); }
  static __device__ __forceinline__ void sc(double x, double* s, double* c) { sincos(x, s, c); }
  static __device__ __forceinline__ double sq(double x) { return sqrt(x); }
  static __device__ __forceinline__ double ab(double x) { return fabs(x); }
  static __device__ __forceinline__ double wrap(double a) {
    const double r = remainder(a, kTwoPi);  // exact, identical to glibc
    return r <= -kPi ? r + kTwoPi : r;
  }
  static __device__ __forceinline__ double ndiv(double a, double d, double) { return a / d; }
};

template <typename Real>
__device__ __forceinline__ Real clampr(Real v, Real lo, Real hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// Kernel-entry copy of the round constants in the compute precision.
template <typename Real>
struct Consts {
  Real gx, gy, gphi, gv, gcos, gsin;
  Real v0, act0, pa0;
  Real inv_xi, inv_eta, inv_phi, inv_v;
  double d_xi, d_eta, d_phi, d_v;  // FP64 path divides (src/planner.cpp:117-120)
  Real eps_xi, eps_eta, eps_phi, eps_v;
  Real dmax, window, l_r, wb, Ts, umin, umax;
  Real fe, re, hw, r2;
  __device__ __forceinline__ void load(const RoundArgs& a) {
    gx = Real(a.gx); gy = Real(a.gy); gphi = Real(a.gphi); gv = Real(a.gv);
    gcos = Real(a.gcos); gsin = Real(a.gsin);
    v0 = Real(a.v0); act0 = Real(a.act0); pa0 = Real(a.pa0);
    inv_xi = Real(1.0 / a.d_xi); inv_eta = Real(1.0 / a.d_eta);
    inv_phi = Real(1.0 / a.d_phi); inv_v = Real(1.0 / a.d_v);
    d_xi = a.d_xi; d_eta = a.d_eta; d_phi = a.d_phi; d_v = a.d_v;
    eps_xi = Real(a.eps_xi); eps_eta = Real(a.eps_eta);
    eps_phi = Real(a.eps_phi); eps_v = Real(a.eps_v);
    dmax = Real(a.delta_max); window = Real(a.window); l_r = Real(a.l_r);
    wb = Real(a.wheelbase); Ts = Real(a.T_s); umin = Real(a.u_v_min); umax = Real(a.u_v_max);
    fe = Real(a.fe); re = Real(a.re); hw = Real(a.hw); r2 = Real(a.r2);
  }
};

// ----------------------------------------------------------- networks ----
// [5, H1, 2], theta in registers; layout per layer W (out x in, row-major)
// then b (include/paraplan/policy.hpp:50-53, src/policy.cpp:53-80).
template <typename Real, int H1>
struct NetReg {
  static constexpr int P = 6 * H1 + (H1 + 1) * 2;
  static constexpr int kP = P;  // compile-time parameter count
  Real w[P];
  __device__ __forceinline__ void set(int i, Real v) { w[i] = v; }
  __device__ __forceinline__ void eval(const Real s[5], Real& a0, Real& a1) const {
    Real hdn[H1];
#pragma unroll
    for (int o = 0; o < H1; ++o) {
      Real acc = w[5 * H1 + o];
#pragma unroll
      for (int i = 0; i < 5; ++i) acc += w[o * 5 + i] * s[i];
      hdn[o] = M<Real>::th(acc);
    }
    constexpr int off = 6 * H1;
    Real out[2];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      Real acc = w[off + 2 * H1 + o];
#pragma unroll
      for (int i = 0; i < H1; ++i) acc += w[off + o * H1 + i] * hdn[i];
      out[o] = M<Real>::th(acc);
    }
    a0 = out[0];
    a1 = out[1];
  }
};

// Any architecture (sizes <= 256): theta in a per-thread column of a global
// scratch buffer (coalesced across the warp), activations in local memory.
template <typename Real>
struct NetGlobal {
  static constexpr int kP = 0;  // runtime parameter count
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
// theta for candidate c of restart r (src/planner.cpp:207-226): c == 0 is the
// centre; otherwise sigma first, then Box-Muller pairs (cos value first).
// The stream is always evaluated in FP64, then rounded to Real.
template <typename Real, class Net>
__device__ __forceinline__ void draw_theta(Net& net, const RoundArgs& a, uint64_t prefix,
                                           int64_t c) {
  // KP > 0: fully unrolled so theta stays in registers.
  constexpr int KP = Net::kP;
  const int P = KP > 0 ? KP : a.n_params;
  const double* center = a.center;
  if (c == 0) {
#pragma unroll
    for (int i = 0; i < P; ++i) net.set(i, Real(__ldg(center + i)));
    return;
  }
  Stream g{fold(prefix, static_cast<uint64_t>(c))};
  const double sigma = pow(10.0, a.sig_lo + unit53(g.next()) * a.sig_span);
#pragma unroll
  for (int i = 0; i < P; i += 2) {
    const double u1 = 1.0 - unit53(g.next());
    const double u2 = unit53(g.next());
    const double r = sqrt(-2.0 * log(u1));
    const double t = kTwoPi * u2;
    double sn, cs;
    sincos(t, &sn, &cs);
    net.set(i, Real(__ldg(center + i) + sigma * (r * cs)));
    if (i + 1 < P) net.set(i + 1, Real(__ldg(center + i + 1) + sigma * (r * sn)));
  }
}

template <typename Real, class Net>
__device__ __forceinline__ void load_theta(Net& net, const double* src, int Pdyn) {
  constexpr int KP = Net::kP;
  const int P = KP > 0 ? KP : Pdyn;
#pragma unroll
  for (int i = 0; i < P; ++i) net.set(i, Real(src[i]));
}

template <typename Real>
struct Outcome {
  int cls;  // 2 reached, 1 free, 0 collided
  int t_goal;
  int steps;
  Real path, terminal, f0, f1;
};

// src/planner.cpp:66-191 (simulate<false>) in Real arithmetic.
template <typename Real, class Net>
__device__ __forceinline__ Outcome<Real> simulate(const Net& net, const Consts<Real>& K,
                                                  const typename Vec2T<Real>::type* field,
                                                  int N, int H) {
  using R2 = typename Vec2T<Real>::type;
  Real x = Real(0), y = Real(0), phi = Real(0), v = K.v0;
  Real act = K.act0, pa0 = K.pa0;
  Real path = Real(0);
  int status = 1;
  int t_goal = -1;
  int h = 0;

  Real ephi = M<Real>::wrap(K.gphi - phi);
  Real s[5] = {M<Real>::ndiv(K.gx - x, K.d_xi, K.inv_xi), M<Real>::ndiv(K.gy - y, K.d_eta, K.inv_eta),
               M<Real>::ndiv(ephi, K.d_phi, K.inv_phi), M<Real>::ndiv(K.gv - v, K.d_v, K.inv_v), pa0};
  Real f0, f1;
  net.eval(s, f0, f1);  // first action exists even if the rollout ends at h = 0

  for (;; ++h) {
    Real sphi, cphi;
    M<Real>::sc(phi, &sphi, &cphi);
    if (N > 0) {
      // src/geometry.cpp:63-76 against row h; strict half-planes
      const R2* row = field + static_cast<size_t>(h) * N;
      bool hit = false;
      for (int j = 0; j < N; ++j) {
        const R2 m = row[j];
        const Real dx = m.x - x, dy = m.y - y;
        if (dx * dx + dy * dy < K.r2) {
          const Real bx = cphi * dx + sphi * dy;
          const Real by = -sphi * dx + cphi * dy;
          hit |= (bx < K.fe) & (-bx < K.re) & (by < K.hw) & (-by < K.hw);
        }
      }
      if (hit) {
        status = 0;
        break;
      }
    }
    ephi = M<Real>::wrap(K.gphi - phi);
    {
      const Real gdx = K.gx - x, gdy = K.gy - y;
      if (M<Real>::ab(K.gcos * gdx + K.gsin * gdy) <= K.eps_xi &&
          M<Real>::ab(-K.gsin * gdx + K.gcos * gdy) <= K.eps_eta &&
          M<Real>::ab(ephi) <= K.eps_phi && M<Real>::ab(K.gv - v) <= K.eps_v) {
        status = 2;
        t_goal = h;
        break;
      }
    }
    if (h == H) break;

    Real a0, a1;
    if (h == 0) {
      a0 = f0;
      a1 = f1;
    } else {
      s[0] = M<Real>::ndiv(K.gx - x, K.d_xi, K.inv_xi);
      s[1] = M<Real>::ndiv(K.gy - y, K.d_eta, K.inv_eta);
      s[2] = M<Real>::ndiv(ephi, K.d_phi, K.inv_phi);
      s[3] = M<Real>::ndiv(K.gv - v, K.d_v, K.inv_v);
      s[4] = pa0;
      net.eval(s, a0, a1);
    }
    // map_controls (src/dynamics.cpp:30-43)
    const Real c0 = clampr(a0, Real(-1), Real(1));
    const Real c1 = clampr(a1, Real(-1), Real(1));
    Real delta = clampr(K.dmax * c0, act - K.window, act + K.window);
    delta = clampr(delta, -K.dmax, K.dmax);
    const Real w = Real(0.5) * (c1 + Real(1));
    const Real u_v = (Real(1) - w) * K.umin + w * K.umax;
    // explicit Euler (src/dynamics.cpp:45-62)
    const Real tan_d = M<Real>::tn(delta);
    const Real tb = K.l_r * tan_d / K.wb;
    const Real tv = K.Ts * v;
    const Real nx = x + tv * (cphi - tb * sphi);
    const Real ny = y + tv * (sphi + tb * cphi);
    const Real nphi = phi + tv * tan_d / K.wb;
    const Real nv = v + K.Ts * u_v;
    const Real dx = nx - x, dy = ny - y;
    path += M<Real>::sq(dx * dx + dy * dy);
    x = nx;
    y = ny;
    phi = nphi;
    v = nv;
    act = delta;
    pa0 = a0;
  }
  if (status == 0) ephi = M<Real>::wrap(K.gphi - phi);
  Outcome<Real> o;
  o.cls = status;
  o.t_goal = t_goal;
  o.steps = h;  // states 0..h were checked; h dynamics steps simulated
  o.path = path;
  o.terminal = M<Real>::ndiv(M<Real>::ab(K.gx - x), K.d_xi, K.inv_xi) +
               M<Real>::ndiv(M<Real>::ab(K.gy - y), K.d_eta, K.inv_eta) +
               M<Real>::ndiv(M<Real>::ab(ephi), K.d_phi, K.inv_phi) +
               M<Real>::ndiv(M<Real>::ab(K.gv - v), K.d_v, K.inv_v);
  o.f0 = f0;
  o.f1 = f1;
  return o;
}


// ---------------------------------------------------------- reduction ----
// Lexicographic (cls, k1, k2) descending, index ascending: a total order, so
// any reduction tree gives the reference's "strict better, lowest index wins"
// result (src/planner.cpp:40-44, 295, 316).
template <typename K>
struct Key {
  int cls;
  int idx;
  K k1, k2;
};

template <typename K>
__device__ __forceinline__ bool prefer(const Key<K>& a, const Key<K>& b) {
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  if (a.k2 != b.k2) return a.k2 > b.k2;
  return static_cast<unsigned>(a.idx) < static_cast<unsigned>(b.idx);
}

template <typename K>
__device__ __forceinline__ Key<K> shfl_key(const Key<K>& k, int src) {
  Key<K> o;
  o.cls = __shfl_down_sync(0xffffffffu, k.cls, src);
  o.idx = __shfl_down_sync(0xffffffffu, k.idx, src);
  o.k1 = __shfl_down_sync(0xffffffffu, k.k1, src);
  o.k2 = __shfl_down_sync(0xffffffffu, k.k2, src);
  return o;
}

// Block argmin; result valid in thread 0. `scratch` holds >= 32 keys.
template <typename K>
__device__ __forceinline__ Key<K> block_best(Key<K> k, Key<K>* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Key<K> o = shfl_key(k, off);
    if (prefer(o, k)) k = o;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = k;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    k = lane < nw ? scratch[lane] : Key<K>{-1, -1, K(0), K(0)};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const Key<K> o = shfl_key(k, off);
      if (prefer(o, k)) k = o;
    }
  }
  __syncthreads();
  return k;
}

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v,
                                                        unsigned long long* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? scratch[lane] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  }
  __syncthreads();
  return v;
}

// ------------------------------------------------------------- kernel ----
template <typename Real, class Net>
struct NetFactory;

template <typename Real, int H1>
struct NetFactory<Real, NetReg<Real, H1>> {
  static __device__ __forceinline__ NetReg<Real, H1> make(const RoundArgs&) { return {}; }
  static constexpr bool kStaticP = true;
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
  static constexpr bool kStaticP = false;
};

template <typename Real, class Net>
__global__ void __launch_bounds__(128) round_kernel(const RoundArgs a) {
  using R2 = typename Vec2T<Real>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Key<double> red[32];
  __shared__ unsigned long long red_sum[32];
  __shared__ int s_tile;

  Consts<Real> K;
  K.load(a);
  const int N = a.n_points;
  const int H = a.H;
  const int P = a.n_params;

  // Stage the obstacle field once per persistent CTA (read by every warp as
  // a broadcast); large fields stay in L2 and are read through the RO path.
  const R2* field = static_cast<const R2*>(a.field);
  if (a.field_smem_bytes > 0) {
    R2* dst = reinterpret_cast<R2*>(smem_raw);
    const int total = (H + 1) * N;
    for (int i = threadIdx.x; i < total; i += blockDim.x) dst[i] = field[i];
    field = dst;
    __syncthreads();
  }

  Net net = NetFactory<Real, Net>::make(a);
  unsigned long long my_steps = 0, my_states = 0;

  for (;;) {
    if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(&a.counters[0], 1u));
    __syncthreads();
    const int tile = s_tile;
    __syncthreads();
    if (tile >= a.n_tiles) break;
    const int r = tile / a.tiles_per_restart;
    const int64_t local = static_cast<int64_t>(tile - r * a.tiles_per_restart) * blockDim.x +
                          threadIdx.x;
    Key<double> key{-1, -1, 0.0, 0.0};
    if (local < a.count) {
      const int64_t c = a.cand_begin + local;
      if (a.injected != nullptr) {
        load_theta<Real>(net, a.injected + local * P, P);
      } else {
        draw_theta<Real>(net, a, __ldg(a.key_prefix + r), c);
      }
      const Outcome<Real> o = simulate<Real>(net, K, field, N, H);
      key.cls = o.cls;
      key.idx = static_cast<int>(c);
      if (o.cls == 2) {  // src/planner.cpp:27-38
        key.k1 = -static_cast<double>(o.t_goal);
        key.k2 = -static_cast<double>(o.path);
      } else {
        key.k1 = -static_cast<double>(o.terminal);
        key.k2 = 0.0;
      }
      my_steps += static_cast<unsigned long long>(o.steps);
      my_states += static_cast<unsigned long long>(o.steps + 1);
      if (a.per_sample != nullptr) {
        SampleOut& so = a.per_sample[static_cast<int64_t>(r) * a.count + local];
        so.reached = o.cls == 2;
        so.t_goal = o.t_goal;
        so.collided = o.cls == 0;
        so.steps = o.steps;
        so.path_length = static_cast<double>(o.path);
        so.terminal_cost = static_cast<double>(o.terminal);
        so.first_a0 = static_cast<double>(o.f0);
        so.first_a1 = static_cast<double>(o.f1);
      }
    }
    const Key<double> best = block_best(key, red);
    if (threadIdx.x == 0) a.tile_recs[tile] = Rec{best.cls, best.idx, best.k1, best.k2};
  }

  // Work accounting, one atomic per CTA.
  const unsigned long long steps = block_sum(my_steps, red_sum);
  const unsigned long long states = block_sum(my_states, red_sum);
  if (threadIdx.x == 0) {
    atomicAdd(&a.exec[0], steps);
    atomicAdd(&a.exec[1], states);
  }

  // Last CTA reduces the tile winners of every restart (ordered merge).
  __threadfence();
  if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(&a.counters[1], 1u));
  __syncthreads();
  if (s_tile != static_cast<int>(gridDim.x) - 1) return;
  __threadfence();
  for (int r = 0; r < a.restart_count; ++r) {
    Key<double> k{-1, -1, 0.0, 0.0};
    for (int t = threadIdx.x; t < a.tiles_per_restart; t += blockDim.x) {
      // written by other CTAs: read through L2 (ld.global.cg), never L1
      const Rec* src = a.tile_recs + r * a.tiles_per_restart + t;
      const Key<double> o{__ldcg(&src->cls), __ldcg(&src->cand), __ldcg(&src->k1),
                          __ldcg(&src->k2)};
      if (o.cls >= 0 && (k.cls < 0 || prefer(o, k))) k = o;
    }
    const Key<double> best = block_best(k, red);
    if (threadIdx.x == 0) a.out[r] = Rec{best.cls, best.idx, best.k1, best.k2};
  }
  if (threadIdx.x == 0) {
    // publish the work counters and re-arm everything for the next round
    a.exec[2] = atomicExch(&a.exec[0], 0ull);
    a.exec[3] = atomicExch(&a.exec[1], 0ull);
    a.counters[0] = 0;
    a.counters[1] = 0;
  }
}

// ------------------------------------------------------------ launch ----
template <typename Real, class Net>
int launch_impl(const RoundArgs& a, void* stream) {
  const size_t smem = static_cast<size_t>(a.field_smem_bytes);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(round_kernel<Real, Net>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  }
  round_kernel<Real, Net><<<a.grid, a.block, smem, static_cast<cudaStream_t>(stream)>>>(a);
  return static_cast<int>(cudaGetLastError());
}

template <typename Real, class Net>
int shape_impl(int device, int smem_bytes, LaunchShape* out) {
  int sms = 0, blocks = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return static_cast<int>(e);
  if (smem_bytes > 48 * 1024) {
    e = cudaFuncSetAttribute(round_kernel<Real, Net>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, round_kernel<Real, Net>, 128,
                                                    smem_bytes);
  if (e != cudaSuccess) return static_cast<int>(e);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  out->block = 128;
  out->grid = sms * (blocks > 0 ? blocks : 1);
  out->smem_limit = smem_optin;
  return 0;
}

}  // namespace ppdev
