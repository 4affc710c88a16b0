// nets.cuh -- the tanh MLP policies (src/policy.cpp:53-80): theta in registers
// ([5,H1,2], [5,A,B,2]) or in a per-lane global column (any architecture).
// Part of the sampler kernels (rollout.cuh).
#pragma once

#include "common.cuh"

namespace ppdev {

// ----------------------------------------------------------- networks ----
// [5, H1, 2] forward pass over any weight accessor w(i); layout per layer W
// (out x in, row-major) then b (include/paraplan/policy.hpp:50-53,
// src/policy.cpp:53-80): acc = b, acc += W[o][i] * x[i] ascending, tanh.
// kPre: the weights were prescaled (prescale below): raw features in, and
// each tanh takes its argument already multiplied by 2 log2(e).
template <typename Real, bool kPre>
__device__ __forceinline__ Real act(Real x) {
  if constexpr (kPre) {
    return M<Real>::th_pre(x);
  } else {
    return M<Real>::th(x);
  }
}

template <typename Real, int H1, bool kPre, class W>
__device__ __forceinline__ void mlp_5h2(W&& w, const Real s[5], Real& a0, Real& a1) {
  Real hdn[H1];
#pragma unroll
  for (int o = 0; o < H1; ++o) {
    Real acc = w(5 * H1 + o);
#pragma unroll
    for (int i = 0; i < 5; ++i) acc += w(o * 5 + i) * s[i];
    hdn[o] = act<Real, kPre>(acc);
  }
  constexpr int off = 6 * H1;
  Real out[2];
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    Real acc = w(off + 2 * H1 + o);
#pragma unroll
    for (int i = 0; i < H1; ++i) acc += w(off + o * H1 + i) * hdn[i];
    out[o] = act<Real, kPre>(acc);
  }
  a0 = out[0];
  a1 = out[1];
}

// FP32 refill schedule: the generator folds the feature normalisation
// (1 / d_xi, 1 / d_eta, 1 / d_phi, 1 / d_v; src/planner.cpp:117-120) into the
// first layer's weights and the fast tanh's 2 log2(e) into every layer, so a
// rollout step skips 4 + (hidden + 2) multiplies. Layers of `sizes` (W out x
// in row-major, then b), in place.
template <class Net>
__device__ __forceinline__ void prescale(float* w, const float in_scale[5]) {
  constexpr float k = 2.8853900817779268f;  // 2 log2(e)
  int off = 0;
#pragma unroll
  for (int l = 0; l < Net::kLayers; ++l) {
    const int nin = Net::size(l), nout = Net::size(l + 1);
#pragma unroll
    for (int o = 0; o < nout; ++o) {
#pragma unroll
      for (int i = 0; i < nin; ++i) w[off + o * nin + i] *= l == 0 ? in_scale[i] : k;
    }
#pragma unroll
    for (int o = 0; o < nout; ++o) w[off + nout * nin + o] *= k;
    off += (nin + 1) * nout;
  }
}

// [5, H1, 2], theta in registers.
template <typename Real, int H1>
struct NetReg {
  static constexpr int P = 6 * H1 + (H1 + 1) * 2;
  static constexpr int kP = P;
  static constexpr int kH1 = H1;
  static constexpr int kLayers = 2;
  static constexpr int size(int l) { return l == 0 ? 5 : (l == 1 ? H1 : 2); }
  Real w[P];
  __device__ __forceinline__ void set(int i, Real v) { w[i] = v; }
  template <bool kPre = false>
  __device__ __forceinline__ void eval(const Real s[5], Real& a0, Real& a1) const {
    mlp_5h2<Real, H1, kPre>([&](int i) { return w[i]; }, s, a0, a1);
  }
};

// [5, A, B, 2], theta in registers (FP32 [5,10,10,2]: 192 parameters, two
// CTAs of 128 threads per SM at <= 255 registers).
template <typename Real, int A, int B>
struct NetReg3 {
  static constexpr int P = 6 * A + (A + 1) * B + (B + 1) * 2;
  static constexpr int kP = P;
  static constexpr int kLayers = 3;
  static constexpr int size(int l) { return l == 0 ? 5 : (l == 1 ? A : (l == 2 ? B : 2)); }
  Real w[P];
  __device__ __forceinline__ void set(int i, Real v) { w[i] = v; }
  template <bool kPre = false>
  __device__ __forceinline__ void eval(const Real s[5], Real& a0, Real& a1) const {
    Real h1[A], h2[B];
#pragma unroll
    for (int o = 0; o < A; ++o) {
      Real acc = w[5 * A + o];
#pragma unroll
      for (int i = 0; i < 5; ++i) acc += w[o * 5 + i] * s[i];
      h1[o] = act<Real, kPre>(acc);
    }
    constexpr int off2 = 6 * A;
#pragma unroll
    for (int o = 0; o < B; ++o) {
      Real acc = w[off2 + A * B + o];
#pragma unroll
      for (int i = 0; i < A; ++i) acc += w[off2 + o * A + i] * h1[i];
      h2[o] = act<Real, kPre>(acc);
    }
    constexpr int off3 = off2 + (A + 1) * B;
    Real out[2];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      Real acc = w[off3 + 2 * B + o];
#pragma unroll
      for (int i = 0; i < B; ++i) acc += w[off3 + o * B + i] * h2[i];
      out[o] = act<Real, kPre>(acc);
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
  template <bool kPre = false>
  __device__ void eval(const Real s[5], Real& a0, Real& a1) const {
    static_assert(!kPre, "a global-column net is never prescaled");
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

}  // namespace ppdev
