// binning_f64.cu -- device-side extrapolation and cell binning of the moving
// obstacle points (the host path is csrc/capi/field.cpp).
//
// Positions are the reference's extrapolate (src/geometry.cpp:53-57),
// x + h * step with h promoted to double, formed with explicit round-to-
// nearest multiply and add (and this TU is built with --fmad=false), so they
// equal the host's -ffp-contract=off positions bit for bit. The cell of a
// position is the host's formula. Within a cell the order follows the
// atomics; the collision verdict and the marginal flag do not depend on it
// (csrc/cuda/rollout.cuh: an OR over points, early exit only on robust hits).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_api.h"

namespace ppdev {
namespace {

__device__ __forceinline__ int clamp_cell(double t, int n) {
  return t <= 0.0 ? 0 : min(n - 1, static_cast<int>(t));
}

struct Mover {
  double x, y;
  int cell;
};

__device__ __forceinline__ Mover mover_at(const BinArgs& a, int r, int k) {
  const double* q = a.movers + 4 * static_cast<size_t>(k);
  const double rd = static_cast<double>(r);
  Mover m;
  m.x = __dadd_rn(q[0], __dmul_rn(rd, q[2]));
  m.y = __dadd_rn(q[1], __dmul_rn(rd, q[3]));
  const int cx = clamp_cell(__dmul_rn(__dsub_rn(m.x, a.x0), a.inv_g), a.nx);
  const int cy = a.ny == 1 ? 0 : clamp_cell(__dmul_rn(__dsub_rn(m.y, a.y0), a.inv_g), a.ny);
  m.cell = cx * a.ny + cy;
  return m;
}

__global__ void __launch_bounds__(256) count_kernel(const BinArgs a) {
  const int cells = a.nx * a.ny;
  const int64_t total = static_cast<int64_t>(a.rows) * a.Nd;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / a.Nd), k = static_cast<int>(i - static_cast<int64_t>(r) * a.Nd);
    const Mover m = mover_at(a, r, k);
    atomicAdd(a.dst + static_cast<size_t>(r) * (cells + 1) + m.cell + 1, 1);
  }
}

// One block per row: inclusive scan of the counts into starts (entry 0 stays
// 0), and the scatter cursors = starts.
__global__ void __launch_bounds__(1024) scan_kernel(const BinArgs a) {
  __shared__ int warp_sum[32];
  const int cells = a.nx * a.ny;
  int32_t* st = a.dst + static_cast<size_t>(blockIdx.x) * (cells + 1);
  int32_t* cur = a.cursor + static_cast<size_t>(blockIdx.x) * cells;
  const int n = cells + 1;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, static_cast<int>(threadIdx.x) * per), hi = min(n, lo + per);
  int local = 0;
  for (int i = lo; i < hi; ++i) local += st[i];
  // exclusive scan of the thread totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < static_cast<int>(blockDim.x >> 5) ? warp_sum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    warp_sum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int run = incl - local + (warp > 0 ? warp_sum[warp - 1] : 0);
  for (int i = lo; i < hi; ++i) {
    run += st[i];
    st[i] = run;
    if (i < cells) cur[i] = run;  // start of cell i = inclusive sum through i
  }
}

__global__ void __launch_bounds__(256) scatter_kernel(const BinArgs a) {
  const int cells = a.nx * a.ny;
  const int64_t total = static_cast<int64_t>(a.rows) * a.Nd;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / a.Nd), k = static_cast<int>(i - static_cast<int64_t>(r) * a.Nd);
    const Mover m = mover_at(a, r, k);
    const int slot = atomicAdd(a.cursor + static_cast<size_t>(r) * cells + m.cell, 1);
    const size_t o = static_cast<size_t>(r) * a.Nd + slot;
    if (a.fp64) {
      static_cast<double2*>(a.dpts)[o] = make_double2(m.x, m.y);
    } else {
      static_cast<float2*>(a.dpts)[o] = make_float2(static_cast<float>(m.x), static_cast<float>(m.y));
    }
  }
}

}  // namespace

int bin_movers(const BinArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cells = a.nx * a.ny;
  cudaError_t e = cudaMemsetAsync(a.dst, 0, sizeof(int32_t) * a.rows * static_cast<size_t>(cells + 1), st);
  if (e != cudaSuccess) return static_cast<int>(e);
  const int64_t total = static_cast<int64_t>(a.rows) * a.Nd;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, std::max(a.sms, 1) * 32));
  count_kernel<<<blocks, 256, 0, st>>>(a);
  scan_kernel<<<a.rows, 1024, 0, st>>>(a);
  scatter_kernel<<<blocks, 256, 0, st>>>(a);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace ppdev
