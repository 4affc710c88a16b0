// rollout_f64.cu -- double instantiation of the fused sampler (rollout.cuh).
#include "rollout.cuh"

namespace ppdev {

int shape_f64(NetKind k, int device, int smem_bytes, int grid, LaunchShape* out) {
  switch (k) {
    case NetKind::k5_2_2:
      return shape_impl<double, NetReg<double, 2>>(device, smem_bytes, grid, out);
    case NetKind::k5_10_2:
      return shape_impl<double, NetReg<double, 10>>(device, smem_bytes, grid, out);
    default:
      return shape_impl<double, NetGlobal<double>>(device, smem_bytes, grid, out);
  }
}

int launch_generate_f64(NetKind k, const RoundArgs& a, void* stream) {
  switch (k) {
    case NetKind::k5_2_2:
      return launch_generate_impl<double, NetReg<double, 2>>(a, stream);
    case NetKind::k5_10_2:
      return launch_generate_impl<double, NetReg<double, 10>>(a, stream);
    default:
      return launch_generate_impl<double, NetGlobal<double>>(a, stream);
  }
}

int launch_rollout_f64(NetKind k, const RoundArgs& a, void* stream) {
  switch (k) {
    case NetKind::k5_2_2:
      return launch_rollout_impl<double, NetReg<double, 2>>(a, stream);
    case NetKind::k5_10_2:
      return launch_rollout_impl<double, NetReg<double, 10>>(a, stream);
    default:
      return launch_rollout_impl<double, NetGlobal<double>>(a, stream);
  }
}

int launch_draw_f64(const RoundArgs& a, void* out, void* stream) {
  return launch_draw_impl<double>(a, out, stream);
}

}  // namespace ppdev

namespace ppdev {

// The re-ranking kernels live in the --fmad=false translation unit.
int launch_select(const RoundArgs& a, void* stream) { return launch_select_impl(a, stream); }

int launch_pack_keys(const RoundArgs& a, void* stream) {
  return static_cast<int>(
      launch_dependent(pack_keys_kernel, 1, 128, 0, static_cast<cudaStream_t>(stream), true, a));
}

// The round's result block, stored straight into pinned host memory by the
// SMs (a dependent launch after the last round kernel). A cudaMemcpyAsync of
// the same ~7 KB spent 7-15 us of GPU time in the copy engine (measured on
// B200 at C2); these stores reach the host in a few us.
__global__ void __launch_bounds__(256) copy_out_kernel(const uint4* __restrict__ src,
                                                       uint4* __restrict__ dst, int n16,
                                                       int stamp16) {
  wait_prior_grid();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    uint4 v = __ldcg(src + i);
    if (i == stamp16) {  // the chunk holding exec[kExecRoundT0] (its upper half)
      const unsigned long long t0 =
          (static_cast<unsigned long long>(v.w) << 32) | static_cast<unsigned long long>(v.z);
      const unsigned long long span = t0 != 0ull ? global_ns() - t0 : 0ull;
      v.z = static_cast<unsigned>(span);
      v.w = static_cast<unsigned>(span >> 32);
      reinterpret_cast<unsigned long long*>(const_cast<uint4*>(src + i))[1] = 0ull;
    }
    dst[i] = v;
  }
}

int launch_copy_out(const void* src, void* host_dst, size_t bytes, size_t exec_off, void* stream) {
  if (bytes % 16 != 0) return static_cast<int>(cudaErrorInvalidValue);
  // the device alias of the pinned block (cached: one lookup per block)
  thread_local const void* last_host = nullptr;
  thread_local void* last_dev = nullptr;
  void* dst = nullptr;
  if (host_dst == last_host) {
    dst = last_dev;
  } else {
    cudaError_t e = cudaHostGetDevicePointer(&dst, host_dst, 0);
    if (e != cudaSuccess) return static_cast<int>(e);
    last_host = host_dst;
    last_dev = dst;
  }
  const int n16 = static_cast<int>(bytes / 16);
  // exec[kExecRoundT0] is the upper 8 bytes of its 16-byte chunk
  static_assert(kExecRoundT0 % 2 == 1, "stamp in the upper half of a 16-byte chunk");
  const int stamp16 = static_cast<int>((exec_off + 8 * kExecRoundT0) / 16);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(std::max(1, std::min((n16 + 255) / 256, 8))));
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, copy_out_kernel, static_cast<const uint4*>(src),
                                             static_cast<uint4*>(dst), n16, stamp16));
}

// ------------------------------------------------ wide-window filter ----
namespace {

__device__ __forceinline__ uint32_t pick_rank(uint32_t meta) {
  const int cls = meta_cls(meta);
  return (static_cast<uint32_t>(2 - cls) << 16) |
         static_cast<uint32_t>(cls == 2 ? meta_tgoal(meta) : 0);
}
// order-preserving bits of a double (any sign)
__device__ __forceinline__ unsigned long long cost_order(double c) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(c));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ double order_cost(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & ~(1ull << 63)) : ~o;
  return __longlong_as_double(static_cast<long long>(b));
}

// Flush a thread's running minimum of restart r: one atomic per warp when the
// warp agrees on r (the usual case: a window is one restart's or sorted).
template <typename T>
__device__ __forceinline__ void flush_min(T* dst, int r, T v) {
  const int r0 = __shfl_sync(kFull, r, 0);
  if (__all_sync(kFull, r == r0)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T w = __shfl_xor_sync(kFull, v, o);
      v = w < v ? w : v;
    }
    if ((threadIdx.x & 31) == 0 && r0 >= 0) atomicMin(dst + r0, v);
  } else if (r >= 0) {
    atomicMin(dst + r, v);
  }
}

// pass 0: best rank per restart; pass 1: best cost at that rank
template <int kPass>
__global__ void __launch_bounds__(256) list_best_kernel(const ListFilterArgs f) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n_pad = (f.n + 31) / 32 * 32;  // whole warps for the shuffles
  int r_cur = -1;
  unsigned long long v_cur = ~0ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_pad;
       i += stride) {
    int r = -1;
    unsigned long long v = ~0ull;
    if (i < f.n) {
      r = static_cast<int>(__ldg(f.list + i) / f.list_count);
      const SKey k = f.keys[i];
      const uint32_t rank = pick_rank(k.meta);
      if (kPass == 0) {
        v = rank;
      } else if (rank == f.rank[r]) {
        v = cost_order(k.cost);
      }
    }
    if (r != r_cur && r >= 0) {
      if (r_cur >= 0) {
        if (kPass == 0) {
          atomicMin(f.rank + r_cur, static_cast<uint32_t>(v_cur));
        } else {
          atomicMin(f.cost + r_cur, v_cur);
        }
      }
      r_cur = r;
      v_cur = ~0ull;
    }
    if (r >= 0 && v < v_cur) v_cur = v;
  }
  if (kPass == 0) {
    flush_min<uint32_t>(f.rank, r_cur, static_cast<uint32_t>(v_cur));
  } else {
    flush_min<unsigned long long>(f.cost, r_cur, v_cur);
  }
}

__global__ void __launch_bounds__(256) list_pick_kernel(const ListFilterArgs f) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n_pad = (f.n + 31) / 32 * 32;
  const int lane = threadIdx.x & 31;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_pad;
       i += stride) {
    bool keep = false;
    int64_t flat = 0;
    SKey k{};
    if (i < f.n) {
      flat = __ldg(f.list + i);
      const int r = static_cast<int>(flat / f.list_count);
      k = f.keys[i];
      if (meta_flagged(k.meta)) {
        keep = true;
      } else if (pick_rank(k.meta) == f.rank[r]) {
        const double b = order_cost(f.cost[r]);
        const int cls = meta_cls(k.meta);
        const double tol =
            cls == 2 ? rho2_of(f.rho2, f.rho2_floor, meta_tgoal(k.meta)) : f.rho;
        keep = fabs(k.cost - b) <= 2.0 * tol * fmax(1.0, fabs(b));
      }
    }
    const unsigned m = __ballot_sync(kFull, keep);
    if (m == 0u) continue;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(f.count, static_cast<unsigned>(__popc(m)));
    base = __shfl_sync(kFull, base, 0);
    if (keep) f.out[base + __popc(m & ((1u << lane) - 1u))] = ListPick{flat, k};
  }
}

}  // namespace

int launch_list_filter(const ListFilterArgs& f, void* stream) {
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = std::min<int64_t>((f.n + 255) / 256, int64_t{f.sms} * 8);
  const unsigned g = static_cast<unsigned>(std::max<int64_t>(1, blocks));
  list_best_kernel<0><<<g, 256, 0, st>>>(f);
  list_best_kernel<1><<<g, 256, 0, st>>>(f);
  list_pick_kernel<<<g, 256, 0, st>>>(f);
  return static_cast<int>(cudaGetLastError());
}

int refine_occupancy(NetKind k) {
  switch (k) {
    case NetKind::k5_2_2:
      return refine_occupancy_impl<NetReg<double, 2>>();
    case NetKind::k5_10_2:
      return refine_occupancy_impl<NetReg<double, 10>>();
    default:
      return refine_occupancy_impl<NetGlobal<double>>();
  }
}

int launch_refine(NetKind k, const RoundArgs& a, void* stream) {
  switch (k) {
    case NetKind::k5_2_2:
      return launch_refine_impl<NetReg<double, 2>>(a, stream);
    case NetKind::k5_10_2:
      return launch_refine_impl<NetReg<double, 10>>(a, stream);
    default:
      return launch_refine_impl<NetGlobal<double>>(a, stream);
  }
}

}  // namespace ppdev
