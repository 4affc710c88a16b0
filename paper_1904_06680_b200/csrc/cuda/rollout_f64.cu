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
                                                       uint4* __restrict__ dst, int n16) {
  wait_prior_grid();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    dst[i] = __ldcg(src + i);
  }
}

int launch_copy_out(const void* src, void* host_dst, size_t bytes, void* stream) {
  if (bytes % 16 != 0) return static_cast<int>(cudaErrorInvalidValue);
  void* dst = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dst, host_dst, 0);
  if (e != cudaSuccess) return static_cast<int>(e);
  const int n16 = static_cast<int>(bytes / 16);
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
                                             static_cast<uint4*>(dst), n16));
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
