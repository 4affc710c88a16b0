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
