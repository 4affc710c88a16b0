// rollout_f32.cu -- float instantiation of the fused sampler (rollout.cuh).
#include "rollout.cuh"

namespace ppdev {

int shape_f32(NetKind k, int device, int smem_bytes, int grid, LaunchShape* out) {
  switch (k) {
    case NetKind::k5_2_2:
      return shape_impl<float, NetReg<float, 2>>(device, smem_bytes, grid, out);
    case NetKind::k5_10_10_2:
      return shape_impl<float, NetReg3<float, 10, 10>>(device, smem_bytes, grid, out);
    case NetKind::k5_10_2:
      return shape_impl<float, NetReg<float, 10>>(device, smem_bytes, grid, out);
    default:
      return shape_impl<float, NetGlobal<float>>(device, smem_bytes, grid, out);
  }
}

int launch_generate_f32(NetKind k, const RoundArgs& a, void* stream) {
  switch (k) {
    case NetKind::k5_2_2:
      return launch_generate_impl<float, NetReg<float, 2>>(a, stream);
    case NetKind::k5_10_10_2:
      return launch_generate_impl<float, NetReg3<float, 10, 10>>(a, stream);
    case NetKind::k5_10_2:
      return launch_generate_impl<float, NetReg<float, 10>>(a, stream);
    default:
      return launch_generate_impl<float, NetGlobal<float>>(a, stream);
  }
}

int launch_rollout_f32(NetKind k, const RoundArgs& a, void* stream) {
  switch (k) {
    case NetKind::k5_2_2:
      return launch_rollout_impl<float, NetReg<float, 2>>(a, stream);
    case NetKind::k5_10_10_2:
      return launch_rollout_impl<float, NetReg3<float, 10, 10>>(a, stream);
    case NetKind::k5_10_2:
      return launch_rollout_impl<float, NetReg<float, 10>>(a, stream);
    default:
      return launch_rollout_impl<float, NetGlobal<float>>(a, stream);
  }
}

int launch_draw_f32(const RoundArgs& a, void* out, void* stream) {
  return launch_draw_impl<float>(a, out, stream);
}

}  // namespace ppdev
