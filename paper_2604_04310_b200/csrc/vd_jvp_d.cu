// JVP kernels, fp64 views (vd_jvp.cuh), and the launch_jvp dispatcher.
#include "vd_jvp.cuh"

namespace vdk {

int launch_jvp_f32(const Launch& L, const JvpArgs& a);
int launch_manip_jvp_f32(const Launch& L, const void* q, const void* dq, const TaskShared& P, void* w, void* dw);

int launch_manip_jvp(const Launch& L, const void* q, const void* dq, const TaskShared& P, void* w, void* dw) {
  if (L.N == 0) return 0;
  // generated dual-number routine on a generated frame joint (builtin robot or JIT module)
  if (L.jit_task && P.frame_joint >= 0 && P.frame_joint < 64 && ((L.jit_task_mask >> P.frame_joint) & 1)) {
    if (const int rc = L.jit_task(4, &L, P.frame_joint, q, dq, &P, w, dw, nullptr); rc >= 0) return rc;
  }
  if (const int rc = launch_gen_task(L, 4, P.frame_joint, P, q, w, dw, nullptr, dq); rc >= 0) return rc;
  if (L.dtype != 0) return launch_manip_jvp_f32(L, q, dq, P, w, dw);
  if (L.spec == kChain7) return launch_manip_jvp_view(Chain7D{}, L, q, dq, P, w, dw);
  return launch_manip_jvp_view(GenericD{*static_cast<const DevModel<double>*>(L.model)}, L, q, dq, P, w, dw);
}

int launch_jvp(const Launch& L, const JvpArgs& a) {
  if (L.N == 0) return 0;
  if (const int rc = launch_gen_jvp(L, a); rc >= 0) return rc;
  if (L.dtype != 0) return launch_jvp_f32(L, a);
  if (L.spec == kChain7) return launch_jvp_view(Chain7D{}, L, a);
  return launch_jvp_view(GenericD{*static_cast<const DevModel<double>*>(L.model)}, L, a);
}

}  // namespace vdk
