// JVP kernels, fp32 views (vd_jvp.cuh).
#include "vd_jvp.cuh"

namespace vdk {

int launch_manip_jvp_f32(const Launch& L, const void* q, const void* dq, const TaskShared& P, void* w, void* dw) {
  if (L.spec == kChain7) return launch_manip_jvp_view(Chain7F{}, L, q, dq, P, w, dw);
  return launch_manip_jvp_view(GenericF{*static_cast<const DevModel<float>*>(L.model)}, L, q, dq, P, w, dw);
}

int launch_jvp_f32(const Launch& L, const JvpArgs& a) {
  if (L.spec == kChain7) return launch_jvp_view(Chain7F{}, L, a);
  return launch_jvp_view(GenericF{*static_cast<const DevModel<float>*>(L.model)}, L, a);
}

}  // namespace vdk
