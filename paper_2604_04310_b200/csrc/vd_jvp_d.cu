// JVP kernels, fp64 views (vd_jvp.cuh), and the launch_jvp dispatcher.
#include "vd_jvp.cuh"

namespace vdk {

int launch_jvp_f32(const Launch& L, const JvpArgs& a);

int launch_jvp(const Launch& L, const JvpArgs& a) {
  if (L.N == 0) return 0;
  if (const int rc = launch_gen_jvp(L, a); rc >= 0) return rc;
  if (L.dtype != 0) return launch_jvp_f32(L, a);
  if (L.spec == kChain7) return launch_jvp_view(Chain7D{}, L, a);
  return launch_jvp_view(GenericD{*static_cast<const DevModel<double>*>(L.model)}, L, a);
}

}  // namespace vdk
