// Explicit instantiation unit (parallel build); see vd_kernels.cuh.
#include "vd_launcher_impl.cuh"

namespace vdk {
template struct Launcher<GenericD>;
template struct Launcher<GenericF>;
}  // namespace vdk
