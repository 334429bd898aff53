// Explicit instantiation unit (parallel build); see vd_kernels.cuh.
#include "vd_launcher_impl.cuh"

namespace vdk {
template int Launcher<Chain7D>::rnea(const Chain7D&, const Launch&, const void*, const void*, const void*, const double*, const void*, void*);
}  // namespace vdk
