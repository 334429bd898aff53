// Explicit instantiation unit (parallel build); see vd_kernels.cuh.
#include "vd_launcher_impl.cuh"

namespace vdk {
template int Launcher<Tree29D>::aba(const Tree29D&, const Launch&, const void*, const void*, const void*, const double*, const void*, void*, int32_t*);
template int Launcher<Tree29D>::dyn(const Tree29D&, const Launch&, const void*, const void*, const void*, const double*, void*, void*, void*, int32_t*);
}  // namespace vdk
