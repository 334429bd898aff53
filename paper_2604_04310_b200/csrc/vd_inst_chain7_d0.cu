// Explicit instantiation unit (parallel build); see vd_kernels.cuh.
#include "vd_launcher_impl.cuh"

namespace vdk {
template int Launcher<Chain7D>::fk(const Chain7D&, const Launch&, const void*, void*);
template int Launcher<Chain7D>::jac(const Chain7D&, const Launch&, const void*, const FrameArg&, void*, void*);
template int Launcher<Chain7D>::crba(const Chain7D&, const Launch&, const void*, void*);
template int Launcher<Chain7D>::task(const Chain7D&, const Launch&, const void*, const TaskShared&, int, void*, void*, int32_t*);
}  // namespace vdk
