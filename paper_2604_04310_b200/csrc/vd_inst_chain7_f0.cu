// Explicit instantiation unit (parallel build); see vd_kernels.cuh.
#include "vd_launcher_impl.cuh"

namespace vdk {
template int Launcher<Chain7F>::fk(const Chain7F&, const Launch&, const void*, void*);
template int Launcher<Chain7F>::jac(const Chain7F&, const Launch&, const void*, const FrameArg&, void*, void*);
template int Launcher<Chain7F>::crba(const Chain7F&, const Launch&, const void*, void*);
template int Launcher<Chain7F>::task(const Chain7F&, const Launch&, const void*, const TaskShared&, int, void*, void*, int32_t*);
}  // namespace vdk
