// Host-side dispatch from a Launch descriptor to the per-view launchers.
#include "vd_kernels.cuh"

namespace vdk {

extern template struct Launcher<GenericD>;
extern template struct Launcher<GenericF>;
extern template struct Launcher<Chain7D>;
extern template struct Launcher<Chain7F>;

namespace {

// kTreeStatic: whether the compile-time tree29 kernels exist for this op.
// Fully unrolled 29-joint ABA/CRBA/OSC exceed the instruction cache, so those
// run the loop-based kernels with the model in parameter space instead.
template <bool kTreeStatic, class T, class Fn>
int with_view_t(const Launch& L, Fn&& fn) {
  if (L.spec == kChain7) return fn(StaticView<RobotChain7, T>{});
  if constexpr (kTreeStatic) {
    if (L.spec == kTree29) return fn(StaticView<RobotTree29, T>{});
  }
  return fn(RuntimeView<T>{*static_cast<const DevModel<T>*>(L.model)});
}
template <bool kTreeStatic = false, class Fn>
int with_view(const Launch& L, Fn&& fn) {
  return L.dtype == 0 ? with_view_t<kTreeStatic, double>(L, fn) : with_view_t<kTreeStatic, float>(L, fn);
}

}  // namespace

int match_spec(uint64_t fp, int n) { return match_spec_tables(fp, n); }

int launch_fk(const Launch& L, const void* q, void* out) {
  if (L.N == 0) return 0;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::fk(mv, L, q, out); });
}

int launch_jacobian(const Launch& L, const void* q, int frame_joint, const double* frame_R, const double* frame_p,
                    void* pose, void* J) {
  if (L.N == 0) return 0;
  FrameArg fr;
  fr.joint = frame_joint;
  for (int k = 0; k < 9; ++k) fr.R[k] = frame_R[k];
  for (int k = 0; k < 3; ++k) fr.p[k] = frame_p[k];
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::jac(mv, L, q, fr, pose, J); });
}

int launch_rnea(const Launch& L, int mode, const void* q, const void* qd, const void* qdd, const double* g3,
                const void* fext, void* tau) {
  if (L.N == 0) return 0;
  static const double zero3[3] = {0, 0, 0};
  const double* g = (mode == 3) ? zero3 : g3;
  const void* qd_ = (mode == 2) ? nullptr : qd;
  const void* qdd_ = (mode == 0) ? qdd : nullptr;
  return with_view<true>(L, [&](auto mv) { return Launcher<decltype(mv)>::rnea(mv, L, q, qd_, qdd_, g, fext, tau); });
}

int launch_crba(const Launch& L, const void* q, void* M) {
  if (L.N == 0) return 0;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::crba(mv, L, q, M); });
}

int launch_aba(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, const void* fext,
               void* qdd, int32_t* status) {
  if (L.N == 0) return 0;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::aba(mv, L, q, qd, tau, g3, fext, qdd, status); });
}

int launch_dynamics(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* M,
                    void* bias, void* qdd, int32_t* status) {
  if (L.N == 0) return 0;
  return with_view(L,
                   [&](auto mv) { return Launcher<decltype(mv)>::dyn(mv, L, q, qd, tau, g3, M, bias, qdd, status); });
}

int launch_osc(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lambda,
               int32_t* status) {
  if (L.N == 0) return 0;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::osc(mv, L, q, qd, P, tau, lambda, status); });
}

}  // namespace vdk
