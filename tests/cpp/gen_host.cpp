// Host build of the generated straight-line robot routines
// (paper_2604_04310_b200/csrc/vd_gen_robots.cuh) for the CPU test suite:
// the same generated arithmetic the sm_100a kernels run, checked here against
// the oracle (tests/test_gen_host.py).  Test infrastructure only.
#include <cstring>
#include <vector>

#include "vd_gen_robots.cuh"

namespace {
template <class T>
struct HostCx {
  static constexpr bool kFastTrig = false;
  const T* X[3];
  const double* G;
  T* Y;
  long ld, i;
  T* slots;
  // OSC parameters (gen_osc_host layout): fR 9, fp 3, tR 9, tp 3, kp 6, kd 6, aff 6, pkp, pkd, eps, posture n
  const double* P = nullptr;
  T* Y1 = nullptr;
  T* Y2 = nullptr;  // output group 2 (the fused Dyn routine's q̈)
  const T* DX[3] = {nullptr, nullptr, nullptr};  // JVP tangents (NULL = 0)
  const T* FX = nullptr;                         // external wrenches, plane 6 j + k
  T x(int g, int j) const { return X[g] ? X[g][j * ld + i] : T(0); }
  T dx(int g, int j) const { return DX[g] ? DX[g][j * ld + i] : T(0); }
  T fx(int k) const { return FX[k * ld + i]; }
  void prefetch(int, int) const {}
  void fetch_next(int) const {}
  template <int K>
  void phase() const {}
  T g(int k) const { return T(G[k]); }
  void st(int k, T v) { slots[k] = v; }
  T get(int k) const { return slots[k]; }
  void st2(int k, double v) { std::memcpy(&slots[k], &v, sizeof(double)); }  // slots k (and k + 1 for float)
  double get2(int k) const {
    double v;
    std::memcpy(&v, &slots[k], sizeof(double));
    return v;
  }
  void y(int o, int k, T v) const { (o == 0 ? Y : o == 1 ? Y1 : Y2)[k * ld + i] = v; }
  T fR(int k) const { return T(P[k]); }
  T fp(int k) const { return T(P[9 + k]); }
  T tR(int k) const { return T(P[12 + k]); }
  T tp(int k) const { return T(P[21 + k]); }
  T kp(int k) const { return T(P[24 + k]); }
  T kd(int k) const { return T(P[30 + k]); }
  T aff(int k) const { return T(P[36 + k]); }
  T pkp() const { return T(P[42]); }
  T pkd() const { return T(P[43]); }
  T eps() const { return T(P[44]); }
  T post(int k) const { return T(P[45 + k]); }
  T tw(int k) const { return T(P[30 + k]); }  // diff-IK: twist_ff in the kd slots, damping in eps
  T damp() const { return T(P[44]); }
  bool want_lambda() const { return Y1 != nullptr; }
};
template <class Op, class T>
int run(long N, const void* const* x, const double* g, void* y, int* status, const void* fext = nullptr) {
  std::vector<T> slots(Op::kSlots + 1);
  int bad = 0;
  for (long i = 0; i < N; ++i) {
    HostCx<T> cx{{(const T*)x[0], (const T*)x[1], (const T*)x[2]}, g, (T*)y, N, i, slots.data()};
    cx.FX = (const T*)fext;
    const bool ok = Op::template run<T>(cx);
    status[i] = ok ? 0 : 7;
    bad += !ok;
  }
  return bad;
}
template <class R, class T>
int run_op(int op, long N, const void* const* x, const double* g, void* y, int* status, const void* fext = nullptr) {
  switch (op) {
    case 8: return run<typename R::RneaFext, T>(N, x, g, y, status, fext);
    case 9: return run<typename R::RneaBiasFext, T>(N, x, g, y, status, fext);
    case 10:
      if constexpr (sizeof(T) == 4) return run<typename R::AbaMixedFext, T>(N, x, g, y, status, fext);
      else return run<typename R::AbaFext, T>(N, x, g, y, status, fext);
    case 0:  // fp32: the mixed-precision routine the device uses
      if constexpr (sizeof(T) == 4) return run<typename R::AbaMixed, T>(N, x, g, y, status);
      else return run<typename R::Aba, T>(N, x, g, y, status);
    case 6: return run<typename R::Aba, T>(N, x, g, y, status);  // plain fp32 ABA (comparison)
    case 1: return run<typename R::Rnea, T>(N, x, g, y, status);
    case 2: return run<typename R::RneaBias, T>(N, x, g, y, status);
    case 3: return run<typename R::RneaGrav, T>(N, x, g, y, status);
    case 4: return run<typename R::Crba, T>(N, x, g, y, status);
    case 7: return run<typename R::CrbaPacked, T>(N, x, g, y, status);
    default: return run<typename R::Fk, T>(N, x, g, y, status);
  }
}

template <class R>
int osc(int fj, long N, const double* q, const double* qd, const double* g, const double* P, double* tau,
        double* lam, int* status) {
  int bad = -1;
  R::with_osc(fj, [&](auto op) {
    using Op = decltype(op);
    std::vector<double> slots(Op::kSlots + 1);
    bad = 0;
    for (long i = 0; i < N; ++i) {
      HostCx<double> cx{{q, qd, q}, g, tau, N, i, slots.data()};
      cx.P = P;
      cx.Y1 = lam;
      const bool ok = Op::template run<double>(cx);
      status[i] = ok ? 0 : 7;
      bad += !ok;
    }
  });
  return bad;
}
}  // namespace

// the fused chain7 M + bias + q̈ routine (GenChain7::Dyn), fp64
extern "C" int gen_dyn_host(long N, const double* q, const double* qd, const double* tau, const double* g, double* M,
                            double* bias, double* qdd, int* status) {
  using Op = vdk::GenChain7::Dyn;
  std::vector<double> slots(Op::kSlots + 1);
  int bad = 0;
  for (long i = 0; i < N; ++i) {
    HostCx<double> cx{{q, qd, tau}, g, M, N, i, slots.data()};
    cx.Y1 = bias;
    cx.Y2 = qdd;
    const bool ok = Op::template run<double>(cx);
    status[i] = ok ? 0 : 7;
    bad += !ok;
  }
  return bad;
}

// generated osc_step on frame joint fj (fp64); -1 when no variant exists for fj
extern "C" int gen_osc_host(int robot, int fj, long N, const double* q, const double* qd, const double* g,
                            const double* P, double* tau, double* lam, int* status) {
  return robot == 2 ? osc<vdk::GenTree29>(fj, N, q, qd, g, P, tau, lam, status)
                    : osc<vdk::GenChain7>(fj, N, q, qd, g, P, tau, lam, status);
}
template <class Op>
int jvp(long N, const double* const* x, const double* const* dx, const double* g, double* y, double* dy,
        int* status) {
  std::vector<double> slots(Op::kSlots + 1);
  int bad = 0;
  for (long i = 0; i < N; ++i) {
    HostCx<double> cx{{x[0], x[1], x[2]}, g, y, N, i, slots.data()};
    cx.Y1 = dy;
    for (int k = 0; k < 3; ++k) cx.DX[k] = dx[k];
    const bool ok = Op::template run<double>(cx);
    status[i] = ok ? 0 : 7;
    bad += !ok;
  }
  return bad;
}

// generated forward-mode JVP, fp64: op 0 forward dynamics (ABA), 1 RNEA, 2 CRBA, 3 FK (tree29)
extern "C" int gen_jvp_host(int robot, int op, long N, const double* x0, const double* x1, const double* x2,
                            const double* dx0, const double* dx1, const double* dx2, const double* g, double* y,
                            double* dy, int* status) {
  const double* x[3] = {x0, x1, x2};
  const double* dx[3] = {dx0, dx1, dx2};
  if (robot == 2) {
    switch (op) {
      case 0: return jvp<vdk::GenTree29::AbaJvp>(N, x, dx, g, y, dy, status);
      case 1: return jvp<vdk::GenTree29::RneaJvp>(N, x, dx, g, y, dy, status);
      case 2: return jvp<vdk::GenTree29::CrbaJvp>(N, x, dx, g, y, dy, status);
      default: return jvp<vdk::GenTree29::FkJvp>(N, x, dx, g, y, dy, status);
    }
  }
  return op == 0 ? jvp<vdk::GenChain7::AbaJvp>(N, x, dx, g, y, dy, status)
                 : jvp<vdk::GenChain7::RneaJvp>(N, x, dx, g, y, dy, status);
}

// generated task-space routine on frame joint fj (fp64): which 0 Jacobian (y0 pose 12, y1 J 6n),
// 1 diff-IK (y0 q̇, y1 err), 2 manipulability (y0); -1 when no variant exists for fj
extern "C" int gen_task_host(int which, int fj, long N, const double* q, const double* P, double* y0, double* y1,
                             int* status, const double* dq) {
  int bad = -1;
  vdk::GenTree29::with_task(fj, [&](auto jac, auto dik, auto man, auto man_jvp) {
    auto go = [&](auto op) {
      using Op = decltype(op);
      std::vector<double> slots(Op::kSlots + 1);
      bad = 0;
      for (long i = 0; i < N; ++i) {
        HostCx<double> cx{{q, q, q}, nullptr, y0, N, i, slots.data()};
        cx.P = P;
        cx.Y1 = y1;
        cx.DX[0] = dq;
        const bool ok = Op::template run<double>(cx);
        status[i] = ok ? 0 : 7;
        bad += !ok;
      }
    };
    if (which == 0) go(jac);
    else if (which == 1) go(dik);
    else if (which == 2) go(man);
    else go(man_jvp);
  });
  return bad;
}

// op: 0 aba, 1 rnea, 2 bias, 3 gravity, 4 crba, 5 fk; robot: 1 chain7, 2 tree29
extern "C" int gen_run_host(int robot, int op, int f32, long N, const void* x0, const void* x1, const void* x2,
                            const double* g, void* y, int* status) {
  const void* x[3] = {x0, x1 ? x1 : x0, x2 ? x2 : x0};
  if (robot == 2)
    return f32 ? run_op<vdk::GenTree29, float>(op, N, x, g, y, status)
               : run_op<vdk::GenTree29, double>(op, N, x, g, y, status);
  return f32 ? run_op<vdk::GenChain7, float>(op, N, x, g, y, status)
             : run_op<vdk::GenChain7, double>(op, N, x, g, y, status);
}

// op: 8 rnea + f_ext, 9 bias + f_ext, 10 aba + f_ext (fp32: the mixed-precision routine); fext: 6n planes
extern "C" int gen_run_fext_host(int robot, int op, int f32, long N, const void* x0, const void* x1, const void* x2,
                                 const void* fext, const double* g, void* y, int* status) {
  const void* x[3] = {x0, x1 ? x1 : x0, x2 ? x2 : x0};
  if (robot == 2)
    return f32 ? run_op<vdk::GenTree29, float>(op, N, x, g, y, status, fext)
               : run_op<vdk::GenTree29, double>(op, N, x, g, y, status, fext);
  return f32 ? run_op<vdk::GenChain7, float>(op, N, x, g, y, status, fext)
             : run_op<vdk::GenChain7, double>(op, N, x, g, y, status, fext);
}
