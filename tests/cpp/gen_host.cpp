// Host build of the generated straight-line robot routines
// (paper_2604_04310_b200/csrc/vd_gen_robots.cuh) for the CPU test suite:
// the same generated arithmetic the sm_100a kernels run, checked here against
// the oracle (tests/test_gen_host.py).  Test infrastructure only.
#include <vector>

#include "vd_gen_robots.cuh"

namespace {
template <class T>
struct HostCx {
  const T *Q, *QD, *TAU;
  const double* G;
  T* OUT;
  long ld, i;
  T* slots;
  T q(int j) const { return Q[j * ld + i]; }
  T qd(int j) const { return QD[j * ld + i]; }
  T tau(int j) const { return TAU[j * ld + i]; }
  T g(int k) const { return T(G[k]); }
  void st(int k, T v) { slots[k] = v; }
  T get(int k) const { return slots[k]; }
  void qdd(int j, T v) const { OUT[j * ld + i] = v; }
  void sync() const {}
};
template <class R, class T>
int run(long N, const T* q, const T* qd, const T* tau, const double* g, T* out, int* status) {
  std::vector<T> slots(R::kAbaSlots + 1);
  int bad = 0;
  for (long i = 0; i < N; ++i) {
    HostCx<T> cx{q, qd, tau, g, out, N, i, slots.data()};
    const bool ok = R::template aba<T>(cx);
    status[i] = ok ? 0 : 7;
    bad += !ok;
  }
  return bad;
}
}  // namespace

extern "C" int gen_aba_host(int robot, int f32, long N, const void* q, const void* qd, const void* tau,
                            const double* g, void* out, int* status) {
  if (f32) {
    auto f = [&](auto r) {
      return run<decltype(r), float>(N, (const float*)q, (const float*)qd, (const float*)tau, g, (float*)out, status);
    };
    return robot == 2 ? f(vdk::GenTree29{}) : f(vdk::GenChain7{});
  }
  auto d = [&](auto r) {
    return run<decltype(r), double>(N, (const double*)q, (const double*)qd, (const double*)tau, g, (double*)out,
                                    status);
  };
  return robot == 2 ? d(vdk::GenTree29{}) : d(vdk::GenChain7{});
}
extern "C" unsigned long long gen_fingerprint(int robot) {
  return robot == 2 ? vdk::GenTree29::kFingerprint : vdk::GenChain7::kFingerprint;
}
