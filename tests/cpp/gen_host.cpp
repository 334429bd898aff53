// Host build of the generated straight-line robot routines
// (paper_2604_04310_b200/csrc/vd_gen_robots.cuh) for the CPU test suite:
// the same generated arithmetic the sm_100a kernels run, checked here against
// the oracle (tests/test_gen_host.py).  Test infrastructure only.
#include <vector>

#include "vd_gen_robots.cuh"

namespace {
template <class T>
struct HostCx {
  const T* X[3];
  const double* G;
  T* Y;
  long ld, i;
  T* slots;
  T x(int g, int j) const { return X[g][j * ld + i]; }
  T g(int k) const { return T(G[k]); }
  void st(int k, T v) { slots[k] = v; }
  T get(int k) const { return slots[k]; }
  void y(int, int k, T v) const { Y[k * ld + i] = v; }
};
template <class Op, class T>
int run(long N, const void* const* x, const double* g, void* y, int* status) {
  std::vector<T> slots(Op::kSlots + 1);
  int bad = 0;
  for (long i = 0; i < N; ++i) {
    HostCx<T> cx{{(const T*)x[0], (const T*)x[1], (const T*)x[2]}, g, (T*)y, N, i, slots.data()};
    const bool ok = Op::template run<T>(cx);
    status[i] = ok ? 0 : 7;
    bad += !ok;
  }
  return bad;
}
template <class R, class T>
int run_op(int op, long N, const void* const* x, const double* g, void* y, int* status) {
  switch (op) {
    case 0: return run<typename R::Aba, T>(N, x, g, y, status);
    case 1: return run<typename R::Rnea, T>(N, x, g, y, status);
    case 2: return run<typename R::RneaBias, T>(N, x, g, y, status);
    case 3: return run<typename R::RneaGrav, T>(N, x, g, y, status);
    case 4: return run<typename R::Crba, T>(N, x, g, y, status);
    default: return run<typename R::Fk, T>(N, x, g, y, status);
  }
}
}  // namespace

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
