// Launchers for the generated straight-line robot kernels (vd_gen_kernels.cuh).
// tree29 (G1) ABA runs here: the fully unrolled template kernel is dominated
// by flag/select overhead and the loop kernel by local-memory state (see
// DESIGN.md "Generated kernels").
#include <algorithm>
#include <mutex>

#include "vd_gen_kernels.cuh"
#include "vd_launch.hpp"

namespace vdk {
namespace {

// Per-dtype placement of the 267 pass-2 -> pass-3 state slots (ablib/gen_sweep.cu
// on B200): fp64 keeps the last 40 slots in registers and the first 110 (the
// prologue's cos/sin/q̇ of every joint + the first leg) in shared memory at 2
// CTAs/SM; fp32 puts 110 slots in shared memory at 4 CTAs/SM.
template <class T>
struct GenAbaCfg;
template <>
struct GenAbaCfg<double> {
  static constexpr int kReg = 40, kSmem = 110, kMinB = 2;
};
template <>
struct GenAbaCfg<float> {
  static constexpr int kReg = 0, kSmem = 110, kMinB = 4;
};

struct Occ {
  int blocks_per_sm = 0, sms = 0;
};

template <class R, class T>
int launch_gen_aba_t(const Launch& L, const T* q, const T* qd, const T* tau, const double* g3, T* qdd,
                     int32_t* status) {
  using C = GenAbaCfg<T>;
  auto kern = k_gen_aba<R, T, C::kReg, C::kSmem, C::kMinB>;
  constexpr size_t smem = (size_t)C::kSmem * kGenBlock * sizeof(T);
  static std::once_flag once;
  static Occ occ[64];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once, [&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
  Occ o;
  {
    std::lock_guard<std::mutex> lk(mu);
    Occ& c = occ[dev & 63];
    if (!c.blocks_per_sm) {
      cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.blocks_per_sm, kern, kGenBlock, smem);
      if (c.blocks_per_sm < 1) c.blocks_per_sm = 1;
    }
    o = c;
  }
  const int64_t blocks = std::min<int64_t>((L.N + kGenBlock - 1) / kGenBlock, (int64_t)o.sms * o.blocks_per_sm);
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  // L2-resident scratch for the slots that are neither in registers nor in
  // shared memory: one slab per resident thread, stream-ordered from the
  // device's memory pool (no synchronisation, safe for concurrent streams).
  const size_t scratch_bytes = (size_t)blocks * kGenBlock * gen_aba_scratch_per_thread<R, T, C::kReg, C::kSmem>() * sizeof(T);
  T* scratch = nullptr;
  if (scratch_bytes) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), scratch_bytes, s);
    if (e != cudaSuccess) return (int)e;
  }
  // gravity3 == NULL: GravitySpec::standard() (dynamics.hpp:39-50), as g3_of
  const T g0 = g3 ? T(g3[0]) : T(0), g1 = g3 ? T(g3[1]) : T(0), g2 = g3 ? T(g3[2]) : T(9.81);
  kern<<<(unsigned)blocks, kGenBlock, smem, s>>>(L.N, q, qd, tau, L.ld_in, g0, g1, g2, qdd, L.ld_out, status, scratch);
  cudaError_t e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, s);
  return (int)e;
}

}  // namespace

int launch_gen_aba(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* qdd,
                   int32_t* status) {
  if (L.spec != kTree29) return -1;
  if (L.dtype == 0)
    return launch_gen_aba_t<GenTree29, double>(L, (const double*)q, (const double*)qd, (const double*)tau, g3,
                                               (double*)qdd, status);
  return launch_gen_aba_t<GenTree29, float>(L, (const float*)q, (const float*)qd, (const float*)tau, g3, (float*)qdd,
                                            status);
}

}  // namespace vdk
