// Experiment: branch-parallel G1 ABA (codegen.gen_aba_role, three warp roles
// per group of 32 states) against the single-thread generated ABA, across
// batch sizes.  Build: python tools/gen_roles.py && nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr
// -Ipaper_2604_04310_b200/csrc -Iablib tools/roles_sweep.cu -o ablib/roles_sweep
#include <cstdio>
#include <cmath>
#include <vector>
#include <algorithm>
#include "vd_gen_robots.cuh"
#include "vd_gen_kernels.cuh"
#include "roles_gen.cuh"
using namespace vdk;

template <class T, int kSlots, int kReg, int kSmem, int kBlk>
struct GenRoleCx : GenCx<T, kSlots, kReg, kSmem, false, false, 0, kBlk> {
  uint32_t xb;  // exchange element (0, lane)
  __device__ __forceinline__ void xput(int k, T v) const { GenMem<T>::sts(xb + (uint32_t)(k * 32 * sizeof(T)), v); }
  __device__ __forceinline__ T xget(int k) const { return GenMem<T>::lds(xb + (uint32_t)(k * 32 * sizeof(T))); }
  __device__ __forceinline__ void role_sync() const { __syncthreads(); }
};

template <class Cx, class T>
__device__ __forceinline__ void setup(Cx& cx, uint32_t sbase, uint32_t xb, T* scratch, int64_t slot, int kGmax,
                                      const T* x0, const T* x1, const T* x2, int64_t i, int64_t ld, T* y, int64_t ldo,
                                      bool active, T g0, T g1, T g2) {
  cx.sm = sbase + threadIdx.x * (uint32_t)sizeof(T);
  cx.sb = scratch + (slot >> 5) * (int64_t)(kGmax * 32) + (slot & 31);
  cx.xb = xb;
  cx.in_[0] = x0 + i;
  cx.in_[1] = x1 + i;
  cx.in_[2] = x2 + i;
  cx.out_ = y + i;
  cx.fx_ = nullptr;
  cx.ld = ld;
  cx.ldo = ldo;
  cx.active = active;
  cx.g3[0] = g0;
  cx.g3[1] = g1;
  cx.g3[2] = g2;
}

template <class Rs, class T, int kReg, int kSmem, int kMinB>
__global__ void __launch_bounds__(96, kMinB)
    k_gen_roles(int64_t N, const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2, int64_t ldi,
                T g0, T g1, T g2, T* __restrict__ y, int64_t ldo, int32_t* __restrict__ status, T* __restrict__ scratch,
                int kGmax) {
  constexpr int R = 3, kBlk = 96;
  extern __shared__ __align__(16) unsigned char smem[];
  const int role = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t xb = sbase + (uint32_t)(kSmem * kBlk * sizeof(T)) + lane * (uint32_t)sizeof(T);
  int* flags = reinterpret_cast<int*>(smem + kSmem * kBlk * sizeof(T) + (R * 27 + 6) * 32 * sizeof(T));
  const int64_t slot = (int64_t)blockIdx.x * kBlk + threadIdx.x;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < N; base += (int64_t)gridDim.x * 32) {
    const int64_t i0 = base + lane;
    const bool active = i0 < N;
    const int64_t i = active ? i0 : N - 1;
    bool ok;
    if (role == 0) {
      GenRoleCx<T, Rs::Role0::kSlots, kReg, kSmem, kBlk> cx;
      setup(cx, sbase, xb, scratch, slot, kGmax, x0, x1, x2, i, ldi, y, ldo, active, g0, g1, g2);
      ok = Rs::Role0::template run<T>(cx);
    } else if (role == 1) {
      GenRoleCx<T, Rs::Role1::kSlots, kReg, kSmem, kBlk> cx;
      setup(cx, sbase, xb, scratch, slot, kGmax, x0, x1, x2, i, ldi, y, ldo, active, g0, g1, g2);
      ok = Rs::Role1::template run<T>(cx);
    } else {
      GenRoleCx<T, Rs::Role2::kSlots, kReg, kSmem, kBlk> cx;
      setup(cx, sbase, xb, scratch, slot, kGmax, x0, x1, x2, i, ldi, y, ldo, active, g0, g1, g2);
      ok = Rs::Role2::template run<T>(cx);
    }
    flags[role * 32 + lane] = ok;
    __syncthreads();
    if (role == 0 && active) {
      const bool all = flags[lane] && flags[32 + lane] && flags[64 + lane];
      if (!all)
        for (int j = 0; j < Rs::kN; ++j) y[(int64_t)j * ldo + i] = T(0);
      if (status) status[i] = all ? 0 : 7;
    }
    __syncthreads();
  }
}

template <class T>
__global__ void k_fill(T* p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    p[i] = T((double)(x >> 11) * (1.0 / 9007199254740992.0) * 6.283185307179586 - 3.141592653589793);
  }
}

template <class K, class... A>
float timed(K kern, dim3 grid, int blk, size_t smem, A... args) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) kern<<<grid, blk, smem>>>(args...);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) kern<<<grid, blk, smem>>>(args...);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 20;
}

template <int kReg, int kSmem, int kMinB>
void run_roles(const char* name, int64_t N, double* x, double* y, double* y_ref, int32_t* st, double* scratch) {
  using Rs = GenTree29Roles;
  constexpr int kBlk = 96;
  auto kern = k_gen_roles<Rs, double, kReg, kSmem, kMinB>;
  const size_t smem = (size_t)kSmem * kBlk * 8 + (3 * 27 + 6) * 32 * 8 + 3 * 32 * 4;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kBlk, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int kG = std::max(std::max(Rs::Role0::kSlots, Rs::Role1::kSlots), Rs::Role2::kSlots) - kReg - kSmem;
  const int kGmax = kG > 0 ? kG : 0;
  const int64_t grid = std::min<int64_t>((N + 31) / 32, (int64_t)sms * std::max(bps, 1));
  const double* x0 = x;
  const double* x1 = x + N * 29;
  const double* x2 = x + 2 * N * 29;
  float ms = timed(kern, dim3((unsigned)grid), kBlk, smem, N, x0, x1, x2, N, 0.0, 0.0, 9.81, y, N, st, scratch, kGmax);
  std::vector<double> a((size_t)N * 29), b((size_t)N * 29);
  cudaMemcpy(a.data(), y, a.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), y_ref, b.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0;
  for (size_t k = 0; k < a.size(); ++k) md = std::max(md, std::fabs(a[k] - b[k]) / std::max(1.0, std::fabs(b[k])));
  printf("%-28s N %8lld b/SM %d  %.4f ms  %.3e evals/s  maxdiff %.2e  %s\n", name, (long long)N, bps, ms,
         N / (ms * 1e-3), md, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *x, *y, *y_ref, *scratch;
  int32_t* st;
  const int64_t Nmax = 262144;
  cudaMalloc(&x, sizeof(double) * Nmax * 87);
  cudaMalloc(&y, sizeof(double) * Nmax * 29);
  cudaMalloc(&y_ref, sizeof(double) * Nmax * 29);
  cudaMalloc(&scratch, 1ull << 30);
  cudaMalloc(&st, sizeof(int32_t) * Nmax);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int64_t N : {1024LL, 4096LL, 16384LL, 65536LL, 262144LL}) {
    k_fill<<<1184, 256>>>(x, N * 87, 2);
    // reference: the shipped single-thread kernel (r40 s113 b2, evict-first)
    auto kref = k_gen<GenTree29::Aba, double, 40, 113, 2, false, true>;
    const size_t smem = 113 * 128 * 8;
    cudaFuncSetAttribute(kref, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t grid = std::min<int64_t>((N + 127) / 128, (int64_t)sms * 2);
    float ms = timed(kref, dim3((unsigned)grid), 128, smem, N, (const double*)x, (const double*)(x + N * 29),
                     (const double*)(x + 2 * N * 29), N, 0.0, 0.0, 9.81, y_ref, N, st, scratch, (const double*)nullptr,
                     (const double*)nullptr);
    printf("%-28s N %8lld          %.4f ms  %.3e evals/s\n", "single-thread k_gen", (long long)N, ms, N / (ms * 1e-3));
    run_roles<40, 74, 2>("roles r40 s74 b2", N, x, y, y_ref, st, scratch);
    run_roles<40, 40, 3>("roles r40 s40 b3", N, x, y, y_ref, st, scratch);
    run_roles<60, 60, 2>("roles r60 s60 b2", N, x, y, y_ref, st, scratch);
  }
  return 0;
}
