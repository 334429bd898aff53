// Placement/occupancy sweep of the generated kernels (tools/gen_tree_kernels.py) on one GPU.
// Build: nvcc [-DSWEEP_STREAM=true] -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr -Ipaper_2604_04310_b200/csrc tools/gen_sweep.cu -o ablib/gen_sweep
#include <cstdio>
#include <cstring>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include "vd_gen_robots.cuh"
#include "vd_gen_kernels.cuh"
using namespace vdk;
// -DSWEEP_STREAM=true: evict-first state I/O (GenCx kStream) for every k_gen entry
#ifndef SWEEP_STREAM
#define SWEEP_STREAM false
#endif
static const char* g_filter = nullptr;
template <class T>
__global__ void k_fill(T* p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    p[i] = T((double)(x >> 11) * (1.0 / 9007199254740992.0) * 6.283185307179586 - 3.141592653589793);
  }
}
template <class Op, class T, int kReg, int kSmem, int kMinB, bool kFast = false>
void run(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch, size_t cap, int n) {
  if (g_filter && !strstr(name, g_filter)) return;
  auto kern = k_gen<Op, T, kReg, kSmem, kMinB, kFast, SWEEP_STREAM>;
  size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int64_t grid = (int64_t)sms * bps;
  if ((size_t)(grid * kGenBlock * gen_scratch_per_thread<Op, T, kReg, kSmem>() * sizeof(T)) > cap) { printf("%s scratch\n", name); return; }
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const T* x0 = x; const T* x1 = x + N * n; const T* x2 = x + 2 * N * n;
  for (int w = 0; w < 3; ++w) kern<<<grid, kGenBlock, smem>>>(N, x0, x1, x2, N, T(0), T(0), T(9.81), y, N, st, scratch, nullptr, nullptr);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) kern<<<grid, kGenBlock, smem>>>(N, x0, x1, x2, N, T(0), T(0), T(9.81), y, N, st, scratch, nullptr, nullptr);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  double bytes = (double)N * (Op::kIn * n + Op::kOut) * sizeof(T);
  printf("%-26s regs %3d lmem %4zu smem %6zu b/SM %d  %.4f ms  %.3e evals/s  %6.2f TF(gen)  %6.0f GB/s  %s\n", name, fa.numRegs,
         fa.localSizeBytes, smem, bps, ms, N / (ms * 1e-3), (double)Op::kFlops * N / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}
template <class Op, class T, int kReg, int kSmem, int kMinB>
void run_osc(const char* name, int64_t N, T* x, T* y, T* lam, int32_t* st, T* scratch, size_t cap, int n) {
  if (g_filter && !strstr(name, g_filter)) return;
  auto kern = k_gen_osc<Op, T, kReg, kSmem, kMinB>;
  size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // SWEEP_CTAS_PER_SM caps the persistent grid below the occupancy limit so
  // the per-thread L2 scratch slab can be sized to fit L2.
  if (const char* e = getenv("SWEEP_CTAS_PER_SM")) bps = std::min(bps, atoi(e));
  int64_t grid = (int64_t)sms * bps;
  if ((size_t)(grid * kGenBlock * gen_scratch_per_thread<Op, T, kReg, kSmem>() * sizeof(T)) > cap) { printf("%s scratch\n", name); return; }
  OscShared P{};
  for (int k = 0; k < 9; ++k) P.frame_R[k] = P.target_R[k] = (k % 4 == 0) ? 1.0 : 0.0;
  P.target_p[2] = 0.3;
  for (int k = 0; k < 6; ++k) { P.kp[k] = 100; P.kd[k] = 20; }
  P.posture_kp = 10; P.posture_kd = 2; P.gravity[2] = 9.81; P.epsilon = 1e-6;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, N, P, y, lam, N, st, scratch);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, N, P, y, lam, N, st, scratch);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  printf("%-26s regs %3d lmem %4zu smem %6zu b/SM %d scratch %5.0f MB  %.4f ms  %.3e evals/s  %6.2f TF(gen)  %s\n", name, fa.numRegs,
         fa.localSizeBytes, smem, bps, grid * kGenBlock * gen_scratch_per_thread<Op, T, kReg, kSmem>() * sizeof(T) / 1e6, ms,
         N / (ms * 1e-3), (double)Op::kFlops * N / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  if (argc > 1) g_filter = argv[1];
  size_t cap = 1ull << 31;
  const int64_t N = 262144; const int n = 29;
  double *xd, *yd, *sd; float *xf, *yf, *sf; int32_t* st;
  cudaMalloc(&xd, 3 * N * n * 8); cudaMalloc(&yd, N * n * n * 8); cudaMalloc(&sd, cap); cudaMalloc(&st, N * 4);
  k_fill<<<1024, 256>>>(xd, 3 * N * n, 1);
  using R = GenTree29;
  {
    double* lam; cudaMalloc(&lam, 36 * N * 8);
    run_osc<R::Osc23, double, 0, 110, 2>("t29 osc f64 s110 b2", N, xd, yd, lam, st, sd, cap, n);
    run_osc<R::Osc23, double, 0, 110, 1>("t29 osc f64 s110 b1", N, xd, yd, lam, st, sd, cap, n);
    run_osc<R::Osc23, double, 0, 220, 1>("t29 osc f64 s220 b1", N, xd, yd, lam, st, sd, cap, n);
    run_osc<R::Osc23, double, 0, 55, 3>("t29 osc f64 s55 b3", N, xd, yd, lam, st, sd, cap, n);
    run_osc<R::Osc23, double, 0, 0, 2>("t29 osc f64 s0 b2", N, xd, yd, lam, st, sd, cap, n);
    float* lf; cudaMalloc(&lf, 36 * N * 4);
    float *xf0, *yf0; cudaMalloc(&xf0, 3 * N * n * 4); cudaMalloc(&yf0, N * n * 4);
    k_fill<<<1024, 256>>>(xf0, 3 * N * n, 1);
    run_osc<R::Osc23, float, 0, 110, 3>("t29 osc f32 s110 b3", N, xf0, yf0, lf, st, (float*)sd, cap, n);
    run_osc<R::Osc23, float, 0, 220, 2>("t29 osc f32 s220 b2", N, xf0, yf0, lf, st, (float*)sd, cap, n);
    run_osc<R::Osc23, float, 0, 110, 2>("t29 osc f32 s110 b2", N, xf0, yf0, lf, st, (float*)sd, cap, n);
    run_osc<R::Osc23, float, 0, 0, 4>("t29 osc f32 s0 b4", N, xf0, yf0, lf, st, (float*)sd, cap, n);
  }
  run<R::Rnea, double, 0, 55, 3>("t29 rnea f64 s55 b3", N, xd, yd, st, sd, cap, n);
  run<R::Rnea, double, 0, 113, 2>("t29 rnea f64 s113 b2", N, xd, yd, st, sd, cap, n);
  run<R::Rnea, double, 0, 0, 3>("t29 rnea f64 s0 b3", N, xd, yd, st, sd, cap, n);
  run<R::Rnea, double, 58, 55, 2>("t29 rnea f64 r58 s55 b2", N, xd, yd, st, sd, cap, n);
  run<R::Rnea, double, 0, 72, 3>("t29 rnea f64 s72 b3", N, xd, yd, st, sd, cap, n);
  run<R::RneaBias, double, 0, 55, 3>("t29 bias f64 s55 b3", N, xd, yd, st, sd, cap, n);
  run<R::RneaBias, double, 0, 72, 3>("t29 bias f64 s72 b3", N, xd, yd, st, sd, cap, n);
  run<R::RneaGrav, double, 0, 55, 3>("t29 grav f64 s55 b3", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 40, 110, 2>("t29 aba f64 r40 s110 b2", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 20, 110, 2>("t29 aba f64 r20 s110 b2", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 60, 110, 2>("t29 aba f64 r60 s110 b2", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 80, 100, 2>("t29 aba f64 r80 s100 b2", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 40, 84, 2>("t29 aba f64 r40 s84 b2", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 40, 200, 1>("t29 aba f64 r40 s200 b1", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 40, 113, 2>("t29 aba f64 r40 s113 b2", N, xd, yd, st, sd, cap, n);
  run<R::Aba, double, 40, 72, 3>("t29 aba f64 r40 s72 b3", N, xd, yd, st, sd, cap, n);
  run<R::Crba, double, 0, 55, 2>("t29 crba f64 s55 b2", N, xd, yd, st, sd, cap, n);
  run<R::Crba, double, 0, 55, 3>("t29 crba f64 s55 b3", N, xd, yd, st, sd, cap, n);
  run<R::Crba, double, 0, 0, 4>("t29 crba f64 s0 b4", N, xd, yd, st, sd, cap, n);
  run<R::Crba, double, 0, 40, 4>("t29 crba f64 s40 b4", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 40, 4>("t29 crbap f64 s40 b4", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 55, 4>("t29 crbap f64 s55 b4", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 28, 6>("t29 crbap f64 s28 b6", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 24, 6>("t29 crbap f64 s24 b6", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 20, 8>("t29 crbap f64 s20 b8", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 0, 8>("t29 crbap f64 s0 b8", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 0, 0, 6>("t29 crbap f64 s0 b6", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 55, 0, 3>("t29 crbap f64 r55 b3", N, xd, yd, st, sd, cap, n);
  run<R::CrbaPacked, double, 55, 0, 4>("t29 crbap f64 r55 b4", N, xd, yd, st, sd, cap, n);
  run<R::Fk, double, 0, 55, 3>("t29 fk f64 s55 b3", N, xd, yd, st, sd, cap, n);
  run<R::Fk, double, 0, 0, 4>("t29 fk f64 s0 b4", N, xd, yd, st, sd, cap, n);
  run<R::Fk, double, 0, 40, 4>("t29 fk f64 s40 b4", N, xd, yd, st, sd, cap, n);
  run<R::Fk, double, 55, 0, 3>("t29 fk f64 r55 b3", N, xd, yd, st, sd, cap, n);
  cudaMalloc(&xf, 3 * N * n * 4); cudaMalloc(&yf, N * n * n * 4); cudaMalloc(&sf, cap);
  k_fill<<<1024, 256>>>(xf, 3 * N * n, 1);
  run<R::AbaMixed, float, 40, 110, 3>("t29 abamix f32 r40 s110 b3", N, xf, yf, st, sf, cap, n);
  run<R::AbaMixed, float, 40, 122, 3>("t29 abamix f32 r40 s122 b3", N, xf, yf, st, sf, cap, n);
  run<R::AbaMixed, float, 40, 160, 3>("t29 abamix f32 r40 s160 b3", N, xf, yf, st, sf, cap, n);
  run<R::Rnea, float, 0, 55, 4>("t29 rnea f32 s55 b4", N, xf, yf, st, sf, cap, n);
  run<R::Rnea, float, 0, 113, 4>("t29 rnea f32 s113 b4", N, xf, yf, st, sf, cap, n);
  run<R::Rnea, float, 0, 113, 3>("t29 rnea f32 s113 b3", N, xf, yf, st, sf, cap, n);
  run<R::Rnea, float, 55, 0, 3>("t29 rnea f32 r55 b3", N, xf, yf, st, sf, cap, n);
  run<R::Crba, float, 0, 55, 4>("t29 crba f32 s55 b4", N, xf, yf, st, sf, cap, n);
  run<R::Crba, float, 55, 0, 3>("t29 crba f32 r55 b3", N, xf, yf, st, sf, cap, n);
  run<R::CrbaPacked, float, 0, 55, 4>("t29 crbap f32 s55 b4", N, xf, yf, st, sf, cap, n);
  run<R::CrbaPacked, float, 0, 55, 6>("t29 crbap f32 s55 b6", N, xf, yf, st, sf, cap, n);
  run<R::CrbaPacked, float, 0, 40, 8>("t29 crbap f32 s40 b8", N, xf, yf, st, sf, cap, n);
  run<R::CrbaPacked, float, 0, 0, 8>("t29 crbap f32 s0 b8", N, xf, yf, st, sf, cap, n);
  run<R::CrbaPacked, float, 55, 0, 4>("t29 crbap f32 r55 b4", N, xf, yf, st, sf, cap, n);
  run<R::Fk, float, 0, 55, 4>("t29 fk f32 s55 b4", N, xf, yf, st, sf, cap, n);
  run<R::Fk, float, 55, 0, 4>("t29 fk f32 r55 b4", N, xf, yf, st, sf, cap, n);
  // chain7 (N = 4M) vs the template kernels
  const int64_t N7 = 4194304;
  double *x7, *y7; cudaMalloc(&x7, 3 * N7 * 7 * 8); cudaMalloc(&y7, N7 * 49 * 8);
  cudaFree(st); cudaMalloc(&st, N7 * 4);
  k_fill<<<1024, 256>>>(x7, 3 * N7 * 7, 2);
  using C = GenChain7;
  run<C::CrbaPacked, double, 14, 0, 4>("c7 crbap f64 allreg b4", N7, x7, y7, st, sd, cap, 7);
  run<C::CrbaPacked, double, 14, 0, 6>("c7 crbap f64 allreg b6", N7, x7, y7, st, sd, cap, 7);
  run<C::CrbaPacked, double, 14, 0, 8>("c7 crbap f64 allreg b8", N7, x7, y7, st, sd, cap, 7);
  run<C::CrbaPacked, double, 0, 14, 8>("c7 crbap f64 s14 b8", N7, x7, y7, st, sd, cap, 7);
  run<C::Crba, double, 14, 0, 4>("c7 crba f64 allreg b4", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, C::Aba::kSlots, 0, 3>("c7 aba f64 allreg b3", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, C::Aba::kSlots, 0, 4>("c7 aba f64 allreg b4", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, 44, 28, 3>("c7 aba f64 r44 s28 b3", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, 44, 28, 4>("c7 aba f64 r44 s28 b4", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, 44, 28, 4, true>("c7 aba f64 r44 s28 b4 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, 44, 28, 3, true>("c7 aba f64 r44 s28 b3 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, 72, 0, 4, true>("c7 aba f64 allreg b4 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Aba, double, 0, 28, 4>("c7 aba f64 s28 b4", N7, x7, y7, st, sd, cap, 7);
  run<C::Rnea, double, 28, 0, 4, true>("c7 rnea f64 r28 b4 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Rnea, double, 28, 0, 3, true>("c7 rnea f64 r28 b3 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Rnea, double, 0, 28, 4, true>("c7 rnea f64 s28 b4 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Crba, double, 14, 0, 4, true>("c7 crba f64 r14 b4 fast", N7, x7, y7, st, sd, cap, 7);
  run<C::Fk, double, 14, 0, 4, true>("c7 fk f64 r14 b4 fast", N7, x7, y7, st, sd, cap, 7);
  {
    float *x7f, *y7f; cudaMalloc(&x7f, 3 * N7 * 7 * 4); cudaMalloc(&y7f, N7 * 49 * 4);
    k_fill<<<1024, 256>>>(x7f, 3 * N7 * 7, 2);
    run<C::Aba, float, C::Aba::kSlots, 0, 4>("c7 aba f32 allreg b4", N7, x7f, y7f, st, (float*)sd, cap, 7);
    run<C::Aba, float, 44, 28, 4>("c7 aba f32 r44 s28 b4", N7, x7f, y7f, st, (float*)sd, cap, 7);
    run<C::Aba, float, 44, 28, 6>("c7 aba f32 r44 s28 b6", N7, x7f, y7f, st, (float*)sd, cap, 7);
    run<C::Rnea, float, 28, 0, 6>("c7 rnea f32 r28 b6", N7, x7f, y7f, st, (float*)sd, cap, 7);
    double* lam7; cudaMalloc(&lam7, 36 * N7 * 8);
    run_osc<C::Osc6, double, 0, 55, 3>("c7 osc f64 s55 b3", N7, x7, y7, lam7, st, sd, cap, 7);
    run_osc<C::Osc6, double, 60, 55, 2>("c7 osc f64 r60 s55 b2", N7, x7, y7, lam7, st, sd, cap, 7);
    run_osc<C::Osc6, double, 0, 147, 2>("c7 osc f64 s147 b2", N7, x7, y7, lam7, st, sd, cap, 7);
  }

  return 0;
}
