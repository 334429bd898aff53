// A/B of k_gen (plain state loads) against k_gen_async (cp.async prefetch of
// the next state's inputs) for the generated ABA routines, on one GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr
//        -Ipaper_2604_04310_b200/csrc tools/async_sweep.cu -o ablib/async_sweep
// Prints time per launch and the max |difference| of each variant's output
// against the plain kernel's (the same generated arithmetic: expected 0).
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "vd_gen_robots.cuh"
#include "vd_gen_kernels.cuh"
using namespace vdk;

template <class T>
__global__ void k_fill(T* p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    p[i] = T((double)(x >> 11) * (1.0 / 9007199254740992.0) * 6.283185307179586 - 3.141592653589793);
  }
}

static std::vector<double> g_ref;

template <class T, class K>
void time_kernel(const char* name, K kern, size_t smem, size_t scratch_per_thread, int64_t N, int n, int nout, T* x,
                 T* y, int32_t* st, T* scratch, size_t cap, bool is_ref, int blk = kGenBlock) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, blk, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (bps < 1) { printf("%-40s does not fit\n", name); return; }
  const int64_t grid = std::min<int64_t>((int64_t)sms * bps, (N + blk - 1) / blk);
  if ((size_t)grid * blk * scratch_per_thread * sizeof(T) > cap) { printf("%s scratch\n", name); return; }
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const T *x0 = x, *x1 = x + N * n, *x2 = x + 2 * N * n;
  cudaMemset(y, 0, sizeof(T) * N * nout);
  for (int w = 0; w < 3; ++w) kern<<<grid, blk, smem>>>(N, x0, x1, x2, N, T(0), T(0), T(9.81), y, N, st, scratch, nullptr, nullptr);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) kern<<<grid, blk, smem>>>(N, x0, x1, x2, N, T(0), T(0), T(9.81), y, N, st, scratch, nullptr, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  std::vector<T> h((size_t)N * nout);
  cudaMemcpy(h.data(), y, sizeof(T) * h.size(), cudaMemcpyDeviceToHost);
  double md = 0;
  if (is_ref) {
    g_ref.assign(h.begin(), h.end());
  } else {
    for (size_t k = 0; k < h.size(); ++k) md = std::max(md, std::fabs((double)h[k] - g_ref[k]) / std::max(1.0, std::fabs(g_ref[k])));
  }
  printf("%-40s regs %3d lmem %4zu smem %6zu b/SM %d  %.4f ms  %.3e evals/s  maxdiff %.2e  %s\n", name, fa.numRegs,
         fa.localSizeBytes, smem, bps, ms, N / (ms * 1e-3), md, cudaGetErrorString(cudaGetLastError()));
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast, bool kStream, int kSync = 0>
void plain(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch, size_t cap, bool ref = false) {
  time_kernel<T>(name, k_gen<Op, T, kReg, kSmem, kMinB, kFast, kStream, kSync>, (size_t)kSmem * kGenBlock * sizeof(T),
                 gen_scratch_per_thread<Op, T, kReg, kSmem>(), N, Op::kDof, Op::kOut, x, y, st, scratch, cap, ref);
}
template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast, bool kStream, int kSync, int kBlk>
void plainb(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch, size_t cap, bool ref = false) {
  time_kernel<T>(name, k_gen<Op, T, kReg, kSmem, kMinB, kFast, kStream, kSync, kBlk>, (size_t)kSmem * kBlk * sizeof(T),
                 gen_scratch_per_thread<Op, T, kReg, kSmem>(), N, Op::kDof, Op::kOut, x, y, st, scratch, cap, ref, kBlk);
}
template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast, bool kStream = false, int kSync = 0>
void async(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch, size_t cap, bool ref = false) {
  time_kernel<T>(name, k_gen_async<Op, T, kReg, kSmem, kMinB, kFast, kStream, kSync>, gen_async_smem<Op, T, kReg, kSmem>(),
                 gen_scratch_per_thread<Op, T, kReg, kSmem>(), N, Op::kDof, Op::kOut, x, y, st, scratch, cap, ref);
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig = kTrigLib>
void osc(const char* name, int64_t N, T* x, T* y, T* lam, int32_t* st, T* scratch, size_t cap, int n, bool ref = false) {
  auto kern = k_gen_osc<Op, T, kReg, kSmem, kMinB, kTrig>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t grid = std::min<int64_t>((int64_t)sms * bps, (N + kGenBlock - 1) / kGenBlock);
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
  const int reps = 10;
  for (int r = 0; r < reps; ++r) kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, N, P, y, lam, N, st, scratch);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  printf("%-40s regs %3d lmem %4zu smem %6zu b/SM %d  %.4f ms  %.3e evals/s  %s\n", name, fa.numRegs, fa.localSizeBytes,
         smem, bps, ms, N / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}

template <class Op, class T, int kReg, int kSmem, int kMinB>
void task(const char* name, int64_t N, T* x, T* y0, T* y1, int32_t* st) {
  auto kern = k_gen_task<Op, T, kReg, kSmem, kMinB>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t grid = std::min<int64_t>((int64_t)sms * bps, (N + kGenBlock - 1) / kGenBlock);
  TaskShared P{};
  for (int k = 0; k < 9; ++k) P.frame_R[k] = P.target_R[k] = (k % 4 == 0) ? 1.0 : 0.0;
  P.frame_p[2] = 0.1;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) kern<<<grid, kGenBlock, smem>>>(N, x, N, P, y0, y1, N, st, nullptr, (const T*)nullptr);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) kern<<<grid, kGenBlock, smem>>>(N, x, N, P, y0, y1, N, st, nullptr, (const T*)nullptr);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  printf("%-40s regs %3d lmem %4zu smem %6zu b/SM %d  %.4f ms  %.3e evals/s  %s\n", name, fa.numRegs, fa.localSizeBytes,
         smem, bps, ms, N / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig = kTrigLib>
void jvp(const char* name, int64_t N, T* x, T* y, T* scratch, size_t cap) {
  auto kern = k_gen_jvp<Op, T, kReg, kSmem, kMinB, true, kTrig>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t grid = std::min<int64_t>((int64_t)sms * bps, (N + kGenBlock - 1) / kGenBlock);
  if ((size_t)(grid * kGenBlock * gen_scratch_per_thread<Op, T, kReg, kSmem>() * sizeof(T)) > cap) { printf("%s scratch\n", name); return; }
  const int n = Op::kDof;
  JvpArgs a{};
  for (int g = 0; g < Op::kIn; ++g) { a.x[g] = x + g * N * n; a.dx[g] = x + (3 + g) * N * n; }
  a.g[2] = 9.81;
  a.out = y;
  a.dout = y + (int64_t)Op::kOut * N;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) kern<<<grid, kGenBlock, smem>>>(N, a, N, N, scratch);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) kern<<<grid, kGenBlock, smem>>>(N, a, N, N, scratch);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  printf("%-40s regs %3d lmem %4zu smem %6zu b/SM %d  %.4f ms  %.3e evals/s  %s\n", name, fa.numRegs, fa.localSizeBytes,
         smem, bps, ms, N / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}

#define ON(k) (!strcmp(which, "all") || !strcmp(which, k))
int main(int argc, char** argv) {
  const char* which = argc > 1 ? argv[1] : "all";
  const size_t cap = 1ull << 30;
  double *x, *y, *scratch;
  int32_t* st;
  const int64_t Nmax = 4194304;
  cudaMalloc(&x, sizeof(double) * Nmax * 7 * 3);
  cudaMalloc(&y, sizeof(double) * 4194304 * 84);
  cudaMalloc(&scratch, cap);
  cudaMalloc(&st, sizeof(int32_t) * Nmax);
  float* xf = (float*)x;
  float* yf = (float*)y;
  float* sf = (float*)scratch;
  const int64_t N7 = 4194304, N29 = 262144;
  if (ON("c7")) {
    k_fill<<<1184, 256>>>(x, N7 * 21, 1);
    plain<GenChain7::Aba, double, 44, 28, 4, true, false>("c7 aba f64 plain r44 s28 b4", N7, x, y, st, scratch, cap, true);
    async<GenChain7::Aba, double, 30, 35, 4, true>("c7 aba f64 async r30 s35 b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Aba, double, 24, 41, 4, true>("c7 aba f64 async r24 s41 b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Aba, double, 36, 29, 4, true>("c7 aba f64 async r36 s29 b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Aba, double, 16, 49, 4, true>("c7 aba f64 async r16 s49 b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Aba, double, 30, 35, 4, true, true>("c7 aba f64 async r30 s35 b4 cs", N7, x, y, st, scratch, cap);
  }
  if (ON("sync")) {
    k_fill<<<1184, 256>>>(x, N7 * 21, 1);
    async<GenChain7::Aba, double, 24, 41, 3, true, true>("c7 aba f64 async r24 s41 cs", N7, x, y, st, scratch, cap, true);
    async<GenChain7::Aba, double, 24, 41, 3, true, true, 1>("c7 aba f64 async r24 s41 cs sync1", N7, x, y, st, scratch, cap);
    async<GenChain7::Aba, double, 24, 41, 3, true, true, 3>("c7 aba f64 async r24 s41 cs sync3", N7, x, y, st, scratch, cap);
    async<GenChain7::Aba, double, 24, 41, 3, true, true, 7>("c7 aba f64 async r24 s41 cs sync7", N7, x, y, st, scratch, cap);
    k_fill<<<1184, 256>>>(x, N29 * 87, 2);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true>("t29 aba f64 plain", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true, 1>("t29 aba f64 plain sync1", N29, x, y, st, scratch, cap);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true, 2>("t29 aba f64 plain sync2", N29, x, y, st, scratch, cap);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true, 4>("t29 aba f64 plain sync4", N29, x, y, st, scratch, cap);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true, 8>("t29 aba f64 plain sync8", N29, x, y, st, scratch, cap);
    plain<GenTree29::Aba, double, 40, 60, 3, false, true, 2>("t29 aba f64 r40 s60 b3 sync2", N29, x, y, st, scratch, cap);
    plain<GenTree29::Rnea, double, 58, 55, 2, false, false>("t29 rnea f64 plain", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::Rnea, double, 58, 55, 2, false, false, 2>("t29 rnea f64 plain sync2", N29, x, y, st, scratch, cap);
    plain<GenTree29::Rnea, double, 58, 55, 2, false, false, 4>("t29 rnea f64 plain sync4", N29, x, y, st, scratch, cap);
  }
  if (ON("blk")) {
    k_fill<<<1184, 256>>>(x, N29 * 87, 2);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true>("t29 aba f64 plain", N29, x, y, st, scratch, cap, true);
    plainb<GenTree29::Aba, double, 40, 110, 1, false, true, 0, 256>("t29 aba blk256 s110", N29, x, y, st, scratch, cap);
    plainb<GenTree29::Aba, double, 40, 110, 1, false, true, 1, 256>("t29 aba blk256 s110 sync1", N29, x, y, st, scratch, cap);
    plainb<GenTree29::Aba, double, 40, 110, 1, false, true, 2, 256>("t29 aba blk256 s110 sync2", N29, x, y, st, scratch, cap);
    plainb<GenTree29::Aba, double, 40, 110, 1, false, true, 4, 256>("t29 aba blk256 s110 sync4", N29, x, y, st, scratch, cap);
    plainb<GenTree29::Aba, double, 40, 54, 1, false, true, 2, 512>("t29 aba blk512 s54 sync2", N29, x, y, st, scratch, cap);
    plainb<GenTree29::Aba, double, 40, 54, 1, false, true, 0, 512>("t29 aba blk512 s54", N29, x, y, st, scratch, cap);
    plain<GenTree29::Rnea, double, 58, 55, 2, false, false>("t29 rnea f64 plain", N29, x, y, st, scratch, cap, true);
    plainb<GenTree29::Rnea, double, 58, 55, 1, false, false, 2, 256>("t29 rnea blk256 sync2", N29, x, y, st, scratch, cap);
    plainb<GenTree29::Rnea, double, 58, 55, 1, false, false, 0, 256>("t29 rnea blk256", N29, x, y, st, scratch, cap);
  }
  if (ON("more")) {
    k_fill<<<1184, 256>>>(x, N7 * 21, 1);
    constexpr int S7 = GenChain7::Osc6::kSlots;
    double* lam = nullptr;
    cudaMalloc(&lam, sizeof(double) * 36 * N7);
    osc<GenChain7::Osc6, double, 0, 55, 3>("c7 osc f64 s55 b3", N7, x, y, lam, st, scratch, cap, 7);
    osc<GenChain7::Osc6, double, 60, 55, 2>("c7 osc f64 r60 s55 b2", N7, x, y, lam, st, scratch, cap, 7);
    osc<GenChain7::Osc6, double, 0, S7 < 100 ? S7 : 100, 2>("c7 osc f64 s100 b2", N7, x, y, lam, st, scratch, cap, 7);
    osc<GenChain7::Osc6, double, 40, 70, 2>("c7 osc f64 r40 s70 b2", N7, x, y, lam, st, scratch, cap, 7);
    osc<GenChain7::Osc6, double, 60, 87, 2>("c7 osc f64 r60 s87 b2", N7, x, y, lam, st, scratch, cap, 7);
    osc<GenChain7::Osc6, double, 80, 67, 2>("c7 osc f64 r80 s67 b2", N7, x, y, lam, st, scratch, cap, 7);
    osc<GenChain7::Osc6, double, 40, 55, 2>("c7 osc f64 r40 s55 b2", N7, x, y, lam, st, scratch, cap, 7);
    k_fill<<<1184, 256>>>(xf, N7 * 21, 1);
    osc<GenChain7::Osc6, float, 0, 147, 3>("c7 osc f32 s147 b3", N7, xf, yf, (float*)lam, st, sf, cap, 7);
    osc<GenChain7::Osc6, float, 60, 87, 3>("c7 osc f32 r60 s87 b3", N7, xf, yf, (float*)lam, st, sf, cap, 7);
    osc<GenChain7::Osc6, float, 60, 87, 2>("c7 osc f32 r60 s87 b2", N7, xf, yf, (float*)lam, st, sf, cap, 7);
    osc<GenChain7::Osc6, float, 40, 107, 4>("c7 osc f32 r40 s107 b4", N7, xf, yf, (float*)lam, st, sf, cap, 7);
    cudaFree(lam);
    cudaMalloc(&lam, sizeof(double) * 36 * N29);
    k_fill<<<1184, 256>>>(x, N29 * 87, 2);
    osc<GenTree29::Osc23, double, 0, 55, 3>("t29 osc23 f64 s55 b3", N29, x, y, lam, st, scratch, cap, 29);
    osc<GenTree29::Osc23, double, 0, 110, 2>("t29 osc23 f64 s110 b2", N29, x, y, lam, st, scratch, cap, 29);
    osc<GenTree29::Osc23, double, 40, 55, 3>("t29 osc23 f64 r40 s55 b3", N29, x, y, lam, st, scratch, cap, 29);
    osc<GenTree29::Osc23, double, 40, 110, 2>("t29 osc23 f64 r40 s110 b2", N29, x, y, lam, st, scratch, cap, 29);
    osc<GenTree29::Osc23, double, 0, 72, 3>("t29 osc23 f64 s72 b3", N29, x, y, lam, st, scratch, cap, 29);
    osc<GenTree29::Osc23, double, 0, 40, 4>("t29 osc23 f64 s40 b4", N29, x, y, lam, st, scratch, cap, 29);
    osc<GenTree29::Osc23, float, 0, 220, 2>("t29 osc23 f32 s220 b2", N29, xf, yf, (float*)lam, st, sf, cap, 29);
    osc<GenTree29::Osc23, float, 0, 144, 3>("t29 osc23 f32 s144 b3", N29, xf, yf, (float*)lam, st, sf, cap, 29);
    osc<GenTree29::Osc23, float, 40, 144, 3>("t29 osc23 f32 r40 s144 b3", N29, xf, yf, (float*)lam, st, sf, cap, 29);
    osc<GenTree29::Osc23, float, 0, 110, 4>("t29 osc23 f32 s110 b4", N29, xf, yf, (float*)lam, st, sf, cap, 29);
    cudaFree(lam);
    constexpr int SP = GenTree29::CrbaPacked::kSlots;
    plain<GenTree29::CrbaPacked, double, SP, 0, 3, false, false>("t29 crbap f64 plain rall b3", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::CrbaPacked, double, SP, 0, 3, false, true>("t29 crbap f64 plain rall b3 cs", N29, x, y, st, scratch, cap);
    async<GenTree29::CrbaPacked, double, SP, 0, 3, false, true>("t29 crbap f64 async rall b3 cs", N29, x, y, st, scratch, cap);
    async<GenTree29::CrbaPacked, double, SP, 0, 4, false, true>("t29 crbap f64 async rall b4 cs", N29, x, y, st, scratch, cap);
    async<GenTree29::CrbaPacked, double, 0, SP, 4, false, true>("t29 crbap f64 async sall b4 cs", N29, x, y, st, scratch, cap);
    plain<GenTree29::Fk, double, 0, 55, 3, false, true>("t29 fk f64 plain s55 b3 cs", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::Rnea, double, 58, 55, 2, false, true>("t29 rnea f64 plain r58 s55 b2 cs", N29, x, y, st, scratch, cap, true);
  }
  if (ON("jac")) {
    k_fill<<<1184, 256>>>(x, N7 * 21, 1);
    double* J = nullptr;
    cudaMalloc(&J, sizeof(double) * 42 * N7);
    constexpr int SJ = GenChain7::Jac6::kSlots;
    task<GenChain7::Jac6, double, 0, SJ, 3>("c7 jac6 f64 sall b3", N7, x, y, J, st);
    task<GenChain7::Jac6, double, 0, SJ, 4>("c7 jac6 f64 sall b4", N7, x, y, J, st);
    task<GenChain7::Jac6, double, 0, SJ, 5>("c7 jac6 f64 sall b5", N7, x, y, J, st);
    task<GenChain7::Jac6, float, 0, SJ, 6>("c7 jac6 f32 sall b6", N7, xf, yf, (float*)J, st);
    constexpr int SF = GenChain7::Fk::kSlots;
    plain<GenChain7::Fk, double, SF, 0, 4, true, false>("c7 fk f64 plain rall b4", N7, x, y, st, scratch, cap, true);
    plain<GenChain7::Fk, double, SF, 0, 4, true, true>("c7 fk f64 plain rall b4 cs", N7, x, y, st, scratch, cap);
    async<GenChain7::Fk, double, SF, 0, 4, true, true>("c7 fk f64 async rall b4 cs", N7, x, y, st, scratch, cap);
    async<GenChain7::Fk, double, SF, 0, 6, true, true>("c7 fk f64 async rall b6 cs", N7, x, y, st, scratch, cap);
    cudaFree(J);
  }
  if (ON("jvp")) {
    // 6 input planes of N29 x 29 doubles, outputs value + tangent
    double *xj = nullptr, *yj = nullptr;
    cudaMalloc(&xj, sizeof(double) * 6 * 29 * N29);
    cudaMalloc(&yj, sizeof(double) * 2 * 841 * N29);
    k_fill<<<1184, 256>>>(xj, 6 * 29 * N29, 5);
    jvp<GenTree29::CrbaJvp, double, 40, 70, 2>("t29 crbajvp f64 r40 s70 b2", N29, xj, yj, scratch, cap);
    jvp<GenTree29::CrbaJvp, double, 40, 70, 3>("t29 crbajvp f64 r40 s70 b3", N29, xj, yj, scratch, cap);
    jvp<GenTree29::CrbaJvp, double, 0, 55, 3>("t29 crbajvp f64 r0 s55 b3", N29, xj, yj, scratch, cap);
    jvp<GenTree29::CrbaJvp, double, 40, 110, 2>("t29 crbajvp f64 r40 s110 b2 (r1)", N29, xj, yj, scratch, cap);
    jvp<GenTree29::FkJvp, double, 40, 70, 2>("t29 fkjvp f64 r40 s70 b2", N29, xj, yj, scratch, cap);
    jvp<GenTree29::FkJvp, double, 40, 70, 3>("t29 fkjvp f64 r40 s70 b3", N29, xj, yj, scratch, cap);
    jvp<GenTree29::FkJvp, double, 0, 55, 3>("t29 fkjvp f64 r0 s55 b3", N29, xj, yj, scratch, cap);
    jvp<GenTree29::FkJvp, double, 40, 110, 2>("t29 fkjvp f64 r40 s110 b2 (r1)", N29, xj, yj, scratch, cap);
    jvp<GenTree29::CrbaJvp, float, 0, 110, 2>("t29 crbajvp f32 s110 b2", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::CrbaJvp, float, 0, 110, 3>("t29 crbajvp f32 s110 b3", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::FkJvp, float, 0, 110, 2>("t29 fkjvp f32 s110 b2", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::FkJvp, float, 0, 110, 3>("t29 fkjvp f32 s110 b3", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::AbaJvp, double, 40, 110, 2>("t29 abajvp f64 r40 s110 b2", N29, xj, yj, scratch, cap);
    jvp<GenTree29::AbaJvp, double, 40, 220, 1>("t29 abajvp f64 r40 s220 b1", N29, xj, yj, scratch, cap);
    jvp<GenTree29::AbaJvp, double, 60, 110, 2>("t29 abajvp f64 r60 s110 b2", N29, xj, yj, scratch, cap);
    jvp<GenTree29::AbaJvp, double, 0, 55, 3>("t29 abajvp f64 r0 s55 b3", N29, xj, yj, scratch, cap);
    jvp<GenTree29::AbaJvp, float, 0, 220, 2>("t29 abajvp f32 s220 b2", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::AbaJvp, float, 40, 220, 2>("t29 abajvp f32 r40 s220 b2", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::AbaJvp, float, 0, 144, 3>("t29 abajvp f32 s144 b3", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::RneaJvp, double, 40, 110, 2>("t29 rneajvp f64 r40 s110 b2", N29, xj, yj, scratch, cap);
    jvp<GenTree29::RneaJvp, double, 40, 55, 3>("t29 rneajvp f64 r40 s55 b3", N29, xj, yj, scratch, cap);
    jvp<GenTree29::RneaJvp, float, 0, 220, 2>("t29 rneajvp f32 s220 b2", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenTree29::RneaJvp, float, 0, 144, 3>("t29 rneajvp f32 s144 b3", N29, (float*)xj, (float*)yj, sf, cap);
    jvp<GenChain7::AbaJvp, double, 40, 89, 2>("c7 abajvp f64 r40 s89 b2", 1048576, xj, yj, scratch, cap);
    jvp<GenChain7::AbaJvp, double, 40, 40, 3>("c7 abajvp f64 r40 s40 b3", 1048576, xj, yj, scratch, cap);
    jvp<GenChain7::AbaJvp, double, 64, 65, 2>("c7 abajvp f64 r64 s65 b2", 1048576, xj, yj, scratch, cap);
    jvp<GenChain7::RneaJvp, double, 40, 16, 2>("c7 rneajvp f64 r40 s16 b2", 1048576, xj, yj, scratch, cap);
    jvp<GenChain7::RneaJvp, double, 56, 0, 3>("c7 rneajvp f64 r56 b3", 1048576, xj, yj, scratch, cap);
    jvp<GenChain7::RneaJvp, double, 56, 0, 4>("c7 rneajvp f64 r56 b4", 1048576, xj, yj, scratch, cap);
    cudaFree(xj);
    cudaFree(yj);
  }
  if (ON("c7f")) {
    k_fill<<<1184, 256>>>(xf, N7 * 21, 1);
    async<GenChain7::Aba, float, 20, 45, 4, false>("c7 aba f32 async r20 s45 b4", N7, xf, yf, st, sf, cap, true);
    async<GenChain7::Aba, float, 30, 35, 5, false>("c7 aba f32 async r30 s35 b5", N7, xf, yf, st, sf, cap);
    async<GenChain7::Aba, float, 40, 25, 6, false>("c7 aba f32 async r40 s25 b6", N7, xf, yf, st, sf, cap);
    async<GenChain7::Aba, float, 65, 0, 6, false>("c7 aba f32 async r65 s0 b6", N7, xf, yf, st, sf, cap);
    async<GenChain7::AbaMixed, float, 20, 52, 4, false>("c7 abamixed f32 async r20 s52 b4", N7, xf, yf, st, sf, cap);
  }
  if (ON("c7r")) {
    k_fill<<<1184, 256>>>(x, N7 * 21, 1);
    constexpr int S = GenChain7::Rnea::kSlots;
    plain<GenChain7::Rnea, double, S, 0, 4, true, false>("c7 rnea f64 plain", N7, x, y, st, scratch, cap, true);
    async<GenChain7::Rnea, double, S, 0, 4, true>("c7 rnea f64 async rall b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Rnea, double, 0, S, 4, true>("c7 rnea f64 async sall b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Rnea, double, S - 14, 14, 4, true>("c7 rnea f64 async r-14 s14 b4", N7, x, y, st, scratch, cap);
    k_fill<<<1184, 256>>>(xf, N7 * 21, 1);
    plain<GenChain7::Rnea, float, S, 0, 6, true, false>("c7 rnea f32 plain", N7, xf, yf, st, sf, cap, true);
    async<GenChain7::Rnea, float, S, 0, 6, true>("c7 rnea f32 async rall b6", N7, xf, yf, st, sf, cap);
    async<GenChain7::Rnea, float, 0, S, 6, true>("c7 rnea f32 async sall b6", N7, xf, yf, st, sf, cap);
  }
  if (ON("c7c")) {
    k_fill<<<1184, 256>>>(x, N7 * 21, 1);
    constexpr int S = GenChain7::Crba::kSlots;
    plain<GenChain7::Crba, double, S, 0, 4, true, false>("c7 crba f64 plain rall b4", N7, x, y, st, scratch, cap, true);
    plain<GenChain7::Crba, double, S, 0, 4, true, true>("c7 crba f64 plain rall b4 cs", N7, x, y, st, scratch, cap);
    async<GenChain7::Crba, double, S, 0, 4, true>("c7 crba f64 async rall b4", N7, x, y, st, scratch, cap);
    async<GenChain7::Crba, double, S, 0, 4, true, true>("c7 crba f64 async rall b4 cs", N7, x, y, st, scratch, cap);
    async<GenChain7::Crba, double, S, 0, 6, true, true>("c7 crba f64 async rall b6 cs", N7, x, y, st, scratch, cap);
  }
  if (ON("trig")) {  // library sincos inlined (kTrigLib) vs one out-of-line copy (kTrigCall), G1 at 262144
    double* lam = nullptr;
    cudaMalloc(&lam, sizeof(double) * 36 * N29);
    k_fill<<<1184, 256>>>(x, N29 * 87, 2);
    osc<GenTree29::Osc23, double, 40, 110, 2>("t29 osc23 f64 lib", N29, x, y, lam, st, scratch, cap, 29, true);
    osc<GenTree29::Osc23, double, 40, 110, 2, kTrigCall>("t29 osc23 f64 call", N29, x, y, lam, st, scratch, cap, 29);
    k_fill<<<1184, 256>>>(xf, N29 * 87, 2);
    osc<GenTree29::Osc23, float, 40, 144, 3>("t29 osc23 f32 lib", N29, xf, yf, (float*)lam, st, sf, cap, 29, true);
    osc<GenTree29::Osc23, float, 40, 144, 3, kTrigCall>("t29 osc23 f32 call", N29, xf, yf, (float*)lam, st, sf, cap, 29);
    k_fill<<<1184, 256>>>(x, N29 * 29 * 6, 2);
    jvp<GenTree29::AbaJvp, double, 40, 220, 1>("t29 abajvp f64 r40 s220 b1 lib", N29, x, y, scratch, cap);
    jvp<GenTree29::AbaJvp, double, 40, 220, 1, kTrigCall>("t29 abajvp f64 r40 s220 b1 call", N29, x, y, scratch, cap);
    jvp<GenTree29::RneaJvp, double, 40, 110, 2>("t29 rneajvp f64 lib", N29, x, y, scratch, cap);
    k_fill<<<1184, 256>>>(xf, N29 * 29 * 6, 2);
    jvp<GenTree29::AbaJvp, float, 40, 220, 2>("t29 abajvp f32 r40 s220 b2 lib", N29, xf, yf, sf, cap);
    jvp<GenTree29::AbaJvp, float, 40, 220, 2, kTrigCall>("t29 abajvp f32 r40 s220 b2 call", N29, xf, yf, sf, cap);
    jvp<GenTree29::RneaJvp, float, 0, 144, 3>("t29 rneajvp f32 s144 b3 lib", N29, xf, yf, sf, cap);
    jvp<GenTree29::RneaJvp, float, 0, 144, 3, kTrigCall>("t29 rneajvp f32 s144 b3 call", N29, xf, yf, sf, cap);
    k_fill<<<1184, 256>>>(x, N29 * 87, 2);
    plain<GenTree29::RneaGrav, double, 0, 55, 3, false, false>("t29 rneagrav f64 lib", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::RneaGrav, double, 0, 55, 3, kTrigCall, false>("t29 rneagrav f64 call", N29, x, y, st, scratch, cap);
    plain<GenTree29::Crba, double, 0, 55, 3, false, true>("t29 crba f64 lib", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::Crba, double, 0, 55, 3, kTrigCall, true>("t29 crba f64 call", N29, x, y, st, scratch, cap);
  }
  if (ON("t29")) {
    k_fill<<<1184, 256>>>(x, N29 * 87, 2);
    plain<GenTree29::Aba, double, 40, 113, 2, false, true>("t29 aba f64 plain r40 s113 b2 cs", N29, x, y, st, scratch, cap, true);
    plain<GenTree29::Rnea, double, 58, 55, 2, false, false>("t29 rnea f64 plain r58 s55 b2", N29, x, y, st, scratch, cap, true);
    async<GenTree29::Rnea, double, 58, 20, 2, false>("t29 rnea f64 async r58 s20 b2", N29, x, y, st, scratch, cap);
    async<GenTree29::Rnea, double, 58, 20, 2, false, true>("t29 rnea f64 async r58 s20 b2 cs", N29, x, y, st, scratch, cap);
    plain<GenTree29::Crba, double, 0, 55, 3, false, true>("t29 crba f64 plain s55 b3 cs", N29, x, y, st, scratch, cap, true);
    async<GenTree29::Crba, double, 0, 44, 3, false, true>("t29 crba f64 async s44 b3 cs", N29, x, y, st, scratch, cap);
    plain<GenTree29::Fk, double, 0, GenTree29::Fk::kSlots < 55 ? GenTree29::Fk::kSlots : 55, 3, false, false>("t29 fk f64 plain", N29, x, y, st, scratch, cap, true);
    async<GenTree29::Fk, double, 0, GenTree29::Fk::kSlots < 40 ? GenTree29::Fk::kSlots : 40, 3, false, true>("t29 fk f64 async cs", N29, x, y, st, scratch, cap);
  }
  return 0;
}
