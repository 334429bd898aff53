// A/B of the fused Panda M + bias + q̈ kernel (k_tiled<Chain7, OpDyn>, config 3)
// at 3 vs 4 resident CTAs per SM.  At 65 536 states there are 512 tiles of 128
// states; 3 CTAs/SM (168 registers) give 444 persistent CTAs, so 68 of them run
// a second, lone tile.  4 CTAs/SM (<= 128 registers) fit all 512 in one round.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//          -Xptxas -v -Ipaper_2604_04310_b200/csrc tools/dyn_sweep.cu -o ablib/dyn_sweep
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "vd_kernels.cuh"
#include "vd_gen_robots.cuh"
#include "vd_gen_kernels.cuh"
using namespace vdk;

template <class T, int kMB>
struct OpDynB : OpDyn<T> {
  static constexpr int kMinBlocks = kMB;
};

template <class T>
__global__ void k_fill(T* p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    p[i] = T((double)(x >> 11) * (1.0 / 9007199254740992.0) * 6.283185307179586 - 3.141592653589793);
  }
}

static std::vector<double> g_ref;

template <class T, int kMB>
void run(const char* name, int64_t N, T* x, T* y, int32_t* st) {
  using V = StaticView<RobotChain7, T>;
  using Op = OpDynB<T, kMB>;
  auto kern = k_tiled<V, Op>;
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kBlock, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  const int n = 7;
  Op op{};
  op.g.g[0] = T(0); op.g.g[1] = T(0); op.g.g[2] = T(9.81);
  op.M = y;
  op.bias = y + 49 * N;
  op.qdd = y + 56 * N;
  op.ldo = N;
  op.status = st;
  tma::Inputs<T> in{{x, x + n * N, x + 2 * n * N}, 3};
  const int64_t tiles = (N + kBlock - 1) / kBlock;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)sms * bps);
  V mv{};
  for (int w = 0; w < 3; ++w) kern<<<grid, kBlock>>>(mv, op, N, in, N, true);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = N > 1000000 ? 10 : 200;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) kern<<<grid, kBlock>>>(mv, op, N, in, N, true);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  std::vector<T> h((size_t)N * 63);
  cudaMemcpy(h.data(), y, sizeof(T) * h.size(), cudaMemcpyDeviceToHost);
  double md = 0;
  if (kMB == 3) g_ref.assign(h.begin(), h.end());
  else
    for (size_t k = 0; k < h.size(); ++k) md = std::max(md, std::fabs((double)h[k] - g_ref[k]) / std::max(1.0, std::fabs(g_ref[k])));
  printf("%-10s N %8lld  minB %d regs %3d lmem %4zu b/SM %d grid %u  %.5f ms  %.3e evals/s  maxdiff %.2e  %s\n", name,
         (long long)N, kMB, fa.numRegs, fa.localSizeBytes, bps, grid, ms, N / (ms * 1e-3), md,
         cudaGetErrorString(cudaGetLastError()));
}

// the generated fused routine (GenChain7::Dyn, k_gen_dyn)
template <int kReg, int kSmem, int kMinB, int kTrig, bool kStream, class T = double>
void gen(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch) {
  using Op = GenChain7::Dyn;
  auto kern = k_gen_dyn<Op, T, kReg, kSmem, kMinB, kTrig, kStream>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  if (bps < 1) { printf("%s does not fit\n", name); return; }
  const int64_t grid = std::min<int64_t>((int64_t)sms * bps, (N + kGenBlock - 1) / kGenBlock);
  const int n = 7;
  auto go = [&] {
    kern<<<grid, kGenBlock, smem>>>(N, x, x + n * N, x + 2 * n * N, N, T(0), T(0), T(9.81), y, y + 49 * N, y + 56 * N,
                                    N, st, scratch);
  };
  for (int w = 0; w < 3; ++w) go();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = N > 1000000 ? 10 : 200;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  std::vector<T> h((size_t)N * 63);
  cudaMemcpy(h.data(), y, sizeof(T) * h.size(), cudaMemcpyDeviceToHost);
  double md = 0;
  for (size_t k = 0; k < h.size(); ++k)
    md = std::max(md, std::fabs((double)h[k] - g_ref[k]) / std::max(1.0, std::fabs(g_ref[k])));
  printf("%-26s N %8lld  regs %3d lmem %4zu b/SM %d grid %lld  %.5f ms  %.3e evals/s  maxdiff vs k_tiled %.2e  %s\n",
         name, (long long)N, fa.numRegs, fa.localSizeBytes, bps, (long long)grid, ms, N / (ms * 1e-3), md,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *x, *y;
  int32_t* st;
  const int64_t NM = 4194304;
  cudaMalloc(&x, sizeof(double) * NM * 21);
  cudaMalloc(&y, sizeof(double) * NM * 63);
  cudaMalloc(&st, sizeof(int32_t) * NM);
  double* scratch;
  cudaMalloc(&scratch, 1ull << 30);
  constexpr int S = GenChain7::Dyn::kSlots;
  if (getenv("DYN_F32")) {  // fp32: template kernel vs the generated routine
    float *xf = (float*)x, *yf = (float*)y, *sf = (float*)scratch;
    for (int64_t N : {65536ll, 4194304ll}) {
      k_fill<<<1184, 256>>>(xf, N * 21, 3);
      run<float, 3>("dyn f32", N, xf, yf, st);
      gen<40, S - 40, 3, kTrigFast, false, float>("gen f32 r40 s25 b3 fast", N, xf, yf, st, sf);
      gen<40, S - 40, 4, kTrigFast, false, float>("gen f32 r40 s25 b4 fast", N, xf, yf, st, sf);
      gen<S, 0, 4, kTrigFast, false, float>("gen f32 r65 b4 fast", N, xf, yf, st, sf);
      gen<S, 0, 5, kTrigFast, false, float>("gen f32 r65 b5 fast", N, xf, yf, st, sf);
      gen<24, S - 24, 5, kTrigFast, false, float>("gen f32 r24 s41 b5 fast", N, xf, yf, st, sf);
      gen<24, S - 24, 5, kTrigLib, false, float>("gen f32 r24 s41 b5 lib", N, xf, yf, st, sf);
      gen<0, S, 6, kTrigFast, false, float>("gen f32 s65 b6 fast", N, xf, yf, st, sf);
    }
    return 0;
  }
  for (int64_t N : {65536ll, 262144ll, 4194304ll}) {
    k_fill<<<1184, 256>>>(x, N * 21, 3);
    run<double, 3>("dyn f64", N, x, y, st);
    gen<S, 0, 2, kTrigFast, false>("gen r65 b2 fast", N, x, y, st, scratch);
    gen<S, 0, 3, kTrigFast, false>("gen r65 b3 fast", N, x, y, st, scratch);
    gen<S, 0, 3, kTrigFast, true>("gen r65 b3 fast cs", N, x, y, st, scratch);
    gen<S, 0, 3, kTrigLib, false>("gen r65 b3 lib", N, x, y, st, scratch);
    gen<S, 0, 4, kTrigFast, false>("gen r65 b4 fast", N, x, y, st, scratch);
    gen<40, S - 40, 3, kTrigFast, false>("gen r40 s25 b3 fast", N, x, y, st, scratch);
    gen<24, S - 24, 3, kTrigFast, false>("gen r24 s41 b3 fast", N, x, y, st, scratch);
    gen<24, S - 24, 4, kTrigFast, false>("gen r24 s41 b4 fast", N, x, y, st, scratch);
    gen<0, S, 4, kTrigFast, false>("gen s65 b4 fast", N, x, y, st, scratch);
  }
  return 0;
}
