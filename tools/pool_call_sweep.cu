// A/B for the G1 OSC and JVP routines: persistent loop with the routine inlined
// (k_gen_osc / k_gen_jvp) against the routine called out of line once per
// state (k_gen_osc_call / k_gen_jvp_call).  Built twice, like call_sweep.cu:
// with the product header (fp64 literals) and with a header whose OSC / JVP
// routines read their constants from the robot's __constant__ table:
//   VD_GEN_POOL_OPS="tree29:Aba,AbaFext,Osc,AbaJvp,RneaJvp,CrbaJvp,FkJvp" python -c \
//     'import sys; sys.path[:0] = ["tools", "."]; import gen_tree_kernels as g; \
//      from paper_2604_04310_b200 import _lib; \
//      open("ablib/poolinc/vd_gen_robots.cuh", "w").write(g.generate(_lib.load()))'
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//     -Ipaper_2604_04310_b200/csrc tools/pool_call_sweep.cu -o ablib/pc_lit
//   nvcc ... -Iablib/poolinc -Ipaper_2604_04310_b200/csrc tools/pool_call_sweep.cu -o ablib/pc_pool
// Prints time per launch and a checksum of the outputs (the same arithmetic up
// to constant-operand rounding: checksums agree to ~1e-12 relative).
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

template <class T>
double checksum(const T* d, size_t n) {
  std::vector<T> h(n);
  cudaMemcpy(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost);
  double s = 0;
  for (T v : h) s += std::isfinite((double)v) ? std::fabs((double)v) : 0.0;
  return s;
}

template <class Kern, class Launch>
float time_it(Kern kern, size_t smem, Launch go, int* bps_out, int* regs) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kGenBlock, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  *bps_out = bps;
  *regs = fa.numRegs;
  if (bps < 1) return -1.f;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) go(sms * bps);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) go(sms * bps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig, bool kCall>
void osc(const char* name, int64_t N, T* x, T* y, T* lam, int32_t* st, T* scratch) {
  auto kern = kCall ? k_gen_osc_call<Op, T, kReg, kSmem, kMinB, kTrig> : k_gen_osc<Op, T, kReg, kSmem, kMinB, kTrig>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  OscShared P{};
  for (int k = 0; k < 9; ++k) P.frame_R[k] = P.target_R[k] = (k % 4 == 0) ? 1.0 : 0.0;
  P.target_p[2] = 0.3;
  for (int k = 0; k < 6; ++k) { P.kp[k] = 100; P.kd[k] = 20; }
  P.posture_kp = 10; P.posture_kd = 2; P.gravity[2] = 9.81; P.epsilon = 1e-6;
  const int n = Op::kDof;
  int bps, regs;
  const float ms = time_it(kern, smem, [&](int64_t grid) {
    grid = std::min<int64_t>(grid, (N + kGenBlock - 1) / kGenBlock);
    kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, N, P, y, lam, N, st, scratch);
  }, &bps, &regs);
  printf("%-36s %s regs %3d b/SM %d  %.4f ms  %.3e evals/s  sum %.12e  %s\n", name, kCall ? "call" : "loop", regs, bps,
         ms, N / (ms * 1e-3), checksum(y, (size_t)N * n) + checksum(lam, (size_t)N * 36),
         cudaGetErrorString(cudaGetLastError()));
}

// double-buffered asynchronous input (k_gen_osc_db) against the plain kernel
template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig, bool kDb>
void oscdb(const char* name, int64_t N, T* x, T* y, T* lam, int32_t* st, T* scratch) {
  auto kern = kDb ? k_gen_osc_db<Op, T, kReg, kSmem, kMinB, kTrig> : k_gen_osc<Op, T, kReg, kSmem, kMinB, kTrig>;
  const size_t smem = kDb ? gen_osc_db_smem<Op, T, kSmem>() : (size_t)kSmem * kGenBlock * sizeof(T);
  OscShared P{};
  for (int k = 0; k < 9; ++k) P.frame_R[k] = P.target_R[k] = (k % 4 == 0) ? 1.0 : 0.0;
  P.target_p[2] = 0.3;
  for (int k = 0; k < 6; ++k) { P.kp[k] = 100; P.kd[k] = 20; }
  P.posture_kp = 10; P.posture_kd = 2; P.gravity[2] = 9.81; P.epsilon = 1e-6;
  const int n = Op::kDof;
  int bps, regs;
  const float ms = time_it(kern, smem, [&](int64_t grid) {
    grid = std::min<int64_t>(grid, (N + kGenBlock - 1) / kGenBlock);
    kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, N, P, y, lam, N, st, scratch);
  }, &bps, &regs);
  printf("%-36s %s regs %3d b/SM %d  %.4f ms  %.3e evals/s  sum %.12e  %s\n", name, kDb ? "db  " : "plain", regs, bps,
         ms, N / (ms * 1e-3), checksum(y, (size_t)N * n) + checksum(lam, (size_t)N * 36),
         cudaGetErrorString(cudaGetLastError()));
}

// double-buffered asynchronous input (k_gen_db) against k_gen / k_gen_async
template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig, bool kStream, int kMode>
void gdb(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch) {
  auto kern = kMode == 2 ? k_gen_db<Op, T, kReg, kSmem, kMinB, kTrig, kStream>
              : kMode == 1 ? k_gen_async<Op, T, kReg, kSmem, kMinB, kTrig, kStream>
                           : k_gen<Op, T, kReg, kSmem, kMinB, kTrig, kStream>;
  const size_t smem = kMode == 2 ? gen_db_smem<Op, T, kSmem>()
                      : kMode == 1 ? gen_async_smem<Op, T, kReg, kSmem>() : (size_t)kSmem * kGenBlock * sizeof(T);
  const int n = Op::kDof;
  int bps, regs;
  const float ms = time_it(kern, smem, [&](int64_t grid) {
    grid = std::min<int64_t>(grid, (N + kGenBlock - 1) / kGenBlock);
    kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, x + 2 * N * n, N, T(0), T(0), T(9.81), y, N, st, scratch, nullptr,
                                    nullptr);
  }, &bps, &regs);
  printf("%-36s %s regs %3d b/SM %d  %.4f ms  %.3e evals/s  sum %.12e  %s\n", name,
         kMode == 2 ? "db   " : kMode == 1 ? "async" : "plain", regs, bps, ms, N / (ms * 1e-3),
         checksum(y, (size_t)N * Op::kOut), cudaGetErrorString(cudaGetLastError()));
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig, bool kCall>
void jvp(const char* name, int64_t N, T* x, T* y, T* scratch) {
  auto kern = kCall ? k_gen_jvp_call<Op, T, kReg, kSmem, kMinB, true, kTrig>
                    : k_gen_jvp<Op, T, kReg, kSmem, kMinB, true, kTrig>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  const int n = Op::kDof;
  JvpArgs a{};
  for (int g = 0; g < Op::kIn; ++g) { a.x[g] = x + g * N * n; a.dx[g] = x + (3 + g) * N * n; }
  a.g[2] = 9.81;
  a.out = y;
  a.dout = y + (int64_t)Op::kOut * N;
  int bps, regs;
  const float ms = time_it(kern, smem, [&](int64_t grid) {
    grid = std::min<int64_t>(grid, (N + kGenBlock - 1) / kGenBlock);
    kern<<<grid, kGenBlock, smem>>>(N, a, N, N, scratch);
  }, &bps, &regs);
  printf("%-36s %s regs %3d b/SM %d  %.4f ms  %.3e evals/s  sum %.12e  %s\n", name, kCall ? "call" : "loop", regs, bps,
         ms, N / (ms * 1e-3), checksum(y, (size_t)N * Op::kOut * 2), cudaGetErrorString(cudaGetLastError()));
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig, bool kStream, bool kCall>
void gen(const char* name, int64_t N, T* x, T* y, int32_t* st, T* scratch) {
  auto kern = kCall ? k_gen_call<Op, T, kReg, kSmem, kMinB, kTrig, kStream> : k_gen<Op, T, kReg, kSmem, kMinB, kTrig, kStream>;
  const size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  const int n = Op::kDof;
  int bps, regs;
  const float ms = time_it(kern, smem, [&](int64_t grid) {
    grid = std::min<int64_t>(grid, (N + kGenBlock - 1) / kGenBlock);
    kern<<<grid, kGenBlock, smem>>>(N, x, x + N * n, x + 2 * N * n, N, T(0), T(0), T(9.81), y, N, st, scratch, nullptr,
                                    nullptr);
  }, &bps, &regs);
  printf("%-36s %s regs %3d b/SM %d  %.4f ms  %.3e evals/s  sum %.12e  %s\n", name, kCall ? "call" : "loop", regs, bps,
         ms, N / (ms * 1e-3), checksum(y, (size_t)N * Op::kOut), cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const bool more = argc > 1 && !strcmp(argv[1], "more");
  const int64_t N = 262144;
  const size_t cap = 1ull << 30;
  double *x, *y, *lam, *scratch;
  int32_t* st;
  cudaMalloc(&x, sizeof(double) * 4194304 * 21);  // >= N * 29 * 6; the chain7 sweeps run 4M states
  cudaMalloc(&y, sizeof(double) * N * 841 * 2);
  cudaMalloc(&lam, sizeof(double) * 2097152 * 36);  // sweeps 3 / 9 run chain7 at 1M / 2M states
  cudaMalloc(&scratch, cap);
  cudaMalloc(&st, sizeof(int32_t) * 4194304);  // the chain7 sweeps run up to 4M states
  k_fill<<<1184, 256>>>(x, N * 29 * 6, 7);
  float *xf = (float*)(x), *yf = (float*)y, *lf = (float*)lam, *sf = (float*)scratch;
  using namespace vdk;
  if (argc > 1 && !strcmp(argv[1], "trig")) {  // sweep 4: library sincos vs vd_sincos, both out of line
    gen<GenTree29::Aba, double, 40, 113, 2, kTrigCall, true, true>("t29 aba f64 libcall", N, x, y, st, scratch);
    gen<GenTree29::Aba, double, 40, 113, 2, kTrigFastCall, true, true>("t29 aba f64 fastcall", N, x, y, st, scratch);
    gen<GenTree29::Rnea, double, 58, 55, 2, kTrigCall, false, false>("t29 rnea f64 libcall", N, x, y, st, scratch);
    gen<GenTree29::Rnea, double, 58, 55, 2, kTrigFastCall, false, false>("t29 rnea f64 fastcall", N, x, y, st, scratch);
    gen<GenTree29::RneaBias, double, 0, 72, 3, kTrigCall, false, false>("t29 rneabias f64 libcall", N, x, y, st, scratch);
    gen<GenTree29::RneaBias, double, 0, 72, 3, kTrigFastCall, false, false>("t29 rneabias f64 fastcall", N, x, y, st, scratch);
    gen<GenTree29::Crba, double, 0, 55, 3, kTrigLib, true, false>("t29 crba f64 lib", N, x, y, st, scratch);
    gen<GenTree29::Crba, double, 0, 55, 3, kTrigFastCall, true, false>("t29 crba f64 fastcall", N, x, y, st, scratch);
    gen<GenTree29::Fk, double, 0, 55, 3, kTrigLib, false, false>("t29 fk f64 lib", N, x, y, st, scratch);
    gen<GenTree29::Fk, double, 0, 55, 3, kTrigFastCall, false, false>("t29 fk f64 fastcall", N, x, y, st, scratch);
    osc<GenTree29::Osc23, double, 40, 110, 2, kTrigCall, false>("t29 osc23 f64 libcall", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 40, 110, 2, kTrigFastCall, false>("t29 osc23 f64 fastcall", N, x, y, lam, st, scratch);
    jvp<GenTree29::RneaJvp, double, 40, 110, 2, kTrigCall, true>("t29 rneajvp f64 libcall", N, x, y, scratch);
    jvp<GenTree29::RneaJvp, double, 40, 110, 2, kTrigFastCall, true>("t29 rneajvp f64 fastcall", N, x, y, scratch);
    const int64_t N7 = 1048576;
    gen<GenChain7::Rnea, double, GenChain7::Rnea::kSlots, 0, 4, kTrigFast, false, false>("c7 rnea f64 1M fast", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, GenChain7::Rnea::kSlots, 0, 4, kTrigFastCall, false, false>("c7 rnea f64 1M fastcall", N7, x, y, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    gen<GenTree29::AbaMixed, float, 40, 122, 3, kTrigCall, true, false>("t29 abamixed f32 libcall", N, xf, yf, st, sf);
    gen<GenTree29::AbaMixed, float, 40, 122, 3, kTrigFastCall, true, false>("t29 abamixed f32 fastcall", N, xf, yf, st, sf);
    gen<GenTree29::Rnea, float, 55, 0, 3, kTrigCall, false, false>("t29 rnea f32 libcall", N, xf, yf, st, sf);
    gen<GenTree29::Rnea, float, 55, 0, 3, kTrigFastCall, false, false>("t29 rnea f32 fastcall", N, xf, yf, st, sf);
    osc<GenTree29::Osc23, float, 40, 144, 3, kTrigCall, false>("t29 osc23 f32 libcall", N, xf, yf, lf, st, sf);
    osc<GenTree29::Osc23, float, 40, 144, 3, kTrigFastCall, false>("t29 osc23 f32 fastcall", N, xf, yf, lf, st, sf);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "crbap")) {  // sweep 5: G1 packed CRBA placement / evict-first output
    constexpr int S = GenTree29::CrbaPacked::kSlots;
    gen<GenTree29::CrbaPacked, double, S, 0, 3, kTrigLib, false, false>("t29 crbap f64 r55 b3", N, x, y, st, scratch);
    gen<GenTree29::CrbaPacked, double, S, 0, 3, kTrigLib, true, false>("t29 crbap f64 r55 b3 cs", N, x, y, st, scratch);
    gen<GenTree29::CrbaPacked, double, S, 0, 4, kTrigLib, true, false>("t29 crbap f64 r55 b4 cs", N, x, y, st, scratch);
    gen<GenTree29::CrbaPacked, double, 0, S, 4, kTrigLib, true, false>("t29 crbap f64 s55 b4 cs", N, x, y, st, scratch);
    gen<GenTree29::CrbaPacked, double, 0, S, 5, kTrigLib, true, false>("t29 crbap f64 s55 b5 cs", N, x, y, st, scratch);
    gen<GenTree29::CrbaPacked, double, S, 0, 3, kTrigCall, true, false>("t29 crbap f64 r55 b3 cs trig", N, x, y, st, scratch);
    gen<GenTree29::Crba, double, 0, 55, 3, kTrigLib, true, false>("t29 crba f64 s55 b3 cs", N, x, y, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    gen<GenTree29::CrbaPacked, float, 0, S, 6, kTrigLib, false, false>("t29 crbap f32 s55 b6", N, xf, yf, st, sf);
    gen<GenTree29::CrbaPacked, float, 0, S, 6, kTrigLib, true, false>("t29 crbap f32 s55 b6 cs", N, xf, yf, st, sf);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "fk")) {  // sweep 6: out-of-line sin/cos / evict-first for FK, gravity, CRBA
    gen<GenTree29::Fk, double, 0, 55, 3, kTrigLib, false, false>("t29 fk f64 lib", N, x, y, st, scratch);
    gen<GenTree29::Fk, double, 0, 55, 3, kTrigCall, false, false>("t29 fk f64 trig", N, x, y, st, scratch);
    gen<GenTree29::Fk, double, 0, 55, 3, kTrigLib, true, false>("t29 fk f64 lib cs", N, x, y, st, scratch);
    gen<GenTree29::Fk, double, 0, 55, 3, kTrigCall, true, false>("t29 fk f64 trig cs", N, x, y, st, scratch);
    gen<GenTree29::RneaGrav, double, 0, 55, 3, kTrigLib, false, false>("t29 grav f64 lib", N, x, y, st, scratch);
    gen<GenTree29::RneaGrav, double, 0, 55, 3, kTrigCall, false, false>("t29 grav f64 trig", N, x, y, st, scratch);
    gen<GenTree29::Crba, double, 0, 55, 3, kTrigLib, true, false>("t29 crba f64 lib cs", N, x, y, st, scratch);
    gen<GenTree29::Crba, double, 0, 55, 3, kTrigCall, true, false>("t29 crba f64 trig cs", N, x, y, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    constexpr int S = GenTree29::CrbaPacked::kSlots;
    gen<GenTree29::CrbaPacked, float, 0, S, 6, kTrigLib, false, false>("t29 crbap f32 lib", N, xf, yf, st, sf);
    gen<GenTree29::CrbaPacked, float, 0, S, 6, kTrigCall, false, false>("t29 crbap f32 trig", N, xf, yf, st, sf);
    gen<GenTree29::Fk, float, 0, 55, 4, kTrigLib, false, false>("t29 fk f32 lib", N, xf, yf, st, sf);
    gen<GenTree29::Fk, float, 0, 55, 4, kTrigCall, false, false>("t29 fk f32 trig", N, xf, yf, st, sf);
    gen<GenTree29::Crba, float, 0, 55, 4, kTrigLib, true, false>("t29 crba f32 lib cs", N, xf, yf, st, sf);
    gen<GenTree29::Crba, float, 0, 55, 4, kTrigCall, true, false>("t29 crba f32 trig cs", N, xf, yf, st, sf);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "c7rnea")) {  // sweep 7: Panda RNEA placement / evict-first, 1M states
    const int64_t N7 = 1048576;
    constexpr int S = GenChain7::Rnea::kSlots;
    gen<GenChain7::Rnea, double, S, 0, 4, kTrigFast, false, false>("c7 rnea f64 r b4", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, S, 0, 4, kTrigFast, true, false>("c7 rnea f64 r b4 cs", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, S, 0, 3, kTrigFast, true, false>("c7 rnea f64 r b3 cs", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, 0, S, 5, kTrigFast, true, false>("c7 rnea f64 s b5 cs", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, 0, S, 6, kTrigFast, true, false>("c7 rnea f64 s b6 cs", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, S, 0, 4, kTrigLib, true, false>("c7 rnea f64 r b4 cs lib", N7, x, y, st, scratch);
    gen<GenChain7::RneaBias, double, GenChain7::RneaBias::kSlots, 0, 4, kTrigFast, false, false>("c7 bias f64 r b4", N7, x, y, st, scratch);
    gen<GenChain7::RneaBias, double, GenChain7::RneaBias::kSlots, 0, 4, kTrigFast, true, false>("c7 bias f64 r b4 cs", N7, x, y, st, scratch);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "gdb")) {  // sweep 11: double-buffered input, Panda RNEA / ABA at 2M
    const int64_t N7 = 2097152;
    constexpr int SR = GenChain7::Rnea::kSlots;
    gdb<GenChain7::Rnea, double, SR, 0, 4, kTrigFast, false, 0>("c7 rnea f64 b4", N7, x, y, st, scratch);
    gdb<GenChain7::Rnea, double, SR, 0, 4, kTrigFast, false, 2>("c7 rnea f64 b4", N7, x, y, st, scratch);
    gdb<GenChain7::Rnea, double, SR, 0, 4, kTrigFast, true, 2>("c7 rnea f64 b4 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Rnea, double, SR, 0, 3, kTrigFast, false, 2>("c7 rnea f64 b3", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 24, 41, 3, kTrigFast, true, 1>("c7 aba f64 r24 s41 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 24, 41, 3, kTrigFast, true, 2>("c7 aba f64 r24 s41 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 44, 21, 3, kTrigFast, true, 2>("c7 aba f64 r44 s21 b3 cs", N7, x, y, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    constexpr int SRf = GenChain7::Rnea::kSlots;
    gdb<GenChain7::Rnea, float, SRf, 0, 6, kTrigLib, false, 0>("c7 rnea f32 b6", N7, xf, yf, st, sf);
    gdb<GenChain7::Rnea, float, SRf, 0, 6, kTrigLib, false, 2>("c7 rnea f32 b6", N7, xf, yf, st, sf);
    gdb<GenChain7::Aba, float, 30, 35, 5, kTrigFast, false, 1>("c7 aba f32 r30 s35 b5", N7, xf, yf, st, sf);
    gdb<GenChain7::Aba, float, 30, 35, 5, kTrigFast, false, 2>("c7 aba f32 r30 s35 b5", N7, xf, yf, st, sf);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "gdb4")) {  // sweep 12: double-buffered input at 4M states (headline size)
    const int64_t N7 = 4194304;
    k_fill<<<1184, 256>>>(x, N7 * 21, 9);
    constexpr int SA = GenChain7::Aba::kSlots, SR = GenChain7::Rnea::kSlots;
    gdb<GenChain7::Aba, double, 24, 41, 3, kTrigFast, true, 1>("c7 aba f64 r24 s41 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 44, SA - 44, 3, kTrigFast, true, 2>("c7 aba f64 r44 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 44, SA - 44, 3, kTrigFast, false, 2>("c7 aba f64 r44 b3", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 34, SA - 34, 3, kTrigFast, true, 2>("c7 aba f64 r34 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 54, SA - 54, 3, kTrigFast, true, 2>("c7 aba f64 r54 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, SA, 0, 3, kTrigFast, true, 2>("c7 aba f64 rall b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 24, 41, 3, kTrigFast, true, 1>("c7 aba f64 r24 s41 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Rnea, double, SR, 0, 4, kTrigFast, false, 0>("c7 rnea f64 b4", N7, x, y, st, scratch);
    gdb<GenChain7::Rnea, double, SR, 0, 4, kTrigFast, false, 2>("c7 rnea f64 b4", N7, x, y, st, scratch);
    float* xf4 = (float*)x;
    k_fill<<<1184, 256>>>(xf4, N7 * 21, 9);
    gdb<GenChain7::Aba, float, 30, 35, 5, kTrigFast, false, 1>("c7 aba f32 r30 s35 b5", N7, xf4, yf, st, sf);
    gdb<GenChain7::Aba, float, 30, 35, 5, kTrigFast, false, 2>("c7 aba f32 r30 s35 b5", N7, xf4, yf, st, sf);
    gdb<GenChain7::Aba, float, 40, 25, 5, kTrigFast, false, 2>("c7 aba f32 r40 s25 b5", N7, xf4, yf, st, sf);
    gdb<GenChain7::Aba, float, 30, 35, 6, kTrigFast, false, 2>("c7 aba f32 r30 s35 b6", N7, xf4, yf, st, sf);
    gdb<GenChain7::Rnea, float, SR, 0, 6, kTrigLib, false, 0>("c7 rnea f32 b6", N7, xf4, yf, st, sf);
    gdb<GenChain7::Rnea, float, SR, 0, 6, kTrigLib, false, 2>("c7 rnea f32 b6", N7, xf4, yf, st, sf);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "gdb6")) {  // sweep 14: headline ABA fp64 db placements around r44 s21
    const int64_t N7 = 4194304;
    k_fill<<<1184, 256>>>(x, N7 * 21, 9);
    constexpr int SA = GenChain7::Aba::kSlots;
    gdb<GenChain7::Aba, double, 44, SA - 44, 3, kTrigFast, true, 2>("c7 aba f64 r44 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 40, SA - 40, 3, kTrigFast, true, 2>("c7 aba f64 r40 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 48, SA - 48, 3, kTrigFast, true, 2>("c7 aba f64 r48 b3 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 44, SA - 44, 3, kTrigLib, true, 2>("c7 aba f64 r44 b3 cs lib", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 44, SA - 44, 2, kTrigFast, true, 2>("c7 aba f64 r44 b2 cs", N7, x, y, st, scratch);
    gdb<GenChain7::Aba, double, 44, SA - 44, 3, kTrigFast, true, 2>("c7 aba f64 r44 b3 cs", N7, x, y, st, scratch);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "gdb5")) {  // sweep 13: double-buffered input for further routines
    const int64_t N7 = 4194304;
    k_fill<<<1184, 256>>>(x, N7 * 21, 9);
    constexpr int SP = GenChain7::CrbaPacked::kSlots, SG = GenChain7::RneaGrav::kSlots;
    gdb<GenChain7::CrbaPacked, double, SP, 0, 4, kTrigLib, false, 0>("c7 crbap f64 b4", N7, x, y, st, scratch);
    gdb<GenChain7::CrbaPacked, double, SP, 0, 4, kTrigLib, false, 2>("c7 crbap f64 b4", N7, x, y, st, scratch);
    gdb<GenChain7::CrbaPacked, double, SP, 0, 4, kTrigLib, true, 2>("c7 crbap f64 b4 cs", N7, x, y, st, scratch);
    gdb<GenChain7::RneaGrav, double, SG, 0, 4, kTrigFast, false, 0>("c7 grav f64 b4", N7, x, y, st, scratch);
    gdb<GenChain7::RneaGrav, double, SG, 0, 4, kTrigFast, false, 2>("c7 grav f64 b4", N7, x, y, st, scratch);
    k_fill<<<1184, 256>>>(x, N * 29 * 6, 7);
    gdb<GenTree29::Rnea, float, 55, 0, 3, kTrigCall, false, 0>("t29 rnea f32 r55 b3", N, xf, yf, st, sf);
    gdb<GenTree29::Rnea, float, 55, 0, 2, kTrigCall, false, 2>("t29 rnea f32 r55 b2", N, xf, yf, st, sf);
    gdb<GenTree29::RneaBias, double, 0, 72, 3, kTrigCall, false, 0>("t29 bias f64 s72 b3", N, x, y, st, scratch);
    gdb<GenTree29::RneaBias, double, 0, 40, 3, kTrigCall, false, 2>("t29 bias f64 s40 b3", N, x, y, st, scratch);
    gdb<GenTree29::Crba, double, 0, 55, 3, kTrigLib, true, 0>("t29 crba f64 s55 b3 cs", N, x, y, st, scratch);
    gdb<GenTree29::Crba, double, 0, 55, 3, kTrigLib, true, 2>("t29 crba f64 s55 b3 cs", N, x, y, st, scratch);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "g1osc")) {  // sweep 10: G1 OSC placements with the out-of-line sin/cos
    osc<GenTree29::Osc23, double, 40, 110, 2, kTrigCall, false>("t29 osc23 f64 r40 s110 b2", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 24, 110, 2, kTrigCall, false>("t29 osc23 f64 r24 s110 b2", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 56, 110, 2, kTrigCall, false>("t29 osc23 f64 r56 s110 b2", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 40, 100, 2, kTrigCall, false>("t29 osc23 f64 r40 s100 b2", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 0, 72, 3, kTrigCall, false>("t29 osc23 f64 r0 s72 b3", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 24, 72, 3, kTrigCall, false>("t29 osc23 f64 r24 s72 b3", N, x, y, lam, st, scratch);
    osc<GenTree29::Osc23, double, 40, 214, 1, kTrigCall, false>("t29 osc23 f64 r40 s214 b1", N, x, y, lam, st, scratch);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "oscdb")) {  // sweep 9: Panda OSC, double-buffered asynchronous input
    const int64_t N7 = 2097152;
    oscdb<GenChain7::Osc6, double, 80, 67, 2, kTrigLib, false>("c7 osc6 f64 r80 s67 b2", N7, x, y, lam, st, scratch);
    oscdb<GenChain7::Osc6, double, 80, 67, 2, kTrigLib, true>("c7 osc6 f64 r80 s67 b2", N7, x, y, lam, st, scratch);
    oscdb<GenChain7::Osc6, double, 80, 67, 2, kTrigFast, true>("c7 osc6 f64 r80 s67 b2 fast", N7, x, y, lam, st, scratch);
    oscdb<GenChain7::Osc6, double, 60, 87, 2, kTrigLib, true>("c7 osc6 f64 r60 s87 b2", N7, x, y, lam, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    oscdb<GenChain7::Osc6, float, 60, 87, 2, kTrigLib, false>("c7 osc6 f32 r60 s87 b2", N7, xf, yf, lf, st, sf);
    oscdb<GenChain7::Osc6, float, 60, 87, 2, kTrigLib, true>("c7 osc6 f32 r60 s87 b2", N7, xf, yf, lf, st, sf);
    oscdb<GenChain7::Osc6, float, 60, 87, 3, kTrigLib, true>("c7 osc6 f32 r60 s87 b3", N7, xf, yf, lf, st, sf);
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "c7ck")) {  // sweep 8: generated Panda CRBA / FK at 4M (template: 0.355 / 0.579 ms)
    const int64_t N7 = 4194304;
    constexpr int SC = GenChain7::Crba::kSlots, SF = GenChain7::Fk::kSlots;
    gen<GenChain7::Crba, double, SC, 0, 3, kTrigFast, false, false>("c7 crba f64 r b3", N7, x, y, st, scratch);
    gen<GenChain7::Crba, double, SC, 0, 3, kTrigFast, true, false>("c7 crba f64 r b3 cs", N7, x, y, st, scratch);
    gen<GenChain7::Crba, double, SC, 0, 4, kTrigFast, true, false>("c7 crba f64 r b4 cs", N7, x, y, st, scratch);
    gen<GenChain7::Crba, double, 0, SC, 4, kTrigFast, true, false>("c7 crba f64 s b4 cs", N7, x, y, st, scratch);
    gen<GenChain7::Crba, double, SC, 0, 4, kTrigLib, true, false>("c7 crba f64 r b4 cs lib", N7, x, y, st, scratch);
    gen<GenChain7::Fk, double, SF, 0, 3, kTrigFast, false, false>("c7 fk f64 r b3", N7, x, y, st, scratch);
    gen<GenChain7::Fk, double, SF, 0, 3, kTrigFast, true, false>("c7 fk f64 r b3 cs", N7, x, y, st, scratch);
    gen<GenChain7::Fk, double, SF, 0, 4, kTrigFast, true, false>("c7 fk f64 r b4 cs", N7, x, y, st, scratch);
    gen<GenChain7::Fk, double, SF, 0, 4, kTrigLib, true, false>("c7 fk f64 r b4 cs lib", N7, x, y, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    gen<GenChain7::Crba, float, SC, 0, 4, kTrigLib, true, false>("c7 crba f32 r b4 cs lib", N7, xf, yf, st, sf);
    gen<GenChain7::Crba, float, SC, 0, 6, kTrigLib, true, false>("c7 crba f32 r b6 cs lib", N7, xf, yf, st, sf);
    gen<GenChain7::Fk, float, SF, 0, 4, kTrigLib, true, false>("c7 fk f32 r b4 cs lib", N7, xf, yf, st, sf);
    gen<GenChain7::Fk, float, SF, 0, 6, kTrigLib, true, false>("c7 fk f32 r b6 cs lib", N7, xf, yf, st, sf);
    return 0;
  }
  if (more) {  // sweep 3: the remaining generated routines, loop vs per-state call
    const int64_t N7 = 1048576;
    gen<GenTree29::RneaBias, double, 0, 72, 3, kTrigCall, false, false>("t29 rneabias f64", N, x, y, st, scratch);
    gen<GenTree29::RneaBias, double, 0, 72, 3, kTrigCall, false, true>("t29 rneabias f64", N, x, y, st, scratch);
    gen<GenTree29::RneaGrav, double, 0, 55, 3, kTrigCall, false, false>("t29 rneagrav f64", N, x, y, st, scratch);
    gen<GenTree29::RneaGrav, double, 0, 55, 3, kTrigCall, false, true>("t29 rneagrav f64", N, x, y, st, scratch);
    gen<GenTree29::Rnea, double, 58, 55, 2, kTrigCall, false, false>("t29 rnea f64", N, x, y, st, scratch);
    gen<GenTree29::Rnea, double, 58, 55, 2, kTrigCall, false, true>("t29 rnea f64", N, x, y, st, scratch);
    gen<GenChain7::Rnea, double, GenChain7::Rnea::kSlots, 0, 4, kTrigFast, false, false>("c7 rnea f64 1M", N7, x, y, st, scratch);
    gen<GenChain7::Rnea, double, GenChain7::Rnea::kSlots, 0, 4, kTrigFast, false, true>("c7 rnea f64 1M", N7, x, y, st, scratch);
    jvp<GenChain7::AbaJvp, double, 40, 89, 2, kTrigLib, false>("c7 abajvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::AbaJvp, double, 40, 89, 2, kTrigLib, true>("c7 abajvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::RneaJvp, double, 40, 16, 2, kTrigLib, false>("c7 rneajvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::RneaJvp, double, 40, 16, 2, kTrigLib, true>("c7 rneajvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::CrbaJvp, double, 28, 0, 2, kTrigLib, false>("c7 crbajvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::CrbaJvp, double, 28, 0, 2, kTrigLib, true>("c7 crbajvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::FkJvp, double, 28, 0, 2, kTrigLib, false>("c7 fkjvp f64 1M", N7, x, y, scratch);
    jvp<GenChain7::FkJvp, double, 28, 0, 2, kTrigLib, true>("c7 fkjvp f64 1M", N7, x, y, scratch);
    osc<GenChain7::Osc6, double, 80, 67, 2, kTrigLib, false>("c7 osc6 f64 1M", N7, x, y, lam, st, scratch);
    osc<GenChain7::Osc6, double, 80, 67, 2, kTrigLib, true>("c7 osc6 f64 1M", N7, x, y, lam, st, scratch);
    k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
    jvp<GenChain7::AbaJvp, float, 0, 129, 2, kTrigLib, false>("c7 abajvp f32 1M", N7, xf, yf, sf);
    jvp<GenChain7::AbaJvp, float, 0, 129, 2, kTrigLib, true>("c7 abajvp f32 1M", N7, xf, yf, sf);
    gen<GenTree29::Rnea, float, 55, 0, 3, kTrigCall, false, false>("t29 rnea f32", N, xf, yf, st, sf);
    gen<GenTree29::Rnea, float, 55, 0, 3, kTrigCall, false, true>("t29 rnea f32", N, xf, yf, st, sf);
    osc<GenChain7::Osc6, float, 60, 87, 2, kTrigLib, false>("c7 osc6 f32 1M", N7, xf, yf, lf, st, sf);
    osc<GenChain7::Osc6, float, 60, 87, 2, kTrigLib, true>("c7 osc6 f32 1M", N7, xf, yf, lf, st, sf);
    return 0;
  }
  // product placements (OscCfg default; JvpCfg); sweep 2: every G1 OSC frame
  // joint and the trig mode, the remaining JVPs
#define OSC4(J)                                                                                              \
  osc<GenTree29::Osc##J, double, 40, 110, 2, kTrigLib, false>("t29 osc" #J " f64 lib", N, x, y, lam, st, scratch);  \
  osc<GenTree29::Osc##J, double, 40, 110, 2, kTrigCall, false>("t29 osc" #J " f64 trig", N, x, y, lam, st, scratch); \
  osc<GenTree29::Osc##J, double, 40, 110, 2, kTrigLib, true>("t29 osc" #J " f64 lib", N, x, y, lam, st, scratch);   \
  osc<GenTree29::Osc##J, double, 40, 110, 2, kTrigCall, true>("t29 osc" #J " f64 trig", N, x, y, lam, st, scratch);
  OSC4(11) OSC4(17) OSC4(18) OSC4(23) OSC4(28)
  k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
  osc<GenTree29::Osc23, float, 40, 144, 3, kTrigCall, false>("t29 osc23 f32 trig", N, xf, yf, lf, st, sf);
  osc<GenTree29::Osc17, float, 40, 144, 3, kTrigCall, false>("t29 osc17 f32 trig", N, xf, yf, lf, st, sf);
  k_fill<<<1184, 256>>>(x, N * 29 * 6, 7);
  jvp<GenTree29::RneaJvp, double, 40, 110, 2, kTrigLib, false>("t29 rneajvp f64 lib", N, x, y, scratch);
  jvp<GenTree29::RneaJvp, double, 40, 110, 2, kTrigLib, true>("t29 rneajvp f64 lib", N, x, y, scratch);
  jvp<GenTree29::RneaJvp, double, 40, 110, 2, kTrigCall, true>("t29 rneajvp f64 trig", N, x, y, scratch);
  jvp<GenTree29::RneaJvp, double, 40, 110, 3, kTrigLib, true>("t29 rneajvp f64 lib b3", N, x, y, scratch);
  jvp<GenTree29::RneaJvp, double, 0, 144, 3, kTrigLib, true>("t29 rneajvp f64 lib r0 s144 b3", N, x, y, scratch);
  jvp<GenTree29::CrbaJvp, double, 40, 70, 2, kTrigLib, false>("t29 crbajvp f64 lib", N, x, y, scratch);
  jvp<GenTree29::CrbaJvp, double, 40, 70, 2, kTrigLib, true>("t29 crbajvp f64 lib", N, x, y, scratch);
  jvp<GenTree29::CrbaJvp, double, 40, 70, 2, kTrigCall, true>("t29 crbajvp f64 trig", N, x, y, scratch);
  jvp<GenTree29::FkJvp, double, 40, 70, 2, kTrigLib, false>("t29 fkjvp f64 lib", N, x, y, scratch);
  jvp<GenTree29::FkJvp, double, 40, 70, 2, kTrigLib, true>("t29 fkjvp f64 lib", N, x, y, scratch);
  jvp<GenTree29::AbaJvp, double, 40, 220, 1, kTrigCall, false>("t29 abajvp f64 trig", N, x, y, scratch);
  jvp<GenTree29::AbaJvp, double, 40, 220, 1, kTrigCall, true>("t29 abajvp f64 trig", N, x, y, scratch);
  k_fill<<<1184, 256>>>(xf, N * 29 * 6, 7);
  jvp<GenTree29::RneaJvp, float, 0, 144, 3, kTrigCall, false>("t29 rneajvp f32 trig", N, xf, yf, sf);
  jvp<GenTree29::RneaJvp, float, 0, 144, 3, kTrigCall, true>("t29 rneajvp f32 trig", N, xf, yf, sf);
  jvp<GenTree29::CrbaJvp, float, 0, 110, 3, kTrigLib, false>("t29 crbajvp f32 lib", N, xf, yf, sf);
  jvp<GenTree29::CrbaJvp, float, 0, 110, 3, kTrigLib, true>("t29 crbajvp f32 lib", N, xf, yf, sf);
  jvp<GenTree29::FkJvp, float, 0, 110, 3, kTrigLib, false>("t29 fkjvp f32 lib", N, xf, yf, sf);
  jvp<GenTree29::FkJvp, float, 0, 110, 3, kTrigLib, true>("t29 fkjvp f32 lib", N, xf, yf, sf);
  return 0;
}
