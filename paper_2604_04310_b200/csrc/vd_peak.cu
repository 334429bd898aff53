// FMA-throughput microbenchmark: the measured FP64 / FP32 non-tensor peak used
// as the roofline denominator (MEASURED_PEAKS.json only carries HBM and bf16).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

template <class T>
__global__ void __launch_bounds__(256) k_fma_peak(T* out, int iters, T a, T b) {
  T x0 = T(threadIdx.x) * T(1e-3), x1 = x0 + T(1), x2 = x0 + T(2), x3 = x0 + T(3);
  T x4 = x0 + T(4), x5 = x0 + T(5), x6 = x0 + T(6), x7 = x0 + T(7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == T(-12345.678)) out[0] = s;  // keep the chains live
}

template <class T>
double run(int device, int ms_target) {
  cudaSetDevice(device);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  T* out = nullptr;
  cudaMalloc(&out, sizeof(T));
  const int blocks = prop.multiProcessorCount * 8;
  const int threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 256;
  k_fma_peak<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));  // warm-up
  cudaDeviceSynchronize();
  float ms = 0;
  for (int rep = 0; rep < 8; ++rep) {
    cudaEventRecord(e0);
    k_fma_peak<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms >= ms_target) break;
    iters *= 2;
  }
  double best = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_fma_peak<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    best = flops / (ms * 1e-3) > best ? flops / (ms * 1e-3) : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best / 1e12 : -1.0;
}

}  // namespace

// TFLOP/s of dependent-chain-free FMA streams on `device` (dtype 0 f64, 1 f32).
extern "C" double vdi_fma_peak_tflops(int device, int dtype, int ms_target) {
  return dtype == 0 ? run<double>(device, ms_target) : run<float>(device, ms_target);
}
