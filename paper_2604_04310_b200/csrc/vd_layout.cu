// Layout conversion between a row-major (N, K) batch ("array of structs":
// element (i, k) at i*ld_rows + k, how a torch (N, n) tensor or a C array of
// per-state records sits in memory) and the planes the kernels read and
// write (element (i, k) at k*ld_planes + i, the column-major StateBatch
// layout of batch.hpp:15-19).  A CTA stages a block of rows through shared
// memory so both sides are coalesced (a strided gather/scatter through the
// L1 reaches ~0.4-1.8 TB/s on B200 for these narrow shapes).
#include <algorithm>
#include <cstdint>

#include "vd_launch.hpp"

namespace vdk {
namespace {

constexpr int kLayoutThreads = 256;
constexpr int kLayoutSmem = 46 * 1024;
constexpr int kChunk = 32;  // columns per tile for wide rows (K > 64)

// Narrow rows (K <= 64): the tile holds B whole rows exactly as they sit in a
// dense row-major buffer (row r at tile[r*K]), so the row side is one flat
// contiguous run with no index arithmetic; the plane side walks k outer, row
// inner.  Global -> shared loops are unrolled so several loads are in flight
// before their shared-memory stores.
template <class T, bool kToPlanes>
__global__ void __launch_bounds__(kLayoutThreads) k_layout(int64_t N, int K, int B, const T* __restrict__ src,
                                                           int64_t ld_src, T* __restrict__ dst, int64_t ld_dst) {
  extern __shared__ __align__(16) unsigned char vd_layout_smem[];
  T* tile = reinterpret_cast<T*>(vd_layout_smem);
  const int64_t ld_rows = kToPlanes ? ld_src : ld_dst;
  for (int64_t base = (int64_t)blockIdx.x * B; base < N; base += (int64_t)gridDim.x * B) {
    const int rows = (int)(N - base < B ? N - base : (int64_t)B);
    const int flat = rows * K;
    if constexpr (kToPlanes) {
      if (ld_rows == K) {
        const T* s = src + base * K;
#pragma unroll 8
        for (int e = threadIdx.x; e < flat; e += kLayoutThreads) tile[e] = s[e];
      } else {
        for (int r = 0; r < rows; ++r)
          for (int k = threadIdx.x; k < K; k += kLayoutThreads) tile[r * K + k] = src[(base + r) * ld_rows + k];
      }
      __syncthreads();
      for (int k = 0; k < K; ++k)
        for (int r = threadIdx.x; r < rows; r += kLayoutThreads) dst[(int64_t)k * ld_dst + base + r] = tile[r * K + k];
    } else {
#pragma unroll 8
      for (int k = 0; k < K; ++k)
        for (int r = threadIdx.x; r < rows; r += kLayoutThreads) tile[r * K + k] = src[(int64_t)k * ld_src + base + r];
      __syncthreads();
      if (ld_rows == K) {
        T* d = dst + base * K;
        for (int e = threadIdx.x; e < flat; e += kLayoutThreads) d[e] = tile[e];
      } else {
        for (int r = 0; r < rows; ++r)
          for (int k = threadIdx.x; k < K; k += kLayoutThreads) dst[(base + r) * ld_rows + k] = tile[r * K + k];
      }
    }
    __syncthreads();
  }
}

// Wide rows (K > 64, e.g. 6n external-wrench planes): tiles of 128 rows x 32
// columns (blockIdx.y = column chunk), row segments of 32 elements on one
// side and 128-element plane runs on the other; padded row stride (33)
// keeps the column walk conflict-free.
template <class T, bool kToPlanes>
__global__ void __launch_bounds__(kLayoutThreads) k_layout_wide(int64_t N, int K, const T* __restrict__ src,
                                                                int64_t ld_src, T* __restrict__ dst, int64_t ld_dst) {
  constexpr int B = 128, S = kChunk + 1;
  __shared__ T tile[B * S];
  const int k0 = blockIdx.y * kChunk;
  const int kc = K - k0 < kChunk ? K - k0 : kChunk;
  for (int64_t base = (int64_t)blockIdx.x * B; base < N; base += (int64_t)gridDim.x * B) {
    const int rows = (int)(N - base < B ? N - base : (int64_t)B);
    if constexpr (kToPlanes) {
#pragma unroll 4
      for (int e = threadIdx.x; e < B * kChunk; e += kLayoutThreads) {
        const int r = e >> 5, c = e & (kChunk - 1);
        if (r < rows && c < kc) tile[r * S + c] = src[(base + r) * ld_src + k0 + c];
      }
      __syncthreads();
#pragma unroll 4
      for (int e = threadIdx.x; e < B * kChunk; e += kLayoutThreads) {
        const int c = e >> 7, r = e & (B - 1);
        if (r < rows && c < kc) dst[(int64_t)(k0 + c) * ld_dst + base + r] = tile[r * S + c];
      }
    } else {
#pragma unroll 4
      for (int e = threadIdx.x; e < B * kChunk; e += kLayoutThreads) {
        const int c = e >> 7, r = e & (B - 1);
        if (r < rows && c < kc) tile[r * S + c] = src[(int64_t)(k0 + c) * ld_src + base + r];
      }
      __syncthreads();
#pragma unroll 4
      for (int e = threadIdx.x; e < B * kChunk; e += kLayoutThreads) {
        const int r = e >> 5, c = e & (kChunk - 1);
        if (r < rows && c < kc) dst[(base + r) * ld_dst + k0 + c] = tile[r * S + c];
      }
    }
    __syncthreads();
  }
}

template <class T>
int layout_t(bool to_planes, int64_t N, int K, const void* src, int64_t ld_src, void* dst, int64_t ld_dst,
             void* stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (K > 64) {
    const dim3 grid((unsigned)std::min<int64_t>((N + 127) / 128, (int64_t)sms * 4), (unsigned)((K + kChunk - 1) / kChunk));
    if (to_planes)
      k_layout_wide<T, true><<<grid, kLayoutThreads, 0, s>>>(N, K, (const T*)src, ld_src, (T*)dst, ld_dst);
    else
      k_layout_wide<T, false><<<grid, kLayoutThreads, 0, s>>>(N, K, (const T*)src, ld_src, (T*)dst, ld_dst);
    return (int)cudaGetLastError();
  }
  // rows per CTA: a multiple of 32, at most 256, within the shared-memory budget
  const int B = std::min(256, kLayoutSmem / (K * (int)sizeof(T)) / 32 * 32);
  const size_t smem = (size_t)B * K * sizeof(T);
  const int64_t blocks = std::min<int64_t>((N + B - 1) / B, (int64_t)sms * 8);
  if (to_planes)
    k_layout<T, true><<<(unsigned)blocks, kLayoutThreads, smem, s>>>(N, K, B, (const T*)src, ld_src, (T*)dst, ld_dst);
  else
    k_layout<T, false><<<(unsigned)blocks, kLayoutThreads, smem, s>>>(N, K, B, (const T*)src, ld_src, (T*)dst, ld_dst);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_layout(int dtype, bool to_planes, int64_t N, int K, const void* src, int64_t ld_src, void* dst,
                  int64_t ld_dst, void* stream) {
  if (N == 0 || K == 0) return 0;
  return dtype == 0 ? layout_t<double>(to_planes, N, K, src, ld_src, dst, ld_dst, stream)
                    : layout_t<float>(to_planes, N, K, src, ld_src, dst, ld_dst, stream);
}

}  // namespace vdk
