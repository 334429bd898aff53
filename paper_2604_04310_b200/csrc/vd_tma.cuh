// TMA-staged, persistent tile pipeline for the compile-time (static view)
// kernels.
//
// Each CTA owns tiles of kBlock consecutive instances.  For every input plane
// of a tile (kBlock contiguous values of the SoA layout) one thread issues a
// 1-D bulk tensor copy (cp.async.bulk, the TMA engine) into a shared-memory
// stage, completing on an mbarrier with a transaction count.  Two stages: the
// copies for tile t+2·grid are in flight while tile t is computed, so the
// global-load latency that otherwise stalls the head of every recursion (the
// q -> sincos dependency) is hidden without spending registers on prefetch.
#pragma once

#include <cstdint>

namespace vdk {
namespace tma {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// Input groups of a tile: up to 3 tensors (q, q̇, τ|q̈) of n planes each.
template <class T>
struct Inputs {
  const T* p[3];
  int count;  // number of tensors
};

// Issue the bulk copies of tile `t` (planes of every input tensor) into `buf`.
template <class T, int kTile>
__device__ __forceinline__ void issue_tile(T* buf, const Inputs<T>& in, int n, int64_t ld, int64_t t, uint64_t* bar) {
  constexpr uint32_t bytes = kTile * sizeof(T);
  mbar_expect_tx(bar, bytes * (uint32_t)(n * in.count));
  for (int g = 0; g < in.count; ++g)
    for (int k = 0; k < n; ++k)
      bulk_g2s(buf + (g * n + k) * kTile, in.p[g] + (int64_t)k * ld + t * kTile, bytes, bar);
}

}  // namespace tma

// Shared-memory row accessor: element k of tensor g for this thread.
template <class T, int kTile>
struct SmemRow {
  const T* base;  // buf + g*n*kTile + tid
  __device__ __forceinline__ T operator[](int k) const { return base[k * kTile]; }
};

}  // namespace vdk
