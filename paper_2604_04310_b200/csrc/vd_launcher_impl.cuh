// Out-of-line Launcher<V> members: included only by the vd_inst_*.cu
// instantiation units so vd_dispatch.cu never re-instantiates the kernels.
#pragma once

#include <algorithm>
#include <mutex>

#include "vd_kernels.cuh"

namespace vdk {

// Persistent-grid size of one kernel, cached per device.  host_batch drives
// several devices from concurrent threads, so the cache is mutex-protected
// and keyed by the calling thread's current device.
struct TiledOcc {
  int blocks_per_sm = 0, sms = 0;
};

template <class K>
TiledOcc tiled_occupancy(K kern) {
  static std::mutex mu;
  static TiledOcc occ[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  TiledOcc& c = occ[dev & 63];
  if (!c.blocks_per_sm) {
    int sms = 0, bps = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kBlock, 0);
    c.sms = sms;
    c.blocks_per_sm = bps < 1 ? 1 : bps;
  }
  return c;
}

// Launch the staged persistent kernel when the view is compile-time and the
// two shared-memory stages fit the 48 KB static limit; returns -1 when not
// eligible (caller uses the plain kernel).
template <class V, class Op>
int try_tiled(const V& mv, const Launch& L, const Op& op, const void* a, const void* b, const void* c) {
  using T = typename V::Real;
  if constexpr (!V::kStatic || !Op::kEnabled) {
    return -1;
  } else {
    constexpr size_t smem = 2ull * Op::kGroups * V::kMax * kBlock * sizeof(T);
    if constexpr (smem > 48 * 1024) {
      return -1;
    } else {
      // Compile-time views always run this kernel (one instruction stream for
      // every instance, whatever N, ld or alignment); TMA is used when every
      // input plane is 16-byte aligned, otherwise tiles are staged by plain loads.
      const void* ptrs[3] = {a, b, c};
      bool aligned = (L.ld_in * (int64_t)sizeof(T)) % 16 == 0;
      for (int g = 0; g < Op::kGroups; ++g) aligned = aligned && ptrs[g] && ((uintptr_t)ptrs[g] % 16 == 0);
      const TiledOcc o = tiled_occupancy(k_tiled<V, Op>);
      const int64_t tiles = (L.N + kBlock - 1) / kBlock;
      const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)o.sms * o.blocks_per_sm);
      tma::Inputs<T> in{{(const T*)a, (const T*)b, (const T*)c}, Op::kGroups};
      k_tiled<V, Op><<<grid, kBlock, 0, stream_of(L)>>>(mv, op, L.N, in, L.ld_in, aligned);
      return (int)cudaGetLastError();
    }
  }
}

template <class V>
int Launcher<V>::fk(const V& mv, const Launch& L, const void* q, void* out) {
  using T = typename V::Real;
  const int rc = try_tiled(mv, L, OpFK<T>{(T*)out, L.ld_out}, q, nullptr, nullptr);
  if (rc >= 0) return rc;
  k_fk<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, L.ld_in, (T*)out, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::jac(const V& mv, const Launch& L, const void* q, const FrameArg& fr, void* pose, void* J) {
  using T = typename V::Real;
  const int rc = try_tiled(mv, L, OpJac<T>{fr, (T*)pose, (T*)J, L.ld_out}, q, nullptr, nullptr);
  if (rc >= 0) return rc;
  k_jac<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, L.ld_in, fr, (T*)pose, (T*)J, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::rnea(const V& mv, const Launch& L, const void* q, const void* qd, const void* qdd, const double* g,
                      const void* fext, void* tau) {
  using T = typename V::Real;
  const T* gpl = static_cast<const T*>(L.gravity_planes);
  if (!fext && !gpl) {
    int rc;
    if (qdd) rc = try_tiled(mv, L, OpRNEA<T, 3>{g3_of<T>(g), (T*)tau, L.ld_out}, q, qd, qdd);
    else if (qd) rc = try_tiled(mv, L, OpRNEA<T, 2>{g3_of<T>(g), (T*)tau, L.ld_out}, q, qd, nullptr);
    else rc = try_tiled(mv, L, OpRNEA<T, 1>{g3_of<T>(g), (T*)tau, L.ld_out}, q, nullptr, nullptr);
    if (rc >= 0) return rc;
  }
  if (fext)
    k_rnea<V, true><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, (const T*)qd, (const T*)qdd,
                                                                L.ld_in, g3_of<T>(g), (const T*)fext, (T*)tau, L.ld_out,
                                                                gpl);
  else
    k_rnea<V, false><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, (const T*)qd, (const T*)qdd,
                                                                 L.ld_in, g3_of<T>(g), nullptr, (T*)tau, L.ld_out, gpl);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::crba(const V& mv, const Launch& L, const void* q, void* M) {
  using T = typename V::Real;
  const int rc = try_tiled(mv, L, OpCRBA<T>{(T*)M, L.ld_out}, q, nullptr, nullptr);
  if (rc >= 0) return rc;
  k_crba<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, L.ld_in, (T*)M, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::aba(const V& mv, const Launch& L, const void* q, const void* qd, const void* tau, const double* g,
                     const void* fext, void* qdd, int32_t* status) {
  using T = typename V::Real;
  const T* gpl = static_cast<const T*>(L.gravity_planes);
  if (!fext && !gpl) {
    const int rc = try_tiled(mv, L, OpABA<T>{g3_of<T>(g), (T*)qdd, L.ld_out, status}, q, qd, tau);
    if (rc >= 0) return rc;
  }
  if (fext)
    k_aba<V, true><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, (const T*)qd, (const T*)tau,
                                                               L.ld_in, g3_of<T>(g), (const T*)fext, (T*)qdd, L.ld_out,
                                                               status, gpl);
  else
    k_aba<V, false><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, (const T*)qd, (const T*)tau,
                                                                L.ld_in, g3_of<T>(g), nullptr, (T*)qdd, L.ld_out,
                                                                status, gpl);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::dyn(const V& mv, const Launch& L, const void* q, const void* qd, const void* tau, const double* g,
                     void* M, void* bias, void* qdd, int32_t* status) {
  using T = typename V::Real;
  const int rc = try_tiled(mv, L, OpDyn<T>{g3_of<T>(g), (T*)M, (T*)bias, (T*)qdd, L.ld_out, status}, q, qd,
                           tau ? tau : qd);
  if (rc >= 0) return rc;
  k_dyn<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, (const T*)qd, (const T*)tau, L.ld_in,
                                                        g3_of<T>(g), (T*)M, (T*)bias, (T*)qdd, L.ld_out, status);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::osc(const V& mv, const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau,
                     void* lambda, int32_t* status) {
  using T = typename V::Real;
  const int rc = try_tiled(mv, L, OpOSC<T>{P, (T*)tau, (T*)lambda, L.ld_out, status}, q, qd, nullptr);
  if (rc >= 0) return rc;
  k_osc<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, (const T*)qd, L.ld_in, P, (T*)tau,
                                                        (T*)lambda, L.ld_out, status);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::task(const V& mv, const Launch& L, const void* q, const TaskShared& P, int mode, void* out, void* aux,
                      int32_t* status) {
  using T = typename V::Real;
  k_task<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const T*)q, L.ld_in, P, mode, (T*)out, (T*)aux,
                                                         L.ld_out, status);
  return (int)cudaGetLastError();
}

}  // namespace vdk
