// Out-of-line Launcher<V> members: included only by the vd_inst_*.cu
// instantiation units so vd_dispatch.cu never re-instantiates the kernels.
#pragma once

#include "vd_kernels.cuh"

namespace vdk {

template <class V>
int Launcher<V>::fk(const V& mv, const Launch& L, const void* q, void* out) {
  k_fk<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, L.ld_in, (typename V::Real*)out, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::jac(const V& mv, const Launch& L, const void* q, const FrameArg& fr, void* pose, void* J) {
  k_jac<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, L.ld_in, fr, (typename V::Real*)pose, (typename V::Real*)J, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::rnea(const V& mv, const Launch& L, const void* q, const void* qd, const void* qdd, const double* g,
                  const void* fext, void* tau) {
  if (fext)
    k_rnea<V, true><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, (const typename V::Real*)qd, (const typename V::Real*)qdd,
                                                                L.ld_in, g3_of<typename V::Real>(g), (const typename V::Real*)fext, (typename V::Real*)tau, L.ld_out);
  else
    k_rnea<V, false><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, (const typename V::Real*)qd, (const typename V::Real*)qdd,
                                                                 L.ld_in, g3_of<typename V::Real>(g), nullptr, (typename V::Real*)tau, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::crba(const V& mv, const Launch& L, const void* q, void* M) {
  k_crba<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, L.ld_in, (typename V::Real*)M, L.ld_out);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::aba(const V& mv, const Launch& L, const void* q, const void* qd, const void* tau, const double* g,
                 const void* fext, void* qdd, int32_t* status) {
  if (fext)
    k_aba<V, true><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, (const typename V::Real*)qd, (const typename V::Real*)tau,
                                                               L.ld_in, g3_of<typename V::Real>(g), (const typename V::Real*)fext, (typename V::Real*)qdd, L.ld_out,
                                                               status);
  else
    k_aba<V, false><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, (const typename V::Real*)qd, (const typename V::Real*)tau,
                                                                L.ld_in, g3_of<typename V::Real>(g), nullptr, (typename V::Real*)qdd, L.ld_out,
                                                                status);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::dyn(const V& mv, const Launch& L, const void* q, const void* qd, const void* tau, const double* g, void* M,
                 void* bias, void* qdd, int32_t* status) {
  k_dyn<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, (const typename V::Real*)qd, (const typename V::Real*)tau, L.ld_in,
                                                        g3_of<typename V::Real>(g), (typename V::Real*)M, (typename V::Real*)bias, (typename V::Real*)qdd, L.ld_out, status);
  return (int)cudaGetLastError();
}

template <class V>
int Launcher<V>::osc(const V& mv, const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau,
                 void* lambda, int32_t* status) {
  k_osc<V><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(mv, L.N, (const typename V::Real*)q, (const typename V::Real*)qd, L.ld_in, P, (typename V::Real*)tau,
                                                        (typename V::Real*)lambda, L.ld_out, status);
  return (int)cudaGetLastError();
}

}  // namespace vdk
