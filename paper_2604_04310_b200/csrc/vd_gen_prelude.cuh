// Shared prelude of the generated straight-line routines (vd_gen_robots.cuh
// and the per-model JIT translation units): scalar helpers the emitted code
// calls.  Hand-maintained; tools/gen_tree_kernels.py emits only the robot
// structs.
#pragma once

#include <cmath>
#include <cstdint>

#include "vd_sincos.cuh"

#ifndef VD_HD
#if defined(__CUDACC__)
#define VD_HD __host__ __device__ __forceinline__
#else
#define VD_HD inline
#endif
#endif

namespace vdk {

template <class T> VD_HD T vd_sqrt(T x) { using std::sqrt; return sqrt(x); }
// rotation_log (control.hpp:45-68), the reference acos form and branches
template <class T>
VD_HD void vd_rotation_log(const T* R, T* w) {
  using std::acos; using std::sin; using std::sqrt;
  const T tr = R[0] + R[4] + R[8];
  const T anti[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  T ca = T(0.5) * (tr - T(1));
  ca = ca < T(-1) ? T(-1) : (ca > T(1) ? T(1) : ca);
  const T ang = acos(ca);
  const T pi = T(3.14159265358979323846);
  if (ang < T(1e-9)) {
    for (int k = 0; k < 3; ++k) w[k] = T(0.5) * anti[k];
    return;
  }
  if (ang > pi - T(1e-6)) {
    const T sd[3] = {T(0.5) * (R[0] + T(1)), T(0.5) * (R[4] + T(1)), T(0.5) * (R[8] + T(1))};
    int k = 0;
    if (sd[1] > sd[k]) k = 1;
    if (sd[2] > sd[k]) k = 2;
    T ax[3];
    for (int r = 0; r < 3; ++r) ax[r] = (r == k) ? sd[k] : T(0.5) * R[r * 3 + k];
    const T inv = T(1) / sqrt(sd[k] > T(1e-12) ? sd[k] : T(1e-12));
    for (int r = 0; r < 3; ++r) ax[r] *= inv;
    const T nrm = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    for (int r = 0; r < 3; ++r) ax[r] /= nrm;
    const T sgn = (anti[0] * ax[0] + anti[1] * ax[1] + anti[2] * ax[2]) < T(0) ? T(-1) : T(1);
    for (int r = 0; r < 3; ++r) w[r] = ang * sgn * ax[r];
    return;
  }
  const T f = T(0.5) * ang / sin(ang);
  for (int k = 0; k < 3; ++k) w[k] = f * anti[k];
}

// How a generated routine evaluates sin/cos (Cfg::kFast -> Cx::kFastTrig)
enum : int {
  kTrigLib = 0,   // the library sincos / sincosf, inlined at every joint
  kTrigFast = 1,  // vd_sincos_f64 / vd_sincos_f32 (vd_sincos.cuh), inlined
  kTrigCall = 2,  // the library routine, one out-of-line copy per kernel
  kTrigFastCall = 3,  // vd_sincos_f64 / vd_sincos_f32, one out-of-line copy per kernel
};

#if defined(__CUDA_ARCH__)
// library sincos by default: vd_sincos_f64's __constant__ coefficients get
// hoisted out of the persistent loop into registers and spilled in these
// 168/255-register kernels (measured slower)
__device__ __forceinline__ void vd_sincos(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ void vd_sincos(float x, float* s, float* c) { sincosf(x, s, c); }
// kTrigCall: the G1 routines are instruction-cache bound, and the library
// sincos inlines ~70 instructions at each of 26 joints; one out-of-line copy
// (a call per joint, result in registers) makes the G1 ABA fp64 0.294 ->
// 0.262 ms and RNEA 0.100 -> 0.094 ms (tools/async_sweep.cu t29), while the
// 168-register CRBA / FK routines get slower (the call's register save)
static __device__ __noinline__ double2 vd_sincos_call(double x) {
  double2 r;
  sincos(x, &r.x, &r.y);
  return r;
}
static __device__ __noinline__ float2 vd_sincos_call(float x) {
  float2 r;
  sincosf(x, &r.x, &r.y);
  return r;
}
// kTrigFastCall: the Cody-Waite / fdlibm routine out of line, so its
// __constant__ coefficients are read inside the called function (constant-bank
// operands) and cannot be hoisted out of a persistent loop
static __device__ __noinline__ double2 vd_sincos_fast_call(double x) {
  double2 r;
  vd_sincos_f64(x, &r.x, &r.y);
  return r;
}
static __device__ __noinline__ float2 vd_sincos_fast_call(float x) {
  float2 r;
  vd_sincos_f32(x, &r.x, &r.y);
  return r;
}
template <class T> __device__ __forceinline__ bool vd_isfinite(T x) { return isfinite(x); }
#else
template <class T> inline void vd_sincos(T x, T* s, T* c) { *s = std::sin(x); *c = std::cos(x); }
template <class T> inline bool vd_isfinite(T x) { return std::isfinite(x); }
#endif
// Cx::kFastTrig: kTrigLib / kTrigFast / kTrigCall above.  kTrigFast in fp32
// makes the Panda ABA 0.300 -> 0.287 ms at 4 M states but the G1 fp32
// routines 5-15 % slower (tools/sweep.py).
template <class Cx, class T>
VD_HD void vd_sincos_cx(T x, T* s, T* c) {
#if defined(__CUDA_ARCH__)
  if constexpr (int(Cx::kFastTrig) == kTrigFast && sizeof(T) == 8) { vd_sincos_f64(x, s, c); return; }
  if constexpr (int(Cx::kFastTrig) == kTrigFast && sizeof(T) == 4) { vd_sincos_f32(x, s, c); return; }
  if constexpr (int(Cx::kFastTrig) == kTrigCall) {
    const auto r = vd_sincos_call(x);
    *s = r.x;
    *c = r.y;
    return;
  }
  if constexpr (int(Cx::kFastTrig) == kTrigFastCall) {
    const auto r = vd_sincos_fast_call(x);
    *s = r.x;
    *c = r.y;
    return;
  }
#endif
  vd_sincos(x, s, c);
}

}  // namespace vdk
