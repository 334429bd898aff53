// Device-side model views and spatial algebra for the sm_100a kernels.
//
// Every algorithm in vd_algos.cuh is written once against a *model view*:
//   RuntimeView<T>  — topology and constants read from a device-resident
//                     DevModel<T> (any URDF with n <= 64); per-joint state lives
//                     in local memory.
//   StaticView<Robot, T> — generated compile-time tables (vd_robots_gen.cuh):
//                     n, parents, joint kinds/axes, offsets and inertias are
//                     constants, loops fully unroll, per-joint state is
//                     register-resident.
//
// Structural zeros.  IEEE semantics forbid the compiler from folding x*0.0, so
// a model with axis-aligned joints and sparse offsets/inertias would still pay
// for every zero term.  All arithmetic therefore goes through `sp<T, F>`: a
// scalar that carries a "may be non-zero" flag.  For static views (F = true)
// the flags are compile-time constants after unrolling and every product with a
// structural zero disappears; for runtime views (F = false) the flag is a
// static `true` and sp<T,false> is a plain T.
//
// Conventions follow the reference (spatial.hpp): 6-vectors angular first;
// transforms map child -> parent, x_parent = R x + p; spatial inertias about
// the body-frame origin.  A joint transform is kept in two stages, the constant
// offset X_off (model.hpp:68) and the joint motion X_J(q) (model.hpp:167-173),
// so X = X_off ∘ X_J as in kinematics.hpp:35-38.
#pragma once

#include <cstdint>

#include "vd_shared.hpp"
#include "vd_sincos.cuh"

#ifndef VD_RT_MINBLOCKS
#define VD_RT_MINBLOCKS 4
#endif

namespace vdk {

// ================================================================== sparse-aware scalar
template <class T, bool F>
struct sp;

template <class T>
struct sp<T, true> {
  T v;
  bool nz;
  __device__ __forceinline__ sp() : v(T(0)), nz(false) {}
  __device__ __forceinline__ sp(T x) : v(x), nz(true) {}
  __device__ __forceinline__ sp(T x, bool n) : v(n ? x : T(0)), nz(n) {}
};
template <class T>
struct sp<T, false> {
  T v;
  static constexpr bool nz = true;
  // Trivial default constructor: per-joint scratch arrays of the loop kernels
  // must not be zero-filled on entry (that turned into kilobytes of local
  // memory stores per thread).  S() still value-initialises to zero.
  sp() = default;
  __device__ __forceinline__ sp(T x) : v(x) {}
  __device__ __forceinline__ sp(T x, bool) : v(x) {}
};

template <class T, bool F>
__device__ __forceinline__ sp<T, F> operator*(const sp<T, F>& a, const sp<T, F>& b) {
  if constexpr (F) {
    return (a.nz && b.nz) ? sp<T, F>(a.v * b.v, true) : sp<T, F>();
  } else {
    return sp<T, F>(a.v * b.v);
  }
}
template <class T, bool F>
__device__ __forceinline__ sp<T, F> operator+(const sp<T, F>& a, const sp<T, F>& b) {
  if constexpr (F) {
    if (!a.nz) return b;
    if (!b.nz) return a;
    return sp<T, F>(a.v + b.v, true);
  } else {
    return sp<T, F>(a.v + b.v);
  }
}
template <class T, bool F>
__device__ __forceinline__ sp<T, F> operator-(const sp<T, F>& a) {
  if constexpr (F) {
    return a.nz ? sp<T, F>(-a.v, true) : a;
  } else {
    return sp<T, F>(-a.v);
  }
}
template <class T, bool F>
__device__ __forceinline__ sp<T, F> operator-(const sp<T, F>& a, const sp<T, F>& b) {
  if constexpr (F) {
    if (!b.nz) return a;
    if (!a.nz) return sp<T, F>(-b.v, true);
    return sp<T, F>(a.v - b.v, true);
  } else {
    return sp<T, F>(a.v - b.v);
  }
}
template <class T, bool F>
__device__ __forceinline__ sp<T, F>& operator+=(sp<T, F>& a, const sp<T, F>& b) {
  a = a + b;
  return a;
}
template <class T, bool F>
__device__ __forceinline__ sp<T, F>& operator-=(sp<T, F>& a, const sp<T, F>& b) {
  a = a - b;
  return a;
}

// ================================================================== model storage / views


template <class T>
struct RuntimeView {
  using Real = T;
  using S = sp<T, false>;
  static constexpr bool kStatic = false;
  static constexpr int kMax = kMaxDof;
  static constexpr int kMaxDepthC = kMaxDof;
  // >= 4 resident 128-thread blocks per SM (<= 128 registers): the loop
  // kernels are latency-bound on their per-joint local-memory state.
  static constexpr int kMinBlocks = VD_RT_MINBLOCKS;
  // The whole model travels by value in the kernel's parameter space
  // (__grid_constant__): warp-uniform indexed reads hit the constant cache.
  DevModel<T> m;
  __device__ __forceinline__ int n() const { return m.n; }
  __device__ __forceinline__ int max_depth() const { return m.n; }
  __device__ __forceinline__ int parent(int i) const { return m.parent[i]; }
  __device__ __forceinline__ int kind(int i) const { return m.kind[i]; }
  __device__ __forceinline__ int axis_code(int i) const { return m.axis_code[i]; }
  __device__ __forceinline__ int depth(int i) const { return m.depth[i]; }
  __device__ __forceinline__ uint64_t anc(int i) const { return m.anc[i]; }
  __device__ __forceinline__ int flags(int i) const { return m.flags[i]; }
  __device__ __forceinline__ int oflags(int i) const { return m.oflags[i]; }
  __device__ __forceinline__ S axis(int i, int k) const { return S(m.axis[i][k]); }
  __device__ __forceinline__ S R(int i, int k) const { return S(m.R[i][k]); }
  __device__ __forceinline__ S p(int i, int k) const { return S(m.p[i][k]); }
  __device__ __forceinline__ S I(int i, int k) const { return S(m.I[i][k]); }
};

// Robot tables generated by tools/gen_robot_tables.py provide a struct with
// static __device__ const arrays; StaticView reads them with indices that are
// constants after unrolling, so every lookup folds.
template <class Robot, class T>
struct StaticView {
  using Real = T;
  using S = sp<T, true>;
  static constexpr bool kStatic = true;
  static constexpr int kMax = Robot::kN;
  static constexpr int kMaxDepthC = Robot::kMaxDepth;
  // 0 = no .minnctapersm: ptxas then keeps register use (and occupancy) as
  // in a plain __launch_bounds__(128); minBlocks=1 let it grow FK from 64 to
  // 126 registers and cost 10-30% on the chain kernels.
  static constexpr int kMinBlocks = 0;
  __device__ __forceinline__ static constexpr int n() { return Robot::kN; }
  __device__ __forceinline__ static constexpr int max_depth() { return Robot::kMaxDepth; }
  __device__ __forceinline__ int parent(int i) const { return Robot::parent()[i]; }
  __device__ __forceinline__ int kind(int i) const { return Robot::kind()[i]; }
  __device__ __forceinline__ int axis_code(int i) const { return Robot::axis_code()[i]; }
  __device__ __forceinline__ int depth(int i) const { return Robot::depth()[i]; }
  __device__ __forceinline__ uint64_t anc(int i) const { return Robot::anc()[i]; }
  __device__ __forceinline__ int flags(int i) const { return Robot::flags()[i]; }
  __device__ __forceinline__ int oflags(int i) const { return Robot::oflags()[i]; }
  __device__ __forceinline__ S cst(double x) const { return S(T(x), x != 0.0); }
  __device__ __forceinline__ S axis(int i, int k) const { return cst(Robot::axis()[i * 3 + k]); }
  __device__ __forceinline__ S R(int i, int k) const { return cst(Robot::rot()[i * 9 + k]); }
  __device__ __forceinline__ S p(int i, int k) const { return cst(Robot::pos()[i * 3 + k]); }
  __device__ __forceinline__ S I(int i, int k) const { return cst(Robot::inertia()[i * 10 + k]); }
};

// ================================================================== spatial vectors
template <class S>
struct SV {  // angular first
  S a[3], l[3];
};
template <class S>
__device__ __forceinline__ void cross3(const S* x, const S* y, S* o) {
  o[0] = x[1] * y[2] - x[2] * y[1];
  o[1] = x[2] * y[0] - x[0] * y[2];
  o[2] = x[0] * y[1] - x[1] * y[0];
}
template <class S>
__device__ __forceinline__ S dot3(const S* x, const S* y) {
  return x[0] * y[0] + x[1] * y[1] + x[2] * y[2];
}
template <class S>
__device__ __forceinline__ SV<S> operator+(const SV<S>& x, const SV<S>& y) {
  SV<S> o;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o.a[k] = x.a[k] + y.a[k];
    o.l[k] = x.l[k] + y.l[k];
  }
  return o;
}
template <class S>
__device__ __forceinline__ SV<S> operator-(const SV<S>& x, const SV<S>& y) {
  SV<S> o;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o.a[k] = x.a[k] - y.a[k];
    o.l[k] = x.l[k] - y.l[k];
  }
  return o;
}
template <class S>
__device__ __forceinline__ SV<S> scale(const SV<S>& x, const S& s) {
  SV<S> o;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o.a[k] = x.a[k] * s;
    o.l[k] = x.l[k] * s;
  }
  return o;
}
// v × m  (spatial.hpp:204-208)
template <class S>
__device__ __forceinline__ SV<S> crm(const SV<S>& v, const SV<S>& m) {
  SV<S> o;
  S t[3];
  cross3(v.a, m.a, o.a);
  cross3(v.a, m.l, o.l);
  cross3(v.l, m.a, t);
#pragma unroll
  for (int k = 0; k < 3; ++k) o.l[k] += t[k];
  return o;
}
// v ×* f  (spatial.hpp:212-216)
template <class S>
__device__ __forceinline__ SV<S> crf(const SV<S>& v, const SV<S>& f) {
  SV<S> o;
  S t[3];
  cross3(v.a, f.a, o.a);
  cross3(v.l, f.l, t);
#pragma unroll
  for (int k = 0; k < 3; ++k) o.a[k] += t[k];
  cross3(v.a, f.l, o.l);
  return o;
}
template <class S>
__device__ __forceinline__ S sdot(const SV<S>& f, const SV<S>& m) {
  return dot3(f.a, m.a) + dot3(f.l, m.l);
}

// ================================================================== joint motion X_J(q)
template <class S>
struct JM {  // revolute: (c, s) = (cos q, sin q); prismatic: q
  S c, s, q;
};
template <class T>
__device__ __forceinline__ void sincos_t(T x, T* s, T* c);
template <>
__device__ __forceinline__ void sincos_t<double>(double x, double* s, double* c) {
  sincos(x, s, c);
}
template <>
__device__ __forceinline__ void sincos_t<float>(float x, float* s, float* c) {
  // vd_sincos_f32 in the template / loop kernels (tools/sweep.py fp32 against
  // sincosf: Panda fused M + bias + q̈ 0.695 -> 0.657 ms, generic OSC 11.7 ->
  // 8.4 ms, the other loop kernels unchanged to +2.5 %)
  vd_sincos_f32(x, s, c);
}
// kFastTrig: fp64 sin/cos by vd_sincos_f64 (vd_sincos.cuh).  Measured on B200
// it is 2.5 % faster for the chain7 ABA kernel and 2-5 % slower for RNEA /
// fused dynamics / OSC than the library routine, so only ABA opts in.
template <class V, class T, bool kFastTrig = false>
__device__ __forceinline__ JM<typename V::S> joint_motion(const V& mv, int i, T q) {
  using S = typename V::S;
  JM<S> j;
  j.q = S(q);
  if (mv.kind(i) == 0) {
    T s, c;
    if constexpr (kFastTrig && sizeof(T) == 8) vd_sincos_f64(q, &s, &c);
    else sincos_t<T>(q, &s, &c);
    j.s = S(s);
    j.c = S(c);
  }
  return j;
}

// 3x3 joint rotation Q (row-major) with its structural zeros: axis-aligned
// codes give a plane rotation, the general axis uses Rodrigues (spatial.hpp:302-308).
template <class V>
__device__ __forceinline__ void joint_rotation(const V& mv, int i, const JM<typename V::S>& j,
                                               typename V::S* Q) {
  using S = typename V::S;
  using T = typename V::Real;
  const S one(T(1), true);
  const int code = mv.axis_code(i);
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = S();
  if (code < 6) {
    const int k = code % 3, k1 = (k + 1) % 3, k2 = (k + 2) % 3;
    const S s = code < 3 ? j.s : -j.s;
    Q[k * 3 + k] = one;
    Q[k1 * 3 + k1] = j.c;
    Q[k2 * 3 + k2] = j.c;
    Q[k1 * 3 + k2] = -s;
    Q[k2 * 3 + k1] = s;
  } else {
    const S a[3] = {mv.axis(i, 0), mv.axis(i, 1), mv.axis(i, 2)};
    const S omc = one - j.c;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) Q[r * 3 + c] = a[r] * a[c] * omc + (r == c ? j.c : S());
    Q[0 * 3 + 1] -= a[2] * j.s;
    Q[0 * 3 + 2] += a[1] * j.s;
    Q[1 * 3 + 0] += a[2] * j.s;
    Q[1 * 3 + 2] -= a[0] * j.s;
    Q[2 * 3 + 0] -= a[1] * j.s;
    Q[2 * 3 + 1] += a[0] * j.s;
  }
}
template <class V>
__device__ __forceinline__ void offset_rotation(const V& mv, int i, typename V::S* Q) {
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = mv.R(i, k);
}
template <class V>
__device__ __forceinline__ void offset_translation(const V& mv, int i, typename V::S* t) {
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = mv.p(i, k);
}
// prismatic translation t = axis q
template <class V>
__device__ __forceinline__ void joint_translation(const V& mv, int i, const JM<typename V::S>& j, typename V::S* t) {
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = mv.axis(i, k) * j.q;
}

template <class S>
__device__ __forceinline__ void matvec(const S* Q, const S* x, S* y) {  // y = Q x
#pragma unroll
  for (int r = 0; r < 3; ++r) y[r] = Q[r * 3] * x[0] + Q[r * 3 + 1] * x[1] + Q[r * 3 + 2] * x[2];
}
template <class S>
__device__ __forceinline__ void matTvec(const S* Q, const S* x, S* y) {  // y = Qᵀ x
#pragma unroll
  for (int r = 0; r < 3; ++r) y[r] = Q[r] * x[0] + Q[3 + r] * x[1] + Q[6 + r] * x[2];
}

// A generic rigid transform stage (Q, t): x_parent = Q x + t.
// inverse_transform_motion (spatial.hpp:233-238)
template <class S>
__device__ __forceinline__ SV<S> motion_in(const S* Q, const S* t, bool has_t, const SV<S>& m) {
  SV<S> o;
  matTvec(Q, m.a, o.a);
  if (has_t) {
    S tw[3], d[3];
    cross3(t, m.a, tw);
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = m.l[k] - tw[k];
    matTvec(Q, d, o.l);
  } else {
    matTvec(Q, m.l, o.l);
  }
  return o;
}
// transform_motion (spatial.hpp:225-230)
template <class S>
__device__ __forceinline__ SV<S> motion_out(const S* Q, const S* t, bool has_t, const SV<S>& m) {
  SV<S> o;
  matvec(Q, m.a, o.a);
  matvec(Q, m.l, o.l);
  if (has_t) {
    S tw[3];
    cross3(t, o.a, tw);
#pragma unroll
    for (int k = 0; k < 3; ++k) o.l[k] += tw[k];
  }
  return o;
}
// transform_force (spatial.hpp:241-246)
template <class S>
__device__ __forceinline__ SV<S> force_out(const S* Q, const S* t, bool has_t, const SV<S>& f) {
  SV<S> o;
  matvec(Q, f.l, o.l);
  matvec(Q, f.a, o.a);
  if (has_t) {
    S tf[3];
    cross3(t, o.l, tf);
#pragma unroll
    for (int k = 0; k < 3; ++k) o.a[k] += tf[k];
  }
  return o;
}
// inverse_transform_force (spatial.hpp:249-254)
template <class S>
__device__ __forceinline__ SV<S> force_in(const S* Q, const S* t, bool has_t, const SV<S>& f) {
  SV<S> o;
  matTvec(Q, f.l, o.l);
  if (has_t) {
    S tf[3], d[3];
    cross3(t, f.l, tf);
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = f.a[k] - tf[k];
    matTvec(Q, d, o.a);
  } else {
    matTvec(Q, f.a, o.a);
  }
  return o;
}

// ------------------------------------------------------------------ axis-specialised helpers
template <int K>
struct IC {
  static constexpr int v = K;
};
// Calls f(IC<k>) for k in {0,1,2}: per-axis code with constant indices (a
// uniform branch for runtime views, folded for static views).
template <class F>
__device__ __forceinline__ void with_axis(int k, F&& f) {
  if (k == 0) f(IC<0>());
  else if (k == 1) f(IC<1>());
  else f(IC<2>());
}
// Same as with_axis but as a plain switch (no lambda), so nothing can stop the
// body from inlining into the unrolled static kernels.
#define VD_WITH_AXIS(kexpr, ...)          \
  switch (kexpr) {                        \
    case 0: {                             \
      constexpr int K = 0;                \
      __VA_ARGS__;                        \
    } break;                              \
    case 1: {                             \
      constexpr int K = 1;                \
      __VA_ARGS__;                        \
    } break;                              \
    default: {                            \
      constexpr int K = 2;                \
      __VA_ARGS__;                        \
    } break;                              \
  }

// y = R x for the plane rotation about axis K by (c, s)
template <int K, class S>
__device__ __forceinline__ void plane_rot(const S& c, const S& s, const S* x, S* y) {
  constexpr int k1 = (K + 1) % 3, k2 = (K + 2) % 3;
  y[K] = x[K];
  y[k1] = c * x[k1] - s * x[k2];
  y[k2] = s * x[k1] + c * x[k2];
}
// symmetric (xx yy zz xy xz yz) rotated in the plane about axis K: R S Rᵀ
template <int K>
__device__ __forceinline__ constexpr int sidx(int r, int c) {
  return r == c ? r : (r + c == 1 ? 3 : (r + c == 2 ? 4 : 5));
}
template <int K, class S>
__device__ __forceinline__ void plane_rot_sym(const S& c, const S& s, const S* a, S* o) {
  constexpr int k1 = (K + 1) % 3, k2 = (K + 2) % 3;
  const S s11 = a[sidx<K>(k1, k1)], s22 = a[sidx<K>(k2, k2)], s12 = a[sidx<K>(k1, k2)];
  const S s1k = a[sidx<K>(k1, K)], s2k = a[sidx<K>(k2, K)];
  const S cc = c * c, ss = s * s, cs = c * s;
  const S t = cs * (s12 + s12);
  o[sidx<K>(K, K)] = a[sidx<K>(K, K)];
  o[sidx<K>(k1, k1)] = cc * s11 - t + ss * s22;
  o[sidx<K>(k2, k2)] = ss * s11 + t + cc * s22;
  o[sidx<K>(k1, k2)] = cs * (s11 - s22) + (cc - ss) * s12;
  o[sidx<K>(k1, K)] = c * s1k - s * s2k;
  o[sidx<K>(k2, K)] = s * s1k + c * s2k;
}
// general 3x3 (row-major) rotated in the plane about axis K: R B Rᵀ
template <int K, class S>
__device__ __forceinline__ void plane_rot_full(const S& c, const S& s, const S* B, S* o) {
  constexpr int k1 = (K + 1) % 3, k2 = (K + 2) % 3;
  S t[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {  // rows
    t[K * 3 + j] = B[K * 3 + j];
    t[k1 * 3 + j] = c * B[k1 * 3 + j] - s * B[k2 * 3 + j];
    t[k2 * 3 + j] = s * B[k1 * 3 + j] + c * B[k2 * 3 + j];
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {  // columns
    o[r * 3 + K] = t[r * 3 + K];
    o[r * 3 + k1] = c * t[r * 3 + k1] - s * t[r * 3 + k2];
    o[r * 3 + k2] = s * t[r * 3 + k1] + c * t[r * 3 + k2];
  }
}

// Stage helpers for X = X_off ∘ X_J.  The joint stage is a plane rotation
// (axis-aligned revolute), Rodrigues (general revolute) or a translation
// along the axis (prismatic); the offset stage skips an identity rotation /
// zero translation (model flags, uniform per joint).
template <class V>
struct JointX {
  using S = typename V::S;
  int code;        // 0..5 unit axis ±x,±y,±z ; 6 general
  bool prismatic;
  bool qo_id, to_zero;
  S c, s;          // revolute: cos q, ±sin q (sign of the axis folded in)
  S QJ[9];         // general revolute only
  S tJ[3];         // prismatic only
  S QO[9], tO[3];
  __device__ __forceinline__ void load(const V& mv, int i, const JM<S>& j) {
    prismatic = mv.kind(i) == 1;
    code = mv.axis_code(i);
    const int of = mv.oflags(i);
    qo_id = (of & kOffRotIdentity) != 0;
    to_zero = (of & kOffTransZero) != 0;
    if (prismatic) {
      joint_translation(mv, i, j, tJ);
    } else if (V::kStatic || code == 6) {
      // static views: a full Q whose structural zeros fold (sp flags)
      joint_rotation(mv, i, j, QJ);
    } else {
      c = j.c;
      s = code < 3 ? j.s : -j.s;
    }
    if (V::kStatic || !qo_id) offset_rotation(mv, i, QO);
    if (V::kStatic || !to_zero) offset_translation(mv, i, tO);
    if (V::kStatic && prismatic) {  // identity joint rotation with folding zeros
      const S one(typename V::Real(1), true);
#pragma unroll
      for (int k = 0; k < 9; ++k) QJ[k] = (k % 4 == 0) ? one : S();
    }
  }
  // R_J x (dir > 0) or R_Jᵀ x (dir < 0); revolute only
  __device__ __forceinline__ void jrot(const S* x, S* y, int dir) const {
    if (!V::kStatic && code < 6) {
      const S sg = dir > 0 ? s : -s;
      VD_WITH_AXIS(code % 3, plane_rot<K>(c, sg, x, y);)
    } else if (dir > 0) {
      matvec(QJ, x, y);
    } else {
      matTvec(QJ, x, y);
    }
  }
  // joint stage, parent side -> child side (inverse_transform_motion)
  __device__ __forceinline__ SV<S> j_motion_in(const SV<S>& m) const {
    SV<S> o;
    if (!prismatic) {
      jrot(m.a, o.a, -1);
      jrot(m.l, o.l, -1);
    } else {
      S tw[3];
      cross3(tJ, m.a, tw);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o.a[k] = m.a[k];
        o.l[k] = m.l[k] - tw[k];
      }
    }
    return o;
  }
  __device__ __forceinline__ SV<S> j_motion_out(const SV<S>& m) const {
    SV<S> o;
    if (!prismatic) {
      jrot(m.a, o.a, 1);
      jrot(m.l, o.l, 1);
    } else {
      S tw[3];
      cross3(tJ, m.a, tw);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o.a[k] = m.a[k];
        o.l[k] = m.l[k] + tw[k];
      }
    }
    return o;
  }
  __device__ __forceinline__ SV<S> j_force_out(const SV<S>& f) const {
    SV<S> o;
    if (!prismatic) {
      jrot(f.a, o.a, 1);
      jrot(f.l, o.l, 1);
    } else {
      S tf[3];
      cross3(tJ, f.l, tf);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o.a[k] = f.a[k] + tf[k];
        o.l[k] = f.l[k];
      }
    }
    return o;
  }
  // offset stage
  __device__ __forceinline__ SV<S> o_motion_in(const SV<S>& m) const {
    if (qo_id && to_zero) return m;
    if (qo_id) {
      SV<S> o = m;
      S tw[3];
      cross3(tO, m.a, tw);
#pragma unroll
      for (int k = 0; k < 3; ++k) o.l[k] = m.l[k] - tw[k];
      return o;
    }
    return motion_in(QO, tO, !to_zero, m);
  }
  __device__ __forceinline__ SV<S> o_motion_out(const SV<S>& m) const {
    if (qo_id && to_zero) return m;
    if (qo_id) {
      SV<S> o = m;
      S tw[3];
      cross3(tO, m.a, tw);
#pragma unroll
      for (int k = 0; k < 3; ++k) o.l[k] = m.l[k] + tw[k];
      return o;
    }
    return motion_out(QO, tO, !to_zero, m);
  }
  __device__ __forceinline__ SV<S> o_force_out(const SV<S>& f) const {
    if (qo_id && to_zero) return f;
    if (qo_id) {
      SV<S> o = f;
      S tf[3];
      cross3(tO, f.l, tf);
#pragma unroll
      for (int k = 0; k < 3; ++k) o.a[k] = f.a[k] + tf[k];
      return o;
    }
    return force_out(QO, tO, !to_zero, f);
  }
  // parent -> child (inverse_transform_motion of X)
  __device__ __forceinline__ SV<S> motion_to_child(const SV<S>& m) const {
    if constexpr (V::kStatic) return motion_in(QJ, tJ, prismatic, motion_in(QO, tO, true, m));
    return j_motion_in(o_motion_in(m));
  }
  // child -> parent (transform_force of X)
  __device__ __forceinline__ SV<S> force_to_parent(const SV<S>& f) const {
    if constexpr (V::kStatic) return force_out(QO, tO, true, force_out(QJ, tJ, prismatic, f));
    return o_force_out(j_force_out(f));
  }
  __device__ __forceinline__ SV<S> motion_to_parent(const SV<S>& m) const {
    if constexpr (V::kStatic) return motion_out(QO, tO, true, motion_out(QJ, tJ, prismatic, m));
    return o_motion_out(j_motion_out(m));
  }
};

// Joint motion subspace S_i and the products with it that the recursions need,
// specialised for unit axes (the column / component selected directly).
template <class V>
struct JAxis {
  using S = typename V::S;
  int kind, code;
  S a[3];  // axis (general code)
  __device__ __forceinline__ JAxis(const V& mv, int i) : kind(mv.kind(i)), code(mv.axis_code(i)) {
    // static views take the generic path (structural zeros fold through sp)
    if (V::kStatic) code = 6;
    if (code == 6)
#pragma unroll
      for (int k = 0; k < 3; ++k) a[k] = mv.axis(i, k);
  }
  __device__ __forceinline__ S sgn(const S& x) const { return code < 3 ? x : -x; }
  // m += S x
  __device__ __forceinline__ void add(SV<S>& m, const S& x) const {
    if (code < 6) {
      const S y = sgn(x);
      VD_WITH_AXIS(code % 3, if (kind == 0) m.a[K] += y;
        else m.l[K] += y;)
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (kind == 0) m.a[k] += a[k] * x;
        else m.l[k] += a[k] * x;
      }
    }
  }
  __device__ __forceinline__ SV<S> scaled(const S& x) const {
    SV<S> m;
#pragma unroll
    for (int k = 0; k < 3; ++k) m.a[k] = m.l[k] = S();
    add(m, x);
    return m;
  }
  // Sᵀ f
  __device__ __forceinline__ S dot(const SV<S>& f) const {
    if (code < 6) {
      S r;
      VD_WITH_AXIS(code % 3, r = kind == 0 ? f.a[K] : f.l[K];)
      return sgn(r);
    }
    return kind == 0 ? dot3(a, f.a) : dot3(a, f.l);
  }
  // v × (S x)  (spatial.hpp:204-208 with m = S x)
  __device__ __forceinline__ SV<S> crm(const SV<S>& v, const S& x) const {
    if (code < 6) {
      SV<S> o;
      const S y = sgn(x);
      VD_WITH_AXIS(code % 3, constexpr int k = K, k1 = (k + 1) % 3, k2 = (k + 2) % 3;
        // w × e_k = (.., w_k2 at k1, -w_k1 at k2)
        if (kind == 0) {
          o.a[k] = S();
          o.a[k1] = v.a[k2] * y;
          o.a[k2] = -(v.a[k1] * y);
          o.l[k] = S();
          o.l[k1] = v.l[k2] * y;
          o.l[k2] = -(v.l[k1] * y);
        } else {
#pragma unroll
          for (int j = 0; j < 3; ++j) o.a[j] = S();
          o.l[k] = S();
          o.l[k1] = v.a[k2] * y;
          o.l[k2] = -(v.a[k1] * y);
        })
      return o;
    }
    SV<S> m;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      m.a[k] = kind == 0 ? a[k] * x : S();
      m.l[k] = kind == 1 ? a[k] * x : S();
    }
    return vdk::crm(v, m);
  }
};

// ================================================================== rigid-body inertia (10 params)
template <class S>
struct RB {  // m, h = m c, I = {xx, yy, zz, xy, xz, yz} about the origin
  S m, h[3], I[6];
};
template <class V>
__device__ __forceinline__ RB<typename V::S> body_inertia(const V& mv, int i) {
  RB<typename V::S> b;
  b.m = mv.I(i, 0);
#pragma unroll
  for (int k = 0; k < 3; ++k) b.h[k] = mv.I(i, 1 + k);
#pragma unroll
  for (int k = 0; k < 6; ++k) b.I[k] = mv.I(i, 4 + k);
  return b;
}
template <class S>
__device__ __forceinline__ void rb_add(RB<S>& a, const RB<S>& b) {
  a.m += b.m;
#pragma unroll
  for (int k = 0; k < 3; ++k) a.h[k] += b.h[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) a.I[k] += b.I[k];
}
// I v = (Io ω + h × v_lin, m v_lin − h × ω)   (spatial.hpp:179-182 on the 10-param form)
template <class S>
__device__ __forceinline__ SV<S> rb_apply(const RB<S>& b, const SV<S>& v) {
  SV<S> f;
  S hv[3], hw[3];
  cross3(b.h, v.l, hv);
  cross3(b.h, v.a, hw);
  f.a[0] = b.I[0] * v.a[0] + b.I[3] * v.a[1] + b.I[4] * v.a[2] + hv[0];
  f.a[1] = b.I[3] * v.a[0] + b.I[1] * v.a[1] + b.I[5] * v.a[2] + hv[1];
  f.a[2] = b.I[4] * v.a[0] + b.I[5] * v.a[1] + b.I[2] * v.a[2] + hv[2];
#pragma unroll
  for (int k = 0; k < 3; ++k) f.l[k] = b.m * v.l[k] - hw[k];
  return f;
}
// symmetric 3x3 (xx yy zz xy xz yz) rotated: Q S Qᵀ
template <class S>
__device__ __forceinline__ void sym_rotate(const S* Q, const S* s6, S* out) {
  const S s[3][3] = {{s6[0], s6[3], s6[4]}, {s6[3], s6[1], s6[5]}, {s6[4], s6[5], s6[2]}};
  S t[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) t[r][c] = Q[r * 3] * s[0][c] + Q[r * 3 + 1] * s[1][c] + Q[r * 3 + 2] * s[2][c];
  const int ir[6] = {0, 1, 2, 0, 0, 1}, ic[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int r = ir[k], c = ic[k];
    out[k] = t[r][0] * Q[c * 3] + t[r][1] * Q[c * 3 + 1] + t[r][2] * Q[c * 3 + 2];
  }
}
template <class S>
__device__ __forceinline__ void full_rotate(const S* Q, const S* B, S* out) {  // Q B Qᵀ
  S t[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) t[r * 3 + c] = Q[r * 3] * B[c] + Q[r * 3 + 1] * B[3 + c] + Q[r * 3 + 2] * B[6 + c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      out[r * 3 + c] = t[r * 3] * Q[c * 3] + t[r * 3 + 1] * Q[c * 3 + 1] + t[r * 3 + 2] * Q[c * 3 + 2];
}
// transform_inertia (spatial.hpp:259-267) on the 10-param form, X = (Q, t):
//   h' = Q h + m t ;  I' = Q I Qᵀ − t gᵀ − g tᵀ + 2 (g·t) 1 + m (|t|² 1 − t tᵀ),  g = Q h
template <class S>
__device__ __forceinline__ RB<S> rb_out(const RB<S>& b, const S* Q, const S* t, bool has_t, bool has_q = true) {
  RB<S> o;
  o.m = b.m;
  S g[3];
  if (has_q) {
    matvec(Q, b.h, g);
    sym_rotate(Q, b.I, o.I);
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) g[k] = b.h[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) o.I[k] = b.I[k];
  }
  if (!has_t) {
#pragma unroll
    for (int k = 0; k < 3; ++k) o.h[k] = g[k];
    return o;
  }
  const S gt = dot3(g, t);
  const S mt[3] = {b.m * t[0], b.m * t[1], b.m * t[2]};
  // d_k = 2 g_k + m t_k  (so the tensor update is  (2 g·t + m|t|²) 1 − t dᵀ − g tᵀ + ... symmetrised)
  S u[3];  // u = g + m t  = h'
#pragma unroll
  for (int k = 0; k < 3; ++k) u[k] = g[k] + mt[k];
  const S diag = gt + dot3(u, t);  // 2 g·t + m |t|²
  // I' = Q I Qᵀ + diag 1 − t uᵀ − g tᵀ   (symmetric: t uᵀ + g tᵀ = t gᵀ + g tᵀ + m t tᵀ)
  o.I[0] += diag - t[0] * u[0] - g[0] * t[0];
  o.I[1] += diag - t[1] * u[1] - g[1] * t[1];
  o.I[2] += diag - t[2] * u[2] - g[2] * t[2];
  o.I[3] -= t[0] * u[1] + g[0] * t[1];
  o.I[4] -= t[0] * u[2] + g[0] * t[2];
  o.I[5] -= t[1] * u[2] + g[1] * t[2];
#pragma unroll
  for (int k = 0; k < 3; ++k) o.h[k] = u[k];
  return o;
}
template <class V>
__device__ __forceinline__ RB<typename V::S> rb_to_parent(const JointX<V>& x, const RB<typename V::S>& b) {
  using S = typename V::S;
  if constexpr (V::kStatic) return rb_out(rb_out(b, x.QJ, x.tJ, x.prismatic), x.QO, x.tO, true);
  RB<S> mid;
  if (x.prismatic) {
    mid = rb_out(b, static_cast<const S*>(nullptr), x.tJ, true, false);
  } else if (!V::kStatic && x.code < 6) {
    mid.m = b.m;
    VD_WITH_AXIS(x.code % 3, plane_rot<K>(x.c, x.s, b.h, mid.h);
      plane_rot_sym<K>(x.c, x.s, b.I, mid.I);)
  } else {
    mid = rb_out(b, x.QJ, x.tJ, false, true);
  }
  if (x.qo_id && x.to_zero) return mid;
  return rb_out(mid, x.QO, x.tO, !x.to_zero, !x.qo_id);
}

// ================================================================== articulated inertia (sym 6x6)
// IA = [[A, B], [Bᵀ, C]], A and C symmetric (xx yy zz xy xz yz), B row-major.
template <class S>
struct AI {
  S A[6], B[9], C[6];
};
template <class S>
__device__ __forceinline__ AI<S> ai_from_rb(const RB<S>& b) {
  AI<S> o;
#pragma unroll
  for (int k = 0; k < 6; ++k) o.A[k] = b.I[k];
  o.B[0] = S(); o.B[1] = -b.h[2]; o.B[2] = b.h[1];
  o.B[3] = b.h[2]; o.B[4] = S(); o.B[5] = -b.h[0];
  o.B[6] = -b.h[1]; o.B[7] = b.h[0]; o.B[8] = S();
  o.C[0] = o.C[1] = o.C[2] = b.m;
  o.C[3] = o.C[4] = o.C[5] = S();
  return o;
}
template <class S>
__device__ __forceinline__ S sym_at(const S* s6, int r, int c) {
  return r == c ? s6[r] : s6[r + c + 2];  // (0,1)->3, (0,2)->4, (1,2)->5
}
template <class S>
__device__ __forceinline__ SV<S> ai_apply(const AI<S>& I, const SV<S>& v) {
  SV<S> f;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    f.a[r] = sym_at(I.A, r, 0) * v.a[0] + sym_at(I.A, r, 1) * v.a[1] + sym_at(I.A, r, 2) * v.a[2] +
             I.B[r * 3] * v.l[0] + I.B[r * 3 + 1] * v.l[1] + I.B[r * 3 + 2] * v.l[2];
    f.l[r] = I.B[r] * v.a[0] + I.B[3 + r] * v.a[1] + I.B[6 + r] * v.a[2] + sym_at(I.C, r, 0) * v.l[0] +
             sym_at(I.C, r, 1) * v.l[1] + sym_at(I.C, r, 2) * v.l[2];
  }
  return f;
}
// IA S for the joint's motion subspace: a column of IA for unit axes.
template <class V>
__device__ __forceinline__ SV<typename V::S> ai_axis(const JAxis<V>& ax, const AI<typename V::S>& I) {
  using S = typename V::S;
  if (!V::kStatic && ax.code < 6) {
    SV<S> o;
    VD_WITH_AXIS(ax.code % 3, constexpr int k = K;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (ax.kind == 0) {  // column k: (A[:,k]; Bᵀ[:,k] = B[k,:])
          o.a[r] = sym_at(I.A, r, k);
          o.l[r] = I.B[k * 3 + r];
        } else {  // column 3+k: (B[:,k]; C[:,k])
          o.a[r] = I.B[r * 3 + k];
          o.l[r] = sym_at(I.C, r, k);
        }
      })
    if (ax.code >= 3) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        o.a[r] = -o.a[r];
        o.l[r] = -o.l[r];
      }
    }
    return o;
  }
  SV<S> s;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    s.a[r] = ax.kind == 0 ? ax.a[r] : S();
    s.l[r] = ax.kind == 1 ? ax.a[r] : S();
  }
  return ai_apply(I, s);
}
template <class S>
__device__ __forceinline__ void ai_add(AI<S>& a, const AI<S>& b) {
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    a.A[k] += b.A[k];
    a.C[k] += b.C[k];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) a.B[k] += b.B[k];
}
// IA − U Uᵀ / D
template <class S>
__device__ __forceinline__ void ai_sub_outer(AI<S>& I, const SV<S>& U, const S& dinv) {
  const int ir[6] = {0, 1, 2, 0, 0, 1}, ic[6] = {0, 1, 2, 1, 2, 2};
  S ua[3], ul[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ua[k] = U.a[k] * dinv;
    ul[k] = U.l[k] * dinv;
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    I.A[k] -= U.a[ir[k]] * ua[ic[k]];
    I.C[k] -= U.l[ir[k]] * ul[ic[k]];
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) I.B[r * 3 + c] -= U.a[r] * ul[c];
}
// X* IA X*ᵀ for X* = [[Q, t×Q], [0, Q]]: rotate all blocks, then shift by t:
//   A' = A1 + P B1ᵀ − B1 P − P C1 P ;  B' = B1 + P C1 ;  C' = C1   (P = t×)
template <class S>
__device__ __forceinline__ AI<S> ai_out(const AI<S>& I, const S* Q, const S* t, bool has_t, bool has_q = true) {
  AI<S> o;
  if (has_q) {
    sym_rotate(Q, I.A, o.A);
    sym_rotate(Q, I.C, o.C);
    full_rotate(Q, I.B, o.B);
  } else {
    o = I;
  }
  if (!has_t) return o;
  S C1[3][3], PC[3][3], W[3][3], Z[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C1[r][c] = sym_at(o.C, r, c);
#pragma unroll
  for (int c = 0; c < 3; ++c) {  // P C1, column c = t × C1[:, c]
    PC[0][c] = t[1] * C1[2][c] - t[2] * C1[1][c];
    PC[1][c] = t[2] * C1[0][c] - t[0] * C1[2][c];
    PC[2][c] = t[0] * C1[1][c] - t[1] * C1[0][c];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {  // W = P B1ᵀ, column c = t × (row c of B1)
    W[0][c] = t[1] * o.B[c * 3 + 2] - t[2] * o.B[c * 3 + 1];
    W[1][c] = t[2] * o.B[c * 3 + 0] - t[0] * o.B[c * 3 + 2];
    W[2][c] = t[0] * o.B[c * 3 + 1] - t[1] * o.B[c * 3 + 0];
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {  // Z = (P C1) P
    Z[r][0] = PC[r][1] * t[2] - PC[r][2] * t[1];
    Z[r][1] = PC[r][2] * t[0] - PC[r][0] * t[2];
    Z[r][2] = PC[r][0] * t[1] - PC[r][1] * t[0];
  }
  const int ir[6] = {0, 1, 2, 0, 0, 1}, ic[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int k = 0; k < 6; ++k) o.A[k] += (W[ir[k]][ic[k]] + W[ic[k]][ir[k]]) - Z[ir[k]][ic[k]];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o.B[r * 3 + c] += PC[r][c];
  return o;
}
template <class V>
__device__ __forceinline__ AI<typename V::S> ai_to_parent(const JointX<V>& x, const AI<typename V::S>& I) {
  using S = typename V::S;
  if constexpr (V::kStatic) return ai_out(ai_out(I, x.QJ, x.tJ, x.prismatic), x.QO, x.tO, true);
  AI<S> mid;
  if (x.prismatic) {
    mid = ai_out(I, static_cast<const S*>(nullptr), x.tJ, true, false);
  } else if (!V::kStatic && x.code < 6) {
    VD_WITH_AXIS(x.code % 3, plane_rot_sym<K>(x.c, x.s, I.A, mid.A);
      plane_rot_sym<K>(x.c, x.s, I.C, mid.C);
      plane_rot_full<K>(x.c, x.s, I.B, mid.B);)
  } else {
    mid = ai_out(I, x.QJ, x.tJ, false, true);
  }
  if (x.qo_id && x.to_zero) return mid;
  return ai_out(mid, x.QO, x.tO, !x.to_zero, !x.qo_id);
}

// ================================================================== world poses
template <class S>
struct WX {  // R row-major, p
  S R[9], p[3];
};
// world_i = world_parent ∘ X_off ∘ X_J  (kinematics.hpp:43-56)
template <class V>
__device__ __forceinline__ WX<typename V::S> world_of(const JointX<V>& x, const WX<typename V::S>* wp) {
  using S = typename V::S;
  // local rotation Rl = R_off R_J, translation pl = p_off + R_off t_J
  S Rl[9], pl[3];
  if constexpr (V::kStatic) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        Rl[r * 3 + c] = x.QO[r * 3] * x.QJ[c] + x.QO[r * 3 + 1] * x.QJ[3 + c] + x.QO[r * 3 + 2] * x.QJ[6 + c];
#pragma unroll
    for (int k = 0; k < 3; ++k) pl[k] = x.tO[k];
    if (x.prismatic) {
      S rt[3];
      matvec(x.QO, x.tJ, rt);
#pragma unroll
      for (int k = 0; k < 3; ++k) pl[k] += rt[k];
    }
  } else {
    S QOm[9];
    const S one(typename V::Real(1), true);
#pragma unroll
    for (int k = 0; k < 9; ++k) QOm[k] = x.qo_id ? ((k % 4 == 0) ? one : S()) : x.QO[k];
    if (x.prismatic) {
#pragma unroll
      for (int k = 0; k < 9; ++k) Rl[k] = QOm[k];
    } else {
      // columns of R_off R_J = R_J applied to rows of R_off: (R_off R_J)[r][:] = R_Jᵀ (row r of R_off)
#pragma unroll
      for (int r = 0; r < 3; ++r) x.jrot(&QOm[r * 3], &Rl[r * 3], -1);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) pl[k] = x.to_zero ? S() : x.tO[k];
    if (x.prismatic) {
      S rt[3];
      matvec(QOm, x.tJ, rt);
#pragma unroll
      for (int k = 0; k < 3; ++k) pl[k] += rt[k];
    }
  }
  WX<S> w;
  if (!wp) {
#pragma unroll
    for (int k = 0; k < 9; ++k) w.R[k] = Rl[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) w.p[k] = pl[k];
    return w;
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      w.R[r * 3 + c] = wp->R[r * 3] * Rl[c] + wp->R[r * 3 + 1] * Rl[3 + c] + wp->R[r * 3 + 2] * Rl[6 + c];
    w.p[r] = wp->R[r * 3] * pl[0] + wp->R[r * 3 + 1] * pl[1] + wp->R[r * 3 + 2] * pl[2] + wp->p[r];
  }
  return w;
}

}  // namespace vdk
