// Forward-mode JVPs of the device algorithms (dual.hpp:14-196, autodiff.hpp:41-56).
//
// The reference makes every algorithm generic over its scalar and obtains
// D f(x)·v by running f on dual numbers.  The device algorithms are generic
// over a model view, so the same recursion runs on duals through JView<V>:
// a view whose scalar is Dual<T> and whose model constants are lifted with a
// zero tangent.  For compile-time views the structural-zero flags of sp<>
// still fold (a zero constant stays a zero dual), so the tangent pass costs
// about one extra multiply-add per value multiply.  One thread per state; the
// output is written as two SoA arrays (values, tangents).
#pragma once

#include "vd_kernels.cuh"

namespace vdk {

template <class T>
struct Dual {
  T value, tangent;
  Dual() = default;
  __host__ __device__ __forceinline__ Dual(T x) : value(x), tangent(T(0)) {}  // NOLINT: lift of constants
  __host__ __device__ __forceinline__ Dual(T x, T dx) : value(x), tangent(dx) {}

  friend __device__ __forceinline__ Dual operator+(const Dual& a, const Dual& b) {
    return {a.value + b.value, a.tangent + b.tangent};
  }
  friend __device__ __forceinline__ Dual operator-(const Dual& a, const Dual& b) {
    return {a.value - b.value, a.tangent - b.tangent};
  }
  friend __device__ __forceinline__ Dual operator-(const Dual& a) { return {-a.value, -a.tangent}; }
  friend __device__ __forceinline__ Dual operator*(const Dual& a, const Dual& b) {
    return {a.value * b.value, a.tangent * b.value + a.value * b.tangent};
  }
  friend __device__ __forceinline__ Dual operator/(const Dual& a, const Dual& b) {
    return {a.value / b.value, (a.tangent * b.value - a.value * b.tangent) / (b.value * b.value)};
  }
  __device__ __forceinline__ Dual& operator+=(const Dual& o) { return *this = *this + o; }
  __device__ __forceinline__ Dual& operator-=(const Dual& o) { return *this = *this - o; }
  __device__ __forceinline__ Dual& operator*=(const Dual& o) { return *this = *this * o; }
  // comparisons act on values only (dual.hpp:77-95)
  friend __device__ __forceinline__ bool operator>(const Dual& a, const Dual& b) { return a.value > b.value; }
  friend __device__ __forceinline__ bool operator<(const Dual& a, const Dual& b) { return a.value < b.value; }
  friend __device__ __forceinline__ bool operator>=(const Dual& a, const Dual& b) { return a.value >= b.value; }
  friend __device__ __forceinline__ bool operator<=(const Dual& a, const Dual& b) { return a.value <= b.value; }
  friend __device__ __forceinline__ bool operator==(const Dual& a, const Dual& b) { return a.value == b.value; }
  friend __device__ __forceinline__ bool operator!=(const Dual& a, const Dual& b) { return a.value != b.value; }
  friend __device__ __forceinline__ Dual sqrt(const Dual& x) {
    const T s = sqrt(x.value);
    return {s, x.tangent / (T(2) * s)};
  }
  // dual.hpp:178-180
  friend __device__ __forceinline__ bool isfinite(const Dual& x) { return isfinite(x.value) && isfinite(x.tangent); }
};

// sin/cos of a dual (dual.hpp:97-102), one sincos of the value.
template <>
__device__ __forceinline__ void sincos_t<Dual<double>>(Dual<double> x, Dual<double>* s, Dual<double>* c) {
  double sv, cv;
  vd_sincos_f64(x.value, &sv, &cv);
  *s = Dual<double>(sv, cv * x.tangent);
  *c = Dual<double>(cv, -sv * x.tangent);
}
template <>
__device__ __forceinline__ void sincos_t<Dual<float>>(Dual<float> x, Dual<float>* s, Dual<float>* c) {
  float sv, cv;
  sincos_t<float>(x.value, &sv, &cv);
  *s = Dual<float>(sv, cv * x.tangent);
  *c = Dual<float>(cv, -sv * x.tangent);
}

// Seeded SoA input: values from x, tangents from dx (NULL = zero tangent), seed() of autodiff.hpp:14-20.
template <class T>
struct Cols<Dual<T>> {
  const T* __restrict__ base;
  const T* __restrict__ dbase;
  int64_t ld, i;
  __device__ __forceinline__ Dual<T> operator[](int k) const {
    const int64_t o = (int64_t)k * ld + i;
    return Dual<T>(base ? __ldg(base + o) : T(0), dbase ? __ldg(dbase + o) : T(0));
  }
};
// values() / tangents() of autodiff.hpp:22-36 as two SoA outputs (either may be NULL).
template <class T>
struct OutCols<Dual<T>> {
  T* __restrict__ base;
  T* __restrict__ dbase;
  int64_t ld, i;
  __device__ __forceinline__ void put(int k, Dual<T> x) const {
    const int64_t o = (int64_t)k * ld + i;
    if (base) base[o] = x.value;
    if (dbase) dbase[o] = x.tangent;
  }
};

// A model view whose scalar is Dual<T>; model constants get a zero tangent.
template <class V>
struct JView {
  using Base = V;
  using Real = Dual<typename V::Real>;
  using S = sp<Real, V::kStatic>;
  static constexpr bool kStatic = V::kStatic;
  static constexpr int kMax = V::kMax;
  static constexpr int kMaxDepthC = V::kMaxDepthC;
  static constexpr int kMinBlocks = V::kMinBlocks;
  V b;
  __device__ __forceinline__ int n() const { return b.n(); }
  __device__ __forceinline__ int max_depth() const { return b.max_depth(); }
  __device__ __forceinline__ int parent(int i) const { return b.parent(i); }
  __device__ __forceinline__ int kind(int i) const { return b.kind(i); }
  __device__ __forceinline__ int axis_code(int i) const { return b.axis_code(i); }
  __device__ __forceinline__ int depth(int i) const { return b.depth(i); }
  __device__ __forceinline__ uint64_t anc(int i) const { return b.anc(i); }
  __device__ __forceinline__ int flags(int i) const { return b.flags(i); }
  __device__ __forceinline__ int oflags(int i) const { return b.oflags(i); }
  __device__ __forceinline__ static S lift(const typename V::S& x) { return S(Real(x.v), x.nz); }
  __device__ __forceinline__ S axis(int i, int k) const { return lift(b.axis(i, k)); }
  __device__ __forceinline__ S R(int i, int k) const { return lift(b.R(i, k)); }
  __device__ __forceinline__ S p(int i, int k) const { return lift(b.p(i, k)); }
  __device__ __forceinline__ S I(int i, int k) const { return lift(b.I(i, k)); }
};

template <class JV, int kOp>
__device__ __forceinline__ void jvp_dynamics(const JV& mv, const JM<typename JV::S>* jm, const JvpArgs& a, int64_t ldi,
                                             int64_t i, const OutCols<typename JV::Real>& o) {
  using D = typename JV::Real;
  using T = typename JV::Base::Real;
  using S = typename JV::S;
  const int n = mv.n();
  D g[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = D(T(a.g[k]));
  const Cols<D> qd{(const T*)a.x[1], (const T*)a.dx[1], ldi, i};
  const Cols<D> x2{(const T*)a.x[2], (const T*)a.dx[2], ldi, i};
  const Cols<D> fc{(const T*)a.fext, nullptr, ldi, i};
  S out[JV::kMax];
  if constexpr (kOp == kJvpRNEA) {
    const bool has_qdd = a.x[2] != nullptr || a.dx[2] != nullptr;
    if (a.fext)
      rnea_one<JV, true>(mv, jm, qd, has_qdd ? &x2 : static_cast<const Cols<D>*>(nullptr), g, &fc, out);
    else
      rnea_one<JV, false>(mv, jm, qd, has_qdd ? &x2 : static_cast<const Cols<D>*>(nullptr), g, nullptr, out);
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) o.put(j, out[j].v);
  } else {
  bool ok;
  if constexpr (JV::kStatic) {
    ok = a.fext ? aba_one<JV, true>(mv, jm, qd, x2, g, &fc, out) : aba_one<JV, false>(mv, jm, qd, x2, g, nullptr, out);
  } else {
    D qdl[JV::kMax], taul[JV::kMax];
    for (int j = 0; j < n; ++j) {
      qdl[j] = qd[j];
      taul[j] = x2[j];
    }
    ok = a.fext ? aba_one<JV, true>(mv, jm, Row<D>{qdl}, Row<D>{taul}, g, &fc, out)
                : aba_one<JV, false>(mv, jm, Row<D>{qdl}, Row<D>{taul}, g, nullptr, out);
  }
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) o.put(j, ok ? out[j].v : D(T(0)));
  if (a.status) a.status[i] = ok ? 0 : 7;
  }
}


template <class JV, int kOp>
__global__ void __launch_bounds__(kBlock) k_jvp(const __grid_constant__ JV mv, int64_t N, JvpArgs a, int64_t ldi,
                                                int64_t ldo) {
  using D = typename JV::Real;
  using T = typename JV::Base::Real;
  using S = typename JV::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const Cols<D> q{(const T*)a.x[0], (const T*)a.dx[0], ldi, i};
  JM<S> jm[JV::kMax];
  load_motion(mv, q, jm);
  const OutCols<D> o{(T*)a.out, (T*)a.dout, ldo, i};
  const int n = mv.n();
  if constexpr (kOp == kJvpFK) {
    WX<S> W[JV::kMax];
    fk_world(mv, jm, W);
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int r = 0; r < 3; ++r) o.put(j * 12 + c * 3 + r, W[j].R[r * 3 + c].v);
#pragma unroll
      for (int r = 0; r < 3; ++r) o.put(j * 12 + 9 + r, W[j].p[r].v);
    }
  } else if constexpr (kOp == kJvpCRBA) {
    crba_one(mv, jm, [&](int r, int c, const S& val) {
      o.put(c * n + r, val.v);
      if (r != c) o.put(r * n + c, val.v);
    });
#pragma unroll
    for (int r = 0; r < mv.n(); ++r)
#pragma unroll
      for (int c = 0; c < mv.n(); ++c)
        if (!((mv.anc(r) >> c) & 1ull) && !((mv.anc(c) >> r) & 1ull)) o.put(c * n + r, D(T(0)));
  } else {
    jvp_dynamics<JV, kOp>(mv, jm, a, ldi, i, o);
  }
}

// JVP of manipulability(geometric_jacobian(frame)) (kinematics.hpp:138-153 on
// dual.hpp scalars): w and D w(q)·dq, one plane each (either may be NULL).
// The building block of lie_derivative for the SPEC's CBF example
// (control.hpp:157-163: L_f h = JVP of h along f).
template <class JV>
__global__ void __launch_bounds__(kBlock) k_manip_jvp(const __grid_constant__ JV mv, int64_t N,
                                                      const typename JV::Base::Real* __restrict__ q,
                                                      const typename JV::Base::Real* __restrict__ dq, int64_t ldi,
                                                      const __grid_constant__ TaskShared P,
                                                      typename JV::Base::Real* __restrict__ w,
                                                      typename JV::Base::Real* __restrict__ dw) {
  using D = typename JV::Real;
  using S = typename JV::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  JM<S> jm[JV::kMax];
  load_motion(mv, Cols<D>{q, dq, ldi, i}, jm);
  const D v = manip_one(mv, jm, P);
  if (w) w[i] = v.value;
  if (dw) dw[i] = v.tangent;
}

template <class V>
int launch_manip_jvp_view(const V& mv, const Launch& L, const void* q, const void* dq, const TaskShared& P, void* w,
                          void* dw) {
  using T = typename V::Real;
  k_manip_jvp<JView<V>><<<grid_for(L.N), kBlock, 0, stream_of(L)>>>(JView<V>{mv}, L.N, (const T*)q, (const T*)dq,
                                                                     L.ld_in, P, (T*)w, (T*)dw);
  return (int)cudaGetLastError();
}

template <class V>
int launch_jvp_view(const V& mv, const Launch& L, const JvpArgs& a) {
  const JView<V> jv{mv};
  const dim3 grid(grid_for(L.N));
  switch (a.op) {
    case kJvpFK: k_jvp<JView<V>, kJvpFK><<<grid, kBlock, 0, stream_of(L)>>>(jv, L.N, a, L.ld_in, L.ld_out); break;
    case kJvpRNEA: k_jvp<JView<V>, kJvpRNEA><<<grid, kBlock, 0, stream_of(L)>>>(jv, L.N, a, L.ld_in, L.ld_out); break;
    case kJvpCRBA: k_jvp<JView<V>, kJvpCRBA><<<grid, kBlock, 0, stream_of(L)>>>(jv, L.N, a, L.ld_in, L.ld_out); break;
    default: k_jvp<JView<V>, kJvpABA><<<grid, kBlock, 0, stream_of(L)>>>(jv, L.N, a, L.ld_in, L.ld_out); break;
  }
  return (int)cudaGetLastError();
}

}  // namespace vdk
