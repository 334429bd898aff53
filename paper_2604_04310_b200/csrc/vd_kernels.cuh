// sm_100a kernels (templates; instantiated per model view in vd_inst_*.cu): one thread per robot state, SoA coalesced loads/stores,
// model either compile-time specialised (generated robot tables) or read from
// a device-resident DevModel (generic trees).  See DESIGN.md.
#pragma once

#include <cuda_runtime.h>

#include "vd_algos.cuh"
#include "vd_launch.hpp"
#include "vd_robots_gen.cuh"
#include "vd_tma.cuh"

namespace vdk {

constexpr int kBlock = 128;

template <class T>
struct G3 {
  T g[3];
};
// a_g of state i from the gravity planes (Launch::gravity_planes)
template <class T>
__device__ __forceinline__ G3<T> per_state_gravity(const T* __restrict__ gpl, int64_t ld, int64_t i) {
  return G3<T>{{gpl[i], gpl[ld + i], gpl[2 * ld + i]}};
}

template <bool kFastTrig = false, class V, class A>
__device__ __forceinline__ void load_motion(const V& mv, const A& q, JM<typename V::S>* jm) {
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) jm[j] = joint_motion<V, typename V::Real, kFastTrig>(mv, j, q[j]);
}

template <class T>
__device__ __forceinline__ Cols<T> cols(const T* p, int64_t ld, int64_t i) {
  return Cols<T>{p, ld, i};
}

// ---------------------------------------------------------------- FK
template <class V, class A>
__device__ __forceinline__ void fk_body(const V& mv, const A& q, int64_t i, typename V::Real* out, int64_t ldo) {
  using T = typename V::Real;
  using S = typename V::S;
  JM<S> jm[V::kMax];
  load_motion(mv, q, jm);
  WX<S> W[V::kMax];
  fk_world(mv, jm, W);
  OutCols<T> o{out, ldo, i};
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int r = 0; r < 3; ++r) o.put(j * 12 + c * 3 + r, W[j].R[r * 3 + c].v);
#pragma unroll
    for (int r = 0; r < 3; ++r) o.put(j * 12 + 9 + r, W[j].p[r].v);
  }
}
template <class V>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_fk(const __grid_constant__ V mv, int64_t N,
                                                              const typename V::Real* __restrict__ q, int64_t ldi,
                                                              typename V::Real* __restrict__ out, int64_t ldo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  fk_body(mv, cols(q, ldi, i), i, out, ldo);
}

// ---------------------------------------------------------------- frame pose + Jacobian
struct FrameArg {
  int joint;
  double R[9], p[3];  // row-major offset
};
template <class V, class A>
__device__ __forceinline__ void jac_body(const V& mv, const A& q, int64_t i, const FrameArg& fr,
                                         typename V::Real* pose, typename V::Real* J, int64_t ldo) {
  using T = typename V::Real;
  using S = typename V::S;
  JM<S> jm[V::kMax];
  load_motion(mv, q, jm);
  WX<S> W[V::kMax];
  fk_world(mv, jm, W);
  // frame_transform (kinematics.hpp:89-96)
  T WR[9], Wp[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) WR[k] = (k % 4 == 0) ? T(1) : T(0);
#pragma unroll
  for (int k = 0; k < 3; ++k) Wp[k] = T(0);
#pragma unroll
  for (int j = 0; j < mv.n(); ++j)
    if (j == fr.joint) {
#pragma unroll
      for (int k = 0; k < 9; ++k) WR[k] = W[j].R[k].v;
#pragma unroll
      for (int k = 0; k < 3; ++k) Wp[k] = W[j].p[k].v;
    }
  T PR[9], Pp[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      PR[r * 3 + c] = WR[r * 3] * T(fr.R[c]) + WR[r * 3 + 1] * T(fr.R[3 + c]) + WR[r * 3 + 2] * T(fr.R[6 + c]);
    Pp[r] = WR[r * 3] * T(fr.p[0]) + WR[r * 3 + 1] * T(fr.p[1]) + WR[r * 3 + 2] * T(fr.p[2]) + Wp[r];
  }
  if (pose) {
    OutCols<T> o{pose, ldo, i};
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int r = 0; r < 3; ++r) o.put(c * 3 + r, PR[r * 3 + c]);
#pragma unroll
    for (int r = 0; r < 3; ++r) o.put(9 + r, Pp[r]);
  }
  if (J) {
    // geometric_jacobian (kinematics.hpp:108-129); zero columns off the path.
    OutCols<T> o{J, ldo, i};
    const uint64_t mask = fr.joint >= 0 ? mv.anc(fr.joint) : 0ull;
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) {
      T col[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
      if ((mask >> j) & 1ull) {
        T ax[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
          ax[r] = (W[j].R[r * 3] * mv.axis(j, 0) + W[j].R[r * 3 + 1] * mv.axis(j, 1) + W[j].R[r * 3 + 2] * mv.axis(j, 2)).v;
        if (mv.kind(j) == 0) {
          const T d[3] = {Pp[0] - W[j].p[0].v, Pp[1] - W[j].p[1].v, Pp[2] - W[j].p[2].v};
          col[0] = ax[0];
          col[1] = ax[1];
          col[2] = ax[2];
          col[3] = ax[1] * d[2] - ax[2] * d[1];
          col[4] = ax[2] * d[0] - ax[0] * d[2];
          col[5] = ax[0] * d[1] - ax[1] * d[0];
        } else {
          col[3] = ax[0];
          col[4] = ax[1];
          col[5] = ax[2];
        }
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) o.put(j * 6 + r, col[r]);
    }
  }
}
template <class V>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_jac(const __grid_constant__ V mv, int64_t N,
                                                               const typename V::Real* __restrict__ q, int64_t ldi,
                                                               FrameArg fr, typename V::Real* __restrict__ pose,
                                                               typename V::Real* __restrict__ J, int64_t ldo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  jac_body(mv, cols(q, ldi, i), i, fr, pose, J, ldo);
}

// ---------------------------------------------------------------- RNEA family
template <class V, bool kFext>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_rnea(const __grid_constant__ V mv, int64_t N, const typename V::Real* __restrict__ q,
                                                  const typename V::Real* __restrict__ qd,
                                                  const typename V::Real* __restrict__ qdd, int64_t ldi,
                                                  G3<typename V::Real> g, const typename V::Real* __restrict__ fext,
                                                  typename V::Real* __restrict__ tau, int64_t ldo,
                                                  const typename V::Real* __restrict__ gpl) {
  using T = typename V::Real;
  using S = typename V::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (gpl) g = per_state_gravity(gpl, ldi, i);
  JM<S> jm[V::kMax];
  load_motion(mv, cols(q, ldi, i), jm);
  const Cols<T> qdc{qd, ldi, i}, qddc{qdd, ldi, i}, fc{fext, ldi, i};
  S out[V::kMax];
  rnea_one<V, kFext>(mv, jm, qdc, qdd ? &qddc : static_cast<const Cols<T>*>(nullptr), g.g, &fc, out);
  OutCols<T> o{tau, ldo, i};
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) o.put(j, out[j].v);
}

// ---------------------------------------------------------------- CRBA
template <class V>
__device__ __forceinline__ void store_mass(const V& mv, const JM<typename V::S>* jm, typename V::Real* M, int64_t ldo,
                                           int64_t i) {
  using T = typename V::Real;
  using S = typename V::S;
  OutCols<T> o{M, ldo, i};
  const int n = mv.n();
  crba_one(mv, jm, [&](int r, int c, const S& val) {
    o.put(c * n + r, val.v);
    if (r != c) o.put(r * n + c, val.v);
  });
  // exact zeros between branches (dynamics.hpp:331-335, test_dynamics.cpp:200-216)
#pragma unroll
  for (int r = 0; r < mv.n(); ++r)
#pragma unroll
    for (int c = 0; c < mv.n(); ++c)
      if (!((mv.anc(r) >> c) & 1ull) && !((mv.anc(c) >> r) & 1ull)) o.put(c * n + r, T(0));
}
template <class V>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_crba(const __grid_constant__ V mv, int64_t N, const typename V::Real* __restrict__ q, int64_t ldi,
                                                  typename V::Real* __restrict__ M, int64_t ldo) {
  using S = typename V::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  JM<S> jm[V::kMax];
  load_motion(mv, cols(q, ldi, i), jm);
  store_mass(mv, jm, M, ldo, i);
}

// ---------------------------------------------------------------- ABA
template <class V, bool kFext>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_aba(const __grid_constant__ V mv, int64_t N, const typename V::Real* __restrict__ q,
                                                 const typename V::Real* __restrict__ qd,
                                                 const typename V::Real* __restrict__ tau, int64_t ldi,
                                                 G3<typename V::Real> g, const typename V::Real* __restrict__ fext,
                                                 typename V::Real* __restrict__ qdd, int64_t ldo,
                                                 int32_t* __restrict__ status, const typename V::Real* __restrict__ gpl) {
  using T = typename V::Real;
  using S = typename V::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (gpl) g = per_state_gravity(gpl, ldi, i);
  JM<S> jm[V::kMax];
  load_motion(mv, cols(q, ldi, i), jm);
  const Cols<T> qdc{qd, ldi, i}, tc{tau, ldi, i}, fc{fext, ldi, i};
  S out[V::kMax];
  bool ok;
  if constexpr (V::kStatic) {
    ok = aba_one<V, kFext>(mv, jm, qdc, tc, g.g, &fc, out);
  } else {
    T qdl[V::kMax], taul[V::kMax];
    for (int j = 0; j < mv.n(); ++j) {
      qdl[j] = qdc[j];
      taul[j] = tc[j];
    }
    ok = aba_one<V, kFext>(mv, jm, Row<T>{qdl}, Row<T>{taul}, g.g, &fc, out);
  }
  OutCols<T> o{qdd, ldo, i};
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) o.put(j, ok ? out[j].v : T(0));
  if (status) status[i] = ok ? 0 : 7;
}

// ---------------------------------------------------------------- fused M + bias + q̈ (config 3)
template <class V, class A>
__device__ __forceinline__ void dyn_body(const V& mv, const A& q, const A& qd, const A& tau, int64_t i,
                                         const G3<typename V::Real>& g, typename V::Real* M, typename V::Real* bias,
                                         typename V::Real* qdd, int64_t ldo, int32_t* status) {
  using T = typename V::Real;
  using S = typename V::S;
  JM<S> jm[V::kMax];
  load_motion(mv, q, jm);
  if (M) store_mass(mv, jm, M, ldo, i);
  if (bias) {
    S b[V::kMax];
    rnea_one<V, false>(mv, jm, qd, static_cast<const A*>(nullptr), g.g, nullptr, b);
    OutCols<T> o{bias, ldo, i};
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) o.put(j, b[j].v);
  }
  if (qdd) {
    S a[V::kMax];
    const bool ok = aba_one<V, false>(mv, jm, qd, tau, g.g, nullptr, a);
    OutCols<T> o{qdd, ldo, i};
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) o.put(j, ok ? a[j].v : T(0));
    if (status) status[i] = ok ? 0 : 7;
  }
}
template <class V>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_dyn(const __grid_constant__ V mv, int64_t N,
                                                               const typename V::Real* __restrict__ q,
                                                               const typename V::Real* __restrict__ qd,
                                                               const typename V::Real* __restrict__ tau, int64_t ldi,
                                                               G3<typename V::Real> g, typename V::Real* __restrict__ M,
                                                               typename V::Real* __restrict__ bias,
                                                               typename V::Real* __restrict__ qdd, int64_t ldo,
                                                               int32_t* __restrict__ status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  dyn_body(mv, cols(q, ldi, i), cols(qd, ldi, i), cols(tau, ldi, i), i, g, M, bias, qdd, ldo, status);
}

// ---------------------------------------------------------------- OSC
template <class V, class A>
__device__ __forceinline__ void osc_body(const V& mv, const A& q, const A& qd, int64_t i, const OscShared& P,
                                         typename V::Real* tau, typename V::Real* lam, int64_t ldo,
                                         int32_t* status) {
  using T = typename V::Real;
  using S = typename V::S;
  JM<S> jm[V::kMax];
  load_motion(mv, q, jm);
  T t[V::kMax], L[36];
  const bool ok = osc_one(mv, jm, q, qd, P, t, lam ? L : nullptr);
  OutCols<T> o{tau, ldo, i};
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) o.put(j, ok ? t[j] : T(0));
  if (lam) {
    OutCols<T> ol{lam, ldo, i};
#pragma unroll
    for (int k = 0; k < 36; ++k) ol.put(k, ok ? L[k] : T(0));
  }
  if (status) status[i] = ok ? 0 : 7;
}
template <class V>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_osc(const __grid_constant__ V mv, int64_t N,
                                                               const typename V::Real* __restrict__ q,
                                                               const typename V::Real* __restrict__ qd, int64_t ldi,
                                                               OscShared P, typename V::Real* __restrict__ tau,
                                                               typename V::Real* __restrict__ lam, int64_t ldo,
                                                               int32_t* __restrict__ status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  osc_body(mv, cols(q, ldi, i), cols(qd, ldi, i), i, P, tau, lam, ldo, status);
}

// ---------------------------------------------------------------- task-space kinematics
// mode 0: diff_ik_step → out = q̇ (n rows), aux = pose error (6 rows, optional)
// mode 1: manipulability → out = w (1 row)
template <class V>
__global__ void __launch_bounds__(kBlock, V::kMinBlocks) k_task(const __grid_constant__ V mv, int64_t N,
                                                                const typename V::Real* __restrict__ q, int64_t ldi,
                                                                const __grid_constant__ TaskShared P, int mode,
                                                                typename V::Real* __restrict__ out,
                                                                typename V::Real* __restrict__ aux, int64_t ldo,
                                                                int32_t* __restrict__ status) {
  using T = typename V::Real;
  using S = typename V::S;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  JM<S> jm[V::kMax];
  load_motion(mv, cols(q, ldi, i), jm);
  if (mode == 0) {
    T qd[V::kMax], err[6];
    const bool ok = diffik_one(mv, jm, P, qd, aux ? err : nullptr);
    OutCols<T> o{out, ldo, i};
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) o.put(j, ok ? qd[j] : T(0));
    if (aux) {
      OutCols<T> oe{aux, ldo, i};
#pragma unroll
      for (int r = 0; r < 6; ++r) oe.put(r, err[r]);
    }
    if (status) status[i] = ok ? 0 : 7;
  } else {
    out[i] = manip_one(mv, jm, P);
  }
}

// ---------------------------------------------------------------- TMA-staged persistent driver (static views)
// Same math as the plain kernels; inputs arrive through the two-stage
// bulk-copy pipeline of vd_tma.cuh.  Requires 16-byte aligned planes (checked
// on the host) and 2 stages x Op::kGroups x n planes x kBlock of shared memory.
template <class V, class Op>
__global__ void __launch_bounds__(kBlock, Op::kMinBlocks) k_tiled(const __grid_constant__ V mv,
                                                                 const __grid_constant__ Op op, int64_t N,
                                                                 tma::Inputs<typename V::Real> in, int64_t ldi,
                                                                 bool use_tma) {
  using T = typename V::Real;
  constexpr int n = V::kMax;
  constexpr int G = Op::kGroups;
  __shared__ __align__(128) T buf[2][G * n * kBlock];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  // tiles [0, full) arrive by TMA; any other tile (the N % kBlock tail, or all
  // of them when the planes are not 16-byte aligned) is staged with plain loads
  const int64_t full = use_tma ? N / kBlock : 0;
  if (tid == 0) {
    tma::mbar_init(&bar[0], 1);
    tma::mbar_init(&bar[1], 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  const int64_t t0 = blockIdx.x, step = gridDim.x;
  if (tid == 0) {
    if (t0 < full) tma::issue_tile<T, kBlock>(buf[0], in, n, ldi, t0, &bar[0]);
    if (t0 + step < full) tma::issue_tile<T, kBlock>(buf[1], in, n, ldi, t0 + step, &bar[1]);
  }
  // The N % kBlock tail is the globally last tile: the CTA that reaches it
  // stages it with plain loads and runs the SAME call site, so every
  // instance is computed by identical instructions (results do not depend on
  // where an instance falls in the batch).
  const int64_t tiles = (N + kBlock - 1) / kBlock;
  int it = 0;
  for (int64_t t = t0; t < tiles; t += step, ++it) {
    const int st = it & 1;
    const int64_t i = t * kBlock + tid;
    if (t < full) {
      tma::mbar_wait(&bar[st], (it >> 1) & 1);
    } else {
      for (int gk = 0; gk < G * n; ++gk) {
        const int g = gk / n, k = gk - g * n;
        buf[st][gk * kBlock + tid] = i < N ? in.p[g][(int64_t)k * ldi + i] : T(0);
      }
    }
    const T* b = buf[st] + tid;
    if (i < N)
      op.run(mv, SmemRow<T, kBlock>{b}, SmemRow<T, kBlock>{b + (G > 1 ? n : 0) * kBlock},
             SmemRow<T, kBlock>{b + (G > 2 ? 2 * n : 0) * kBlock}, i);
    __syncthreads();  // every thread is done reading stage st
    if (tid == 0 && t + 2 * step < full) {
      tma::fence_proxy_async();
      tma::issue_tile<T, kBlock>(buf[st], in, n, ldi, t + 2 * step, &bar[st]);
    }
  }
}

template <class T>
struct OpABA {
  static constexpr int kMinBlocks = 3;
  static constexpr bool kEnabled = true;
  static constexpr int kGroups = 3;
  G3<T> g;
  T* qdd;
  int64_t ldo;
  int32_t* status;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A& qd, const A& tau, int64_t i) const {
    using S = typename V::S;
    JM<S> jm[V::kMax];
    load_motion<true>(mv, q, jm);
    S out[V::kMax];
    const bool ok = aba_one<V, false>(mv, jm, qd, tau, g.g, nullptr, out);
    OutCols<T> o{qdd, ldo, i};
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) o.put(j, ok ? out[j].v : T(0));
    if (status) status[i] = ok ? 0 : 7;
  }
};
// G = 3: rnea(q, qd, qdd); G = 2: qdd = 0 (bias / coriolis); G = 1: qd = qdd = 0 (gravity)
template <class T, int G>
struct OpRNEA {
  static constexpr int kMinBlocks = 0;
  static constexpr bool kEnabled = true;
  static constexpr int kGroups = G;
  G3<T> g;
  T* tau;
  int64_t ldo;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A& qd, const A& qdd, int64_t i) const {
    using S = typename V::S;
    JM<S> jm[V::kMax];
    load_motion(mv, q, jm);
    S out[V::kMax];
    if constexpr (G == 3) {
      rnea_one<V, false>(mv, jm, qd, &qdd, g.g, nullptr, out);
    } else if constexpr (G == 2) {
      rnea_one<V, false>(mv, jm, qd, static_cast<const A*>(nullptr), g.g, nullptr, out);
    } else {
      const Cols<T> zero{nullptr, 0, 0};
      rnea_one<V, false>(mv, jm, zero, static_cast<const Cols<T>*>(nullptr), g.g, nullptr, out);
    }
    OutCols<T> o{tau, ldo, i};
#pragma unroll
    for (int j = 0; j < mv.n(); ++j) o.put(j, out[j].v);
  }
};
template <class T>
struct OpCRBA {
  static constexpr int kMinBlocks = 0;
  static constexpr bool kEnabled = true;
  static constexpr int kGroups = 1;
  T* M;
  int64_t ldo;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A&, const A&, int64_t i) const {
    JM<typename V::S> jm[V::kMax];
    load_motion(mv, q, jm);
    store_mass(mv, jm, M, ldo, i);
  }
};
template <class T>
struct OpFK {
  static constexpr int kMinBlocks = 0;
  static constexpr bool kEnabled = true;
  static constexpr int kGroups = 1;
  T* out;
  int64_t ldo;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A&, const A&, int64_t i) const {
    fk_body(mv, q, i, out, ldo);
  }
};
template <class T>
struct OpJac {
  static constexpr int kMinBlocks = 0;
  static constexpr bool kEnabled = false;
  static constexpr int kGroups = 1;
  FrameArg fr;
  T* pose;
  T* J;
  int64_t ldo;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A&, const A&, int64_t i) const {
    jac_body(mv, q, i, fr, pose, J, ldo);
  }
};
template <class T>
struct OpDyn {
  static constexpr int kMinBlocks = 3;
  static constexpr bool kEnabled = true;
  static constexpr int kGroups = 3;
  G3<T> g;
  T *M, *bias, *qdd;
  int64_t ldo;
  int32_t* status;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A& qd, const A& tau, int64_t i) const {
    dyn_body(mv, q, qd, tau, i, g, M, bias, qdd, ldo, status);
  }
};
template <class T>
struct OpOSC {
  static constexpr int kMinBlocks = 0;
  static constexpr bool kEnabled = false;
  static constexpr int kGroups = 2;
  OscShared P;
  T *tau, *lam;
  int64_t ldo;
  int32_t* status;
  template <class V, class A>
  __device__ __forceinline__ void run(const V& mv, const A& q, const A& qd, const A&, int64_t i) const {
    osc_body(mv, q, qd, i, P, tau, lam, ldo, status);
  }
};

// ================================================================ per-view launchers
inline unsigned grid_for(int64_t N) { return (unsigned)((N + kBlock - 1) / kBlock); }
inline cudaStream_t stream_of(const Launch& L) { return static_cast<cudaStream_t>(L.stream); }
template <class T>
inline G3<T> g3_of(const double* g) {
  G3<T> o;
  for (int k = 0; k < 3; ++k) o.g[k] = g ? T(g[k]) : (k == 2 ? T(9.81) : T(0));
  return o;
}

// Launcher<V> is explicitly instantiated per view (and per member for the
// large tree29 kernels) in vd_inst_*.cu so the build parallelises.
template <class V>
struct Launcher {
  using T = typename V::Real;
  static int fk(const V& mv, const Launch& L, const void* q, void* out);
  static int jac(const V& mv, const Launch& L, const void* q, const FrameArg& fr, void* pose, void* J);
  static int rnea(const V& mv, const Launch& L, const void* q, const void* qd, const void* qdd, const double* g,
                  const void* fext, void* tau);
  static int crba(const V& mv, const Launch& L, const void* q, void* M);
  static int aba(const V& mv, const Launch& L, const void* q, const void* qd, const void* tau, const double* g,
                 const void* fext, void* qdd, int32_t* status);
  static int dyn(const V& mv, const Launch& L, const void* q, const void* qd, const void* tau, const double* g, void* M,
                 void* bias, void* qdd, int32_t* status);
  static int osc(const V& mv, const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau,
                 void* lambda, int32_t* status);
  static int task(const V& mv, const Launch& L, const void* q, const TaskShared& P, int mode, void* out, void* aux,
                  int32_t* status);
};

using GenericD = RuntimeView<double>;
using GenericF = RuntimeView<float>;
using Chain7D = StaticView<RobotChain7, double>;
using Chain7F = StaticView<RobotChain7, float>;
using Tree29D = StaticView<RobotTree29, double>;
using Tree29F = StaticView<RobotTree29, float>;

}  // namespace vdk
