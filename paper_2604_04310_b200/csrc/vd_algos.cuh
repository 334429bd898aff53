// Per-instance rigid-body algorithms (one thread = one robot state), written
// once against a model view (vd_device.cuh).  Each function cites the
// reference routine whose semantics it reproduces.
#pragma once

#include "vd_device.cuh"

namespace vdk {

// SoA column-major access: element (instance i, component k) at k*ld + i.
template <class T>
struct Cols {
  const T* __restrict__ base;
  int64_t ld, i;
  __device__ __forceinline__ T operator[](int k) const { return base ? __ldg(base + (int64_t)k * ld + i) : T(0); }
};
// A per-thread copy of an input row (loop kernels preload their inputs so the
// n independent global loads are all in flight at once).
template <class T>
struct Row {
  const T* v;
  __device__ __forceinline__ T operator[](int k) const { return v[k]; }
};
template <class T>
struct OutCols {
  T* __restrict__ base;
  int64_t ld, i;
  __device__ __forceinline__ void put(int k, T v) const { base[(int64_t)k * ld + i] = v; }
};

template <class V>
__device__ __forceinline__ SV<typename V::S> gravity_accel(const typename V::Real* g3) {
  using S = typename V::S;
  SV<S> a;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    a.a[k] = S();
    a.l[k] = S(g3[k]);
  }
  return a;
}

// ------------------------------------------------------------------ FK
// forward_kinematics (kinematics.hpp:43-56) — world pose of every joint.
template <class V>
__device__ __forceinline__ void fk_world(const V& mv, const JM<typename V::S>* jm, WX<typename V::S>* W) {
#pragma unroll
  for (int i = 0; i < mv.n(); ++i) {
    JointX<V> x;
    x.load(mv, i, jm[i]);
    const int p = mv.parent(i);
    W[i] = world_of(x, p < 0 ? nullptr : &W[p]);
  }
}

// ------------------------------------------------------------------ RNEA
// rnea_loop (dynamics.hpp:272-327): two-pass recursion in local coordinates.
// qdd == nullptr means q̈ = 0 (bias forces, dynamics.hpp:434-435).
template <class V, bool kFext, class QdA, class QddA>
__device__ __forceinline__ void rnea_one(const V& mv, const JM<typename V::S>* jm, const QdA& qd, const QddA* qdd,
                                         const typename V::Real* g3, const Cols<typename V::Real>* fext,
                                         typename V::S* tau) {
  using S = typename V::S;
  SV<S> v[V::kMax], a[V::kMax], f[V::kMax];
  WX<S> W[kFext ? V::kMax : 1];
  const SV<S> ag = gravity_accel<V>(g3);
#pragma unroll
  for (int i = 0; i < mv.n(); ++i) {
    JointX<V> x;
    x.load(mv, i, jm[i]);
    const JAxis<V> ax(mv, i);
    const int p = mv.parent(i);
    const S qdi = S(qd[i]);
    if (p < 0) {
      v[i] = ax.scaled(qdi);
      a[i] = x.motion_to_child(ag);
    } else {
      v[i] = x.motion_to_child(v[p]);
      ax.add(v[i], qdi);
      a[i] = x.motion_to_child(a[p]) + ax.crm(v[i], qdi);
    }
    if (qdd) ax.add(a[i], S((*qdd)[i]));
    if (mv.oflags(i) & kMassless) {
#pragma unroll
      for (int k = 0; k < 3; ++k) f[i].a[k] = f[i].l[k] = S();
    } else {
      const RB<S> I = body_inertia(mv, i);
      f[i] = rb_apply(I, a[i]) + crf(v[i], rb_apply(I, v[i]));
    }
    if constexpr (kFext) {
      W[i] = world_of(x, p < 0 ? nullptr : &W[p]);
      SV<S> fw;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        fw.a[k] = S((*fext)[i * 6 + k]);
        fw.l[k] = S((*fext)[i * 6 + 3 + k]);
      }
      f[i] = f[i] - force_in(W[i].R, W[i].p, true, fw);
    }
  }
#pragma unroll
  for (int i = mv.n() - 1; i >= 0; --i) {
    tau[i] = JAxis<V>(mv, i).dot(f[i]);
    const int p = mv.parent(i);
    if (p >= 0) {
      JointX<V> x;
      x.load(mv, i, jm[i]);
      f[p] = f[p] + x.force_to_parent(f[i]);
    }
  }
}

// ------------------------------------------------------------------ CRBA
// crba_loop (dynamics.hpp:369-400): composite inertias leaf -> root, then
// one force propagation up the ancestor chain per column.  emit(i, j, value)
// receives M(i, j) for j = i and every ancestor j of i.
template <class V, class Emit>
__device__ __forceinline__ void crba_one(const V& mv, const JM<typename V::S>* jm, Emit&& emit) {
  using S = typename V::S;
  RB<S> ic[V::kMax];
#pragma unroll
  for (int i = 0; i < mv.n(); ++i) ic[i] = body_inertia(mv, i);
#pragma unroll
  for (int i = mv.n() - 1; i >= 0; --i) {
    const int p = mv.parent(i);
    if (p >= 0) {
      JointX<V> x;
      x.load(mv, i, jm[i]);
      rb_add(ic[p], rb_to_parent(x, ic[i]));
    }
  }
#pragma unroll
  for (int i = 0; i < mv.n(); ++i) {
    const JAxis<V> ax(mv, i);
    SV<S> F = rb_apply(ic[i], ax.scaled(S(typename V::Real(1), true)));
    emit(i, i, ax.dot(F));
    int j = i;
#pragma unroll
    for (int d = 1; d < mv.max_depth(); ++d) {
      if (d >= mv.depth(i)) break;
      JointX<V> x;
      x.load(mv, j, jm[j]);
      F = x.force_to_parent(F);
      j = mv.parent(j);
      emit(i, j, JAxis<V>(mv, j).dot(F));
    }
  }
}

// ------------------------------------------------------------------ plain storage
// Per-joint values that are always runtime numbers are stored without the sp
// flag: when such an array spills to local memory under a compile-time view,
// a stored flag would become a runtime value and every select built on it
// would survive to SASS.  Loading rebuilds a "non-zero" sp.
template <class S>
struct PV {  // plain spatial vector
  decltype(S::v) a[3], l[3];
  __device__ __forceinline__ void set(const SV<S>& x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      a[k] = x.a[k].v;
      l[k] = x.l[k].v;
    }
  }
  __device__ __forceinline__ SV<S> get() const {
    SV<S> x;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      x.a[k] = S(a[k]);
      x.l[k] = S(l[k]);
    }
    return x;
  }
};
template <class S>
struct PI {  // plain articulated inertia
  decltype(S::v) A[6], B[9], C[6];
  __device__ __forceinline__ void set(const AI<S>& x) {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      A[k] = x.A[k].v;
      C[k] = x.C[k].v;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) B[k] = x.B[k].v;
  }
  __device__ __forceinline__ AI<S> get() const {
    AI<S> x;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      x.A[k] = S(A[k]);
      x.C[k] = S(C[k]);
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) x.B[k] = S(B[k]);
    return x;
  }
};

// ------------------------------------------------------------------ ABA
// Articulated-body forward dynamics (Featherstone RBDA Table 7.1).  Not in the
// reference; its oracle is forward_dynamics (dynamics.hpp:421-444,
// CRBA + bias + LLT).  Returns false when an articulated pivot D_i is not
// positive (the LLT failure of the oracle: the D_i are the pivots of M's
// tree-structured LDLᵀ factorisation) or the result is not finite.
//
// State is kept small so the large-tree kernels stay in L1/L2 and the chain
// kernels stay in registers:
//  * joints are in DFS order, so a non-leaf joint i always has child i+1:
//    contributions to the parent travel in a register "carry" when
//    parent(j) == j-1 and only go through per-joint slots at branch points;
//  * velocities are stored only at leaves and branch joints in pass 1; pass 2
//    (leaf -> root) reconstructs v_{i-1} = X_i (v_i − S_i q̇_i) from its child,
//    pass 3 recomputes them root -> leaf;
//  * the per-joint state carried from pass 2 to pass 3 is U_i, u_i, 1/D_i.
template <class V, bool kFext, class QdAcc, class TauAcc>
__device__ __forceinline__ bool aba_one(const V& mv, const JM<typename V::S>* jm, const QdAcc& qd, const TauAcc& tau,
                                        const typename V::Real* g3, const Cols<typename V::Real>* fext,
                                        typename V::S* qdd) {
  using S = typename V::S;
  using T = typename V::Real;
  constexpr int NM = V::kMax;
  PV<S> U[NM], vkeep[NM];
  T u[NM], dinv[NM];
  SV<S> fl[kFext ? NM : 1];
  WX<S> W[kFext ? NM : 1];
  bool ok = true;
  SV<S> zero;
#pragma unroll
  for (int k = 0; k < 3; ++k) zero.a[k] = zero.l[k] = S();

  // pass 1: velocities root -> leaf (kept at leaves / branch joints)
  {
    SV<S> vprev = zero;
#pragma unroll
    for (int i = 0; i < mv.n(); ++i) {
      JointX<V> x;
      x.load(mv, i, jm[i]);
      const int p = mv.parent(i);
      const JAxis<V> ax(mv, i);
      SV<S> v;
      if (p >= 0) {
        v = x.motion_to_child(p == i - 1 ? vprev : vkeep[p].get());
        ax.add(v, S(qd[i]));
      } else {
        v = ax.scaled(S(qd[i]));
      }
      if (mv.flags(i) & (kFlagLeaf | kFlagBranch)) vkeep[i].set(v);
      vprev = v;
      if constexpr (kFext) {
        W[i] = world_of(x, p < 0 ? nullptr : &W[p]);
        SV<S> fw;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          fw.a[k] = S((*fext)[i * 6 + k]);
          fw.l[k] = S((*fext)[i * 6 + 3 + k]);
        }
        fl[i] = force_in(W[i].R, W[i].p, true, fw);
      }
    }
  }
  // pass 2: articulated inertias leaf -> root
  {
    AI<S> carryI;
    PI<S> slotI[NM];
    SV<S> carryP = zero, vrec = zero;
    PV<S> slotP[NM];
    uint64_t used = 0;
    int carry_to = -1;
#pragma unroll
    for (int i = mv.n() - 1; i >= 0; --i) {
      const JAxis<V> ax(mv, i);
      const S qdi = S(qd[i]);
      const SV<S> v = (mv.flags(i) & kFlagLeaf) ? vkeep[i].get() : vrec;
      AI<S> IA;
      SV<S> pA;
      if (mv.oflags(i) & kMassless) {
#pragma unroll
        for (int k = 0; k < 6; ++k) IA.A[k] = IA.C[k] = S();
#pragma unroll
        for (int k = 0; k < 9; ++k) IA.B[k] = S();
        pA = zero;
      } else {
        const RB<S> I = body_inertia(mv, i);
        IA = ai_from_rb(I);
        pA = crf(v, rb_apply(I, v));
      }
      if constexpr (kFext) pA = pA - fl[i];
      if (carry_to == i) {
        ai_add(IA, carryI);
        pA = pA + carryP;
      }
      if ((used >> i) & 1ull) {
        ai_add(IA, slotI[i].get());
        pA = pA + slotP[i].get();
      }
      const SV<S> Ui = ai_axis(ax, IA);
      U[i].set(Ui);
      const S D = ax.dot(Ui);
      ok = ok && (D.v > T(0));
      const S di = S(T(1) / D.v);
      const S ui = S(tau[i]) - ax.dot(pA);
      dinv[i] = di.v;
      u[i] = ui.v;
      const int p = mv.parent(i);
      if (p >= 0) {
        JointX<V> x;
        x.load(mv, i, jm[i]);
        const SV<S> c = ax.crm(v, qdi);
        AI<S> Ia = IA;
        ai_sub_outer(Ia, Ui, di);
        const SV<S> pa = pA + ai_apply(Ia, c) + scale(Ui, ui * di);
        const AI<S> IAp = ai_to_parent(x, Ia);
        const SV<S> pAp = x.force_to_parent(pa);
        if (p == i - 1) {
          carryI = IAp;
          carryP = pAp;
          carry_to = p;
          SV<S> vmj = v;
          ax.add(vmj, -qdi);
          vrec = x.motion_to_parent(vmj);  // v_{i-1}
        } else if ((used >> p) & 1ull) {
          AI<S> acc = slotI[p].get();
          ai_add(acc, IAp);
          slotI[p].set(acc);
          slotP[p].set(slotP[p].get() + pAp);
        } else {
          slotI[p].set(IAp);
          slotP[p].set(pAp);
          used |= 1ull << p;
        }
      }
    }
  }
  // pass 3: accelerations root -> leaf
  {
    const SV<S> ag = gravity_accel<V>(g3);
    SV<S> aprev = zero, vprev = zero;
    PV<S> akeep[NM];
#pragma unroll
    for (int i = 0; i < mv.n(); ++i) {
      JointX<V> x;
      x.load(mv, i, jm[i]);
      const int p = mv.parent(i);
      const JAxis<V> ax(mv, i);
      const S qdi = S(qd[i]);
      SV<S> v, ap;
      if (p < 0) {
        v = ax.scaled(qdi);
        ap = x.motion_to_child(ag);
      } else {
        const bool adj = p == i - 1;
        v = x.motion_to_child(adj ? vprev : vkeep[p].get());
        ax.add(v, qdi);
        ap = x.motion_to_child(adj ? aprev : akeep[p].get()) + ax.crm(v, qdi);
      }
      qdd[i] = (S(u[i]) - sdot(U[i].get(), ap)) * S(dinv[i]);
      ok = ok && isfinite(qdd[i].v);
      SV<S> a = ap;
      ax.add(a, qdd[i]);
      if (mv.flags(i) & kFlagBranch) akeep[i].set(a);
      aprev = a;
      vprev = v;
    }
  }
  return ok;
}

// ------------------------------------------------------------------ OSC helpers
// rotation_log (control.hpp:45-68), reference acos form and branches.
template <class T>
__device__ __forceinline__ void rotation_log(const T* R, T* w) {
  const T tr = R[0] + R[4] + R[8];
  const T anti[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  T ca = T(0.5) * (tr - T(1));
  ca = ca < T(-1) ? T(-1) : (ca > T(1) ? T(1) : ca);
  const T ang = acos(ca);
  const T pi = T(3.14159265358979323846);
  if (ang < T(1e-9)) {
#pragma unroll
    for (int k = 0; k < 3; ++k) w[k] = T(0.5) * anti[k];
    return;
  }
  if (ang > pi - T(1e-6)) {
    const T sd[3] = {T(0.5) * (R[0] + T(1)), T(0.5) * (R[4] + T(1)), T(0.5) * (R[8] + T(1))};
    int k = 0;
    if (sd[1] > sd[k]) k = 1;
    if (sd[2] > sd[k]) k = 2;
    T ax[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) ax[r] = (r == k) ? sd[k] : T(0.5) * R[r * 3 + k];
    const T inv = T(1) / sqrt(sd[k] > T(1e-12) ? sd[k] : T(1e-12));
#pragma unroll
    for (int r = 0; r < 3; ++r) ax[r] *= inv;
    const T nrm = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
#pragma unroll
    for (int r = 0; r < 3; ++r) ax[r] /= nrm;
    const T sgn = (anti[0] * ax[0] + anti[1] * ax[1] + anti[2] * ax[2]) < T(0) ? T(-1) : T(1);
#pragma unroll
    for (int r = 0; r < 3; ++r) w[r] = ang * sgn * ax[r];
    return;
  }
  const T f = T(0.5) * ang / sin(ang);
#pragma unroll
  for (int k = 0; k < 3; ++k) w[k] = f * anti[k];
}

// frame_transform + geometric_jacobian (kinematics.hpp:89-129) of frame
// (joint fj, offset R_f/p_f): world pose of the frame and the 6 x n Jacobian
// (angular rows first; exact zeros off the ancestor path).
template <class V>
__device__ __forceinline__ void frame_pose_jacobian(const V& mv, const JM<typename V::S>* jm, int fj,
                                                    const double* frame_R, const double* frame_p,
                                                    typename V::Real* pose_R, typename V::Real* pose_p,
                                                    typename V::Real (*J)[V::kMax]) {
  using S = typename V::S;
  using T = typename V::Real;
  WX<S> W[V::kMax];
  fk_world(mv, jm, W);
  T WR[9], Wp[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) WR[k] = (k % 4 == 0) ? T(1) : T(0);
#pragma unroll
  for (int k = 0; k < 3; ++k) Wp[k] = T(0);
  if (fj >= 0) {
#pragma unroll
    for (int i = 0; i < mv.n(); ++i)
      if (i == fj) {
#pragma unroll
        for (int k = 0; k < 9; ++k) WR[k] = W[i].R[k].v;
#pragma unroll
        for (int k = 0; k < 3; ++k) Wp[k] = W[i].p[k].v;
      }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      pose_R[r * 3 + c] =
          WR[r * 3] * T(frame_R[c]) + WR[r * 3 + 1] * T(frame_R[3 + c]) + WR[r * 3 + 2] * T(frame_R[6 + c]);
    pose_p[r] = WR[r * 3] * T(frame_p[0]) + WR[r * 3 + 1] * T(frame_p[1]) + WR[r * 3 + 2] * T(frame_p[2]) + Wp[r];
  }
  const uint64_t fmask = fj >= 0 ? mv.anc(fj) : 0ull;
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) {
    const bool on = (fmask >> j) & 1ull;
    T ax[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      ax[r] = (W[j].R[r * 3] * mv.axis(j, 0) + W[j].R[r * 3 + 1] * mv.axis(j, 1) + W[j].R[r * 3 + 2] * mv.axis(j, 2)).v;
    if (!on) {
#pragma unroll
      for (int r = 0; r < 6; ++r) J[r][j] = T(0);
    } else if (mv.kind(j) == 0) {
      const T d[3] = {pose_p[0] - W[j].p[0].v, pose_p[1] - W[j].p[1].v, pose_p[2] - W[j].p[2].v};
      J[0][j] = ax[0];
      J[1][j] = ax[1];
      J[2][j] = ax[2];
      J[3][j] = ax[1] * d[2] - ax[2] * d[1];
      J[4][j] = ax[2] * d[0] - ax[0] * d[2];
      J[5][j] = ax[0] * d[1] - ax[1] * d[0];
    } else {
      J[0][j] = J[1][j] = J[2][j] = T(0);
      J[3][j] = ax[0];
      J[4][j] = ax[1];
      J[5][j] = ax[2];
    }
  }
}

// pose_error (control.hpp:73-77): (log(R_t R_cᵀ), p_t − p_c); target R row-major.
template <class T>
__device__ __forceinline__ void pose_error(const double* target_R, const double* target_p, const T* pose_R,
                                           const T* pose_p, T* err) {
  T Rrel[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Rrel[r * 3 + c] = T(target_R[r * 3]) * pose_R[c * 3] + T(target_R[r * 3 + 1]) * pose_R[c * 3 + 1] +
                        T(target_R[r * 3 + 2]) * pose_R[c * 3 + 2];
  rotation_log(Rrel, err);
#pragma unroll
  for (int k = 0; k < 3; ++k) err[3 + k] = T(target_p[k]) - pose_p[k];
}

// In-place Cholesky of a 6x6 SPD (lower, row-major), Eigen's LLT criterion.
template <class T>
__device__ __forceinline__ bool chol6(T* L) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    T x = L[k * 6 + k];
#pragma unroll
    for (int j = 0; j < k; ++j) x -= L[k * 6 + j] * L[k * 6 + j];
    ok = ok && (x > T(0));
    x = sqrt(x);
    L[k * 6 + k] = x;
    const T inv = T(1) / x;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      T s = L[i * 6 + k];
#pragma unroll
      for (int j = 0; j < k; ++j) s -= L[i * 6 + j] * L[k * 6 + j];
      L[i * 6 + k] = s * inv;
    }
  }
  return ok;
}
template <class T>
__device__ __forceinline__ void chol6_solve(const T* L, T* b) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    T s = b[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s -= L[i * 6 + j] * b[j];
    b[i] = s / L[i * 6 + i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    T s = b[i];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) s -= L[j * 6 + i] * b[j];
    b[i] = s / L[i * 6 + i];
  }
}

// G = J Jᵀ + d·I, lower triangle, row-major 6x6.
template <class T, int NM>
__device__ __forceinline__ void gram6(int n, const T (*J)[NM], T d, T* G) {
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      T s = r == c ? d : T(0);
#pragma unroll
      for (int k = 0; k < n; ++k) s += J[r][k] * J[c][k];
      G[r * 6 + c] = s;
    }
}

// diff_ik_step (control.hpp:79-97): q̇ = Jᵀ (J Jᵀ + λ² I)⁻¹ (kp ⊙ err + twist_ff).
// Returns false when the damped Gram matrix does not factor (non-finite input).
template <class V>
__device__ __forceinline__ bool diffik_one(const V& mv, const JM<typename V::S>* jm, const TaskShared& P,
                                           typename V::Real* qdot, typename V::Real* err_out) {
  using T = typename V::Real;
  constexpr int NM = V::kMax;
  T pose_R[9], pose_p[3], J[6][NM];
  frame_pose_jacobian(mv, jm, P.frame_joint, P.frame_R, P.frame_p, pose_R, pose_p, J);
  T err[6];
  pose_error(P.target_R, P.target_p, pose_R, pose_p, err);
  T rhs[6], G[36];
#pragma unroll
  for (int r = 0; r < 6; ++r) rhs[r] = T(P.kp[r]) * err[r] + T(P.twist_ff[r]);
  gram6(mv.n(), J, T(P.damping) * T(P.damping), G);
  const bool ok = chol6(G);
  chol6_solve(G, rhs);
#pragma unroll
  for (int j = 0; j < mv.n(); ++j) {
    T s = T(0);
#pragma unroll
    for (int r = 0; r < 6; ++r) s += J[r][j] * rhs[r];
    qdot[j] = s;
  }
  if (err_out) {
#pragma unroll
    for (int r = 0; r < 6; ++r) err_out[r] = err[r];
  }
  return ok;
}

// manipulability (kinematics.hpp:138-153): sqrt(det(J Jᵀ)) as the pivot
// product of the Cholesky factor; 0 when the factorization fails.
template <class V>
__device__ __forceinline__ typename V::Real manip_one(const V& mv, const JM<typename V::S>* jm, const TaskShared& P) {
  using T = typename V::Real;
  constexpr int NM = V::kMax;
  T pose_R[9], pose_p[3], J[6][NM];
  frame_pose_jacobian(mv, jm, P.frame_joint, P.frame_R, P.frame_p, pose_R, pose_p, J);
  T G[36];
  gram6(mv.n(), J, T(0), G);
  if (!chol6(G)) return T(0);
  T d = T(1);
#pragma unroll
  for (int i = 0; i < 6; ++i) d = d * G[i * 6 + i];
  return d;
}

// osc_step (control.hpp:108-155).  The mass matrix is factorised with the
// branch-sparse LTL of RBDA §6.5 (M = Lᵀ L, L with the ancestor sparsity of
// M, no fill-in) instead of a dense LLT; both give M⁻¹ x exactly in exact
// arithmetic, and both fail exactly when M is not positive definite.
template <class V, class QA>
__device__ __forceinline__ bool osc_one(const V& mv, const JM<typename V::S>* jm, const QA& q, const QA& qd,
                                        const OscShared& P, typename V::Real* tau_out, typename V::Real* lambda_out) {
  using S = typename V::S;
  using T = typename V::Real;
  constexpr int NM = V::kMax;
  bool ok = true;
  // --- mass matrix, compact ancestor rows: Mc[i][d] = M(i, anc_d(i)), d = 0 diagonal
  T Mc[NM][V::kMaxDepthC];
  crba_one(mv, jm, [&](int i, int j, const S& val) {
    // depth distance between i and its ancestor j
    const int d = mv.depth(i) - mv.depth(j);
    Mc[i][d] = val.v;
  });
  // --- bias c + g
  S bias[NM];
  {
    const T g3[3] = {T(P.gravity[0]), T(P.gravity[1]), T(P.gravity[2])};
    rnea_one<V, false, QA, QA>(mv, jm, qd, static_cast<const QA*>(nullptr), g3, nullptr, bias);
  }
  // --- frame pose and Jacobian (kinematics.hpp:89-129)
  T pose_R[9], pose_p[3], J[6][NM];
  frame_pose_jacobian(mv, jm, P.frame_joint, P.frame_R, P.frame_p, pose_R, pose_p, J);
  // --- pose error (control.hpp:73-77): log(R_t R_cᵀ), p_t − p_c
  T err[6];
  pose_error(P.target_R, P.target_p, pose_R, pose_p, err);
  // --- LTL factorisation in place (RBDA Table 6.3)
#pragma unroll
  for (int k = mv.n() - 1; k >= 0; --k) {
    const T dkk = Mc[k][0];
    ok = ok && (dkk > T(0));
    const T lkk = sqrt(dkk);
    Mc[k][0] = lkk;
    const T inv = T(1) / lkk;
#pragma unroll
    for (int d = 1; d < mv.max_depth(); ++d)
      if (d < mv.depth(k)) Mc[k][d] *= inv;
    // for ancestors i = anc_d(k) and j = anc_e(k), e >= d: M(i, j) -= L(k,i) L(k,j)
    int i = k;
#pragma unroll
    for (int d = 1; d < mv.max_depth(); ++d) {
      if (d >= mv.depth(k)) break;
      i = mv.parent(i);
#pragma unroll
      for (int e = d; e < mv.max_depth(); ++e)
        if (e < mv.depth(k)) Mc[i][e - d] -= Mc[k][d] * Mc[k][e];
    }
  }
  // --- 7 right-hand sides: rows of J (M⁻¹ Jᵀ) and τ_post (M⁻¹ τ_post)
  T tp[NM];
#pragma unroll
  for (int k = 0; k < mv.n(); ++k) tp[k] = T(P.posture_kp) * (T(P.posture[k]) - q[k]) - T(P.posture_kd) * qd[k];
  T X[7][NM];
#pragma unroll
  for (int r = 0; r < 7; ++r)
#pragma unroll
    for (int k = 0; k < mv.n(); ++k) X[r][k] = r < 6 ? J[r][k] : tp[k];
  // Lᵀ y = b
#pragma unroll
  for (int i = mv.n() - 1; i >= 0; --i) {
    const T inv = T(1) / Mc[i][0];
#pragma unroll
    for (int r = 0; r < 7; ++r) X[r][i] *= inv;
    int j = i;
#pragma unroll
    for (int d = 1; d < mv.max_depth(); ++d) {
      if (d >= mv.depth(i)) break;
      j = mv.parent(j);
#pragma unroll
      for (int r = 0; r < 7; ++r) X[r][j] -= Mc[i][d] * X[r][i];
    }
  }
  // L x = y
#pragma unroll
  for (int i = 0; i < mv.n(); ++i) {
    int j = i;
#pragma unroll
    for (int d = 1; d < mv.max_depth(); ++d) {
      if (d >= mv.depth(i)) break;
      j = mv.parent(j);
#pragma unroll
      for (int r = 0; r < 7; ++r) X[r][i] -= Mc[i][d] * X[r][j];
    }
    const T inv = T(1) / Mc[i][0];
#pragma unroll
    for (int r = 0; r < 7; ++r) X[r][i] *= inv;
  }
  // --- gram = J M⁻¹ Jᵀ, w = J M⁻¹ τ_post, J q̇
  T gram[36], w[6], jqd[6];
#pragma unroll
  for (int r = 0; r < 6; ++r) {
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      T s = T(0);
#pragma unroll
      for (int k = 0; k < mv.n(); ++k) s += J[r][k] * X[c][k];
      if (c < 6) gram[r * 6 + c] = s;
      else w[r] = s;
    }
    T s = T(0);
#pragma unroll
    for (int k = 0; k < mv.n(); ++k) s += J[r][k] * qd[k];
    jqd[r] = s;
  }
  T Lr[36], Lg[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) {
    Lg[k] = gram[k];
    Lr[k] = gram[k] + ((k % 7 == 0) ? T(P.epsilon) : T(0));
  }
  chol6(Lr);
  const bool gram_ok = chol6(Lg);
  T F[6], z[6];
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    F[r] = T(P.kp[r]) * err[r] - T(P.kd[r]) * jqd[r] + T(P.accel_ff[r]);
    z[r] = w[r];
  }
  chol6_solve(Lr, F);
  chol6_solve(gram_ok ? Lg : Lr, z);
  // τ = Jᵀ (F − z) + τ_post + bias
#pragma unroll
  for (int k = 0; k < mv.n(); ++k) {
    T s = tp[k] + bias[k].v;
#pragma unroll
    for (int r = 0; r < 6; ++r) s += J[r][k] * (F[r] - z[r]);
    tau_out[k] = s;
    ok = ok && isfinite(s);
  }
  if (lambda_out) {
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      T e[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) e[r] = r == c ? T(1) : T(0);
      chol6_solve(Lr, e);
#pragma unroll
      for (int r = 0; r < 6; ++r) lambda_out[c * 6 + r] = e[r];
    }
  }
  return ok;
}

}  // namespace vdk
