// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_spatial.hpp header).
//
// Restatement of the reference hot path, templated over the scalar like the
// reference (double / float / op-counting scalar):
//   kinematics.hpp:25-153   FK, scan FK, frame_transform, geometric_jacobian, manipulability
//   dynamics.hpp:167-444    prepare_world_arrays, vectorized (mask) RNEA & CRBA,
//                           loop RNEA & CRBA, gravity/coriolis, LLT forward dynamics
//   control.hpp:44-155      rotation_log, pose_error, diff_ik_step, osc_step
// plus `aba_loop`, a textbook articulated-body forward dynamics that the
// reference does NOT have; it is cross-checked against the
// reference-restated LLT forward dynamics in the oracle's own test port and
// serves only to freeze the algorithmic flop count of ABA.
#pragma once

#include <cmath>
#include <string_view>
#include <vector>

#include "orc_model.hpp"

namespace orc {

// ---------------------------------------------------------------- dense helpers
// Column-major dense matrix (Eigen's default storage order).
template <class T>
struct Dense {
  int rows = 0, cols = 0;
  std::vector<T> d;
  Dense() = default;
  Dense(int r, int c) : rows(r), cols(c), d((size_t)r * c, T(0)) {}
  T& operator()(int r, int c) { return d[(size_t)c * rows + r]; }
  const T& operator()(int r, int c) const { return d[(size_t)c * rows + r]; }
};

// Eigen::LLT (lower, unblocked for the sizes used here).  Returns false when a
// pivot is <= 0 (Eigen's failure criterion).
template <class T>
bool llt_factor(Dense<T>& a) {
  using std::sqrt;
  const int n = a.rows;
  for (int k = 0; k < n; ++k) {
    T x = a(k, k);
    for (int j = 0; j < k; ++j) x = x - a(k, j) * a(k, j);
    if (!(x > T(0))) {
      if (x <= T(0)) return false;
    }
    x = sqrt(x);
    a(k, k) = x;
    for (int i = k + 1; i < n; ++i) {
      T s = a(i, k);
      for (int j = 0; j < k; ++j) s = s - a(i, j) * a(k, j);
      a(i, k) = s / x;
    }
  }
  return true;
}
// Solve (L Lᵀ) X = B in place.
template <class T>
void llt_solve(const Dense<T>& L, Dense<T>& B) {
  const int n = L.rows;
  for (int c = 0; c < B.cols; ++c) {
    for (int i = 0; i < n; ++i) {
      T s = B(i, c);
      for (int j = 0; j < i; ++j) s = s - L(i, j) * B(j, c);
      B(i, c) = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      T s = B(i, c);
      for (int j = i + 1; j < n; ++j) s = s - L(j, i) * B(j, c);
      B(i, c) = s / L(i, i);
    }
  }
}

// ---------------------------------------------------------------- gravity / fext
// GravitySpec, dynamics.hpp:35-50: a_g = -field, default (0,0,0, 0,0,+9.81).
struct Gravity {
  V3<double> lin{0, 0, 9.81};
  static Gravity standard() { return Gravity(); }
  static Gravity zero() { return Gravity{V3<double>(0, 0, 0)}; }
  static Gravity from_field(const V3<double>& f) { return Gravity{-f}; }
};

// ExternalForcesT, dynamics.hpp:52-81: per-joint world Plücker wrenches.
template <class T>
struct ExtForces {
  std::vector<Force<T>> w;  // empty = none
  ExtForces() = default;
  explicit ExtForces(int n) : w((size_t)n) {}
  bool empty() const { return w.empty(); }
  int size() const { return (int)w.size(); }
  void add_at_point(int j, const V3<T>& pt, const V3<T>& f, const V3<T>& couple = V3<T>()) {
    w[(size_t)j].mom = w[(size_t)j].mom + (couple + cross3(pt, f));
    w[(size_t)j].frc = w[(size_t)j].frc + f;
  }
};

namespace detail {
inline void check_size(const Model& m, size_t sz, const char* what) {
  if ((int)sz != m.dof())
    throw DimensionError(std::string(what) + " has size " + std::to_string(sz) + ", model has " +
                         std::to_string(m.dof()) + " dof");
}
template <class T>
void check_fext(const Model& m, const ExtForces<T>& f) {
  if (!f.empty() && f.size() != m.dof())
    throw DimensionError("external forces have " + std::to_string(f.size()) + " rows, model has " +
                         std::to_string(m.dof()) + " dof");
}
// model.hpp:167-173 + kinematics.hpp:35-38
template <class T>
Xform<T> local_transform(const Joint& j, const T& q) {
  Xform<T> motion;
  if (j.type == JointType::Revolute) {
    motion.R = axis_angle_rotation<T>(j.axis, q);
  } else {
    motion.p = j.axis.as<T>() * q;
  }
  return j.offset.as<T>() * motion;
}
// dynamics.hpp:169-175
template <class T>
Motion<T> local_axis(const Joint& j) {
  Motion<T> s;
  if (j.type == JointType::Revolute) s.ang = j.axis.as<T>();
  else s.lin = j.axis.as<T>();
  return s;
}
}  // namespace detail

// ================================================================ kinematics
template <class T>
using Frames = std::vector<Xform<T>>;

// kinematics.hpp:43-56
template <class T>
Frames<T> forward_kinematics(const Model& m, const std::vector<T>& q) {
  detail::check_size(m, q.size(), "configuration vector");
  Frames<T> w((size_t)m.dof());
  for (int i = 0; i < m.dof(); ++i) {
    const Joint& j = m.joints[(size_t)i];
    const Xform<T> loc = detail::local_transform<T>(j, q[(size_t)i]);
    w[(size_t)i] = j.parent < 0 ? loc : w[(size_t)j.parent] * loc;
  }
  return w;
}

// kinematics.hpp:61-86 (Hillis–Steele inclusive scan, serial chains only)
template <class T>
Frames<T> forward_kinematics_scan(const Model& m, const std::vector<T>& q) {
  if (!m.serial)
    throw UnsupportedStructureError(
        "forward_kinematics_scan requires a serial chain (every joint's parent must be its predecessor)");
  detail::check_size(m, q.size(), "configuration vector");
  const int n = m.dof();
  Frames<T> w((size_t)n);
  for (int i = 0; i < n; ++i) w[(size_t)i] = detail::local_transform<T>(m.joints[(size_t)i], q[(size_t)i]);
  for (int step = 1; step < n; step *= 2)
    for (int i = n - 1; i >= step; --i) w[(size_t)i] = w[(size_t)(i - step)] * w[(size_t)i];
  return w;
}

// kinematics.hpp:89-96
template <class T>
Xform<T> frame_transform(const Model& m, const Frames<T>& w, std::string_view name) {
  const Frame& f = m.frame(name);
  const Xform<T> off = f.offset.as<T>();
  return f.joint < 0 ? off : w[(size_t)f.joint] * off;
}

// kinematics.hpp:108-129.  Returns 6 x n column-major.
template <class T>
Dense<T> geometric_jacobian(const Model& m, const Frames<T>& w, std::string_view name) {
  const Frame& f = m.frame(name);
  Dense<T> J(6, m.dof());
  const Xform<T> target = frame_transform(m, w, name);
  for (int j = f.joint; j >= 0; j = m.joints[(size_t)j].parent) {
    const Joint& jt = m.joints[(size_t)j];
    const Xform<T>& x = w[(size_t)j];
    const V3<T> ax = x.R * jt.axis.as<T>();
    if (jt.type == JointType::Revolute) {
      const V3<T> lin = cross3(ax, target.p - x.p);
      for (int r = 0; r < 3; ++r) {
        J(r, j) = ax[r];
        J(r + 3, j) = lin[r];
      }
    } else {
      for (int r = 0; r < 3; ++r) J(r + 3, j) = ax[r];
    }
  }
  return J;
}

// kinematics.hpp:141-153
template <class T>
T manipulability(const Dense<T>& J) {
  Dense<T> g(6, 6);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      T s = T(0);
      for (int k = 0; k < J.cols; ++k) s = s + J(r, k) * J(c, k);
      g(r, c) = s;
    }
  if (!llt_factor(g)) return T(0);
  T d = T(1);
  for (int i = 0; i < 6; ++i) d = d * g(i, i);
  return d;
}

// ================================================================ dynamics
// DynamicsWorkspaceT, dynamics.hpp:178-186: rows of S, I (row-major 6x6), V, A, F, C.
template <class T>
struct Workspace {
  std::vector<Motion<T>> S, V, A;
  std::vector<Force<T>> F;
  std::vector<Mat6<T>> I, C;
};

// dynamics.hpp:182-213
template <class T>
void prepare_world_arrays(const Model& m, const Frames<T>& w, Workspace<T>& ws) {
  const int n = m.dof();
  ws.S.assign((size_t)n, Motion<T>());
  ws.I.assign((size_t)n, Mat6<T>());
  for (int i = 0; i < n; ++i) {
    const Joint& j = m.joints[(size_t)i];
    const Xform<T>& x = w[(size_t)i];
    const V3<T> ax = x.R * j.axis.as<T>();
    if (j.type == JointType::Revolute) {
      ws.S[(size_t)i].ang = ax;
      ws.S[(size_t)i].lin = cross3(x.p, ax);
    } else {
      ws.S[(size_t)i].lin = ax;
    }
    ws.I[(size_t)i] = transform_inertia(x, m.inertias[(size_t)i].as<T>());
  }
}

// dynamics.hpp:222-248: mask-product form
//   V = U (S∘q̇) ; A = a_g + U (S∘q̈ + V × S∘q̇) ; F = Uᵀ (I A + V ×* I V − F_ext) ; τ = S·F
template <class T>
std::vector<T> rnea_from_workspace(const Model& m, Workspace<T>& ws, const std::vector<T>& qd,
                                   const std::vector<T>& qdd, const Gravity& g, const ExtForces<T>& fext) {
  detail::check_size(m, qd.size(), "qd");
  detail::check_size(m, qdd.size(), "qdd");
  detail::check_fext(m, fext);
  const int n = m.dof();
  std::vector<Motion<T>> sqd((size_t)n), inner((size_t)n);
  for (int i = 0; i < n; ++i) sqd[(size_t)i] = ws.S[(size_t)i] * qd[(size_t)i];
  ws.V.assign((size_t)n, Motion<T>());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (m.U(i, j) != 0.0) ws.V[(size_t)i] = ws.V[(size_t)i] + sqd[(size_t)j] * T(m.U(i, j));
  for (int i = 0; i < n; ++i)
    inner[(size_t)i] = ws.S[(size_t)i] * qdd[(size_t)i] + cross_motion(ws.V[(size_t)i], sqd[(size_t)i]);
  ws.A.assign((size_t)n, Motion<T>());
  const V3<T> ag = g.lin.as<T>();
  for (int i = 0; i < n; ++i) {
    Motion<T> a;
    for (int j = 0; j < n; ++j)
      if (m.U(i, j) != 0.0) a = a + inner[(size_t)j] * T(m.U(i, j));
    a.lin = a.lin + ag;
    ws.A[(size_t)i] = a;
  }
  std::vector<Force<T>> fb((size_t)n);
  for (int i = 0; i < n; ++i) {
    fb[(size_t)i] = apply(ws.I[(size_t)i], ws.A[(size_t)i]) +
                    cross_force(ws.V[(size_t)i], apply(ws.I[(size_t)i], ws.V[(size_t)i]));
    if (!fext.empty()) fb[(size_t)i] = fb[(size_t)i] - fext.w[(size_t)i];
  }
  ws.F.assign((size_t)n, Force<T>());
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (m.U(i, j) != 0.0) ws.F[(size_t)j] = ws.F[(size_t)j] + fb[(size_t)i] * T(m.U(i, j));
  std::vector<T> tau((size_t)n);
  for (int i = 0; i < n; ++i) tau[(size_t)i] = dot(ws.F[(size_t)i], ws.S[(size_t)i]);
  return tau;
}

template <class T>
std::vector<T> rnea(const Model& m, const std::vector<T>& q, const std::vector<T>& qd, const std::vector<T>& qdd,
                    const Gravity& g = Gravity::standard(), const ExtForces<T>& fext = ExtForces<T>(),
                    Workspace<T>* wsp = nullptr) {
  Workspace<T> local;
  Workspace<T>& ws = wsp ? *wsp : local;
  prepare_world_arrays(m, forward_kinematics(m, q), ws);
  return rnea_from_workspace(m, ws, qd, qdd, g, fext);
}

// dynamics.hpp:272-327: local-frame two-pass recursion.
template <class T>
std::vector<T> rnea_loop(const Model& m, const std::vector<T>& q, const std::vector<T>& qd,
                         const std::vector<T>& qdd, const Gravity& g = Gravity::standard(),
                         const ExtForces<T>& fext = ExtForces<T>()) {
  detail::check_size(m, q.size(), "configuration vector");
  detail::check_size(m, qd.size(), "qd");
  detail::check_size(m, qdd.size(), "qdd");
  detail::check_fext(m, fext);
  const int n = m.dof();
  std::vector<Xform<T>> xpc((size_t)n), world((size_t)n);
  std::vector<Motion<T>> v((size_t)n), a((size_t)n);
  std::vector<Force<T>> f((size_t)n);
  Motion<T> abase;
  abase.lin = g.lin.as<T>();
  for (int i = 0; i < n; ++i) {
    const Joint& j = m.joints[(size_t)i];
    const int p = j.parent;
    xpc[(size_t)i] = detail::local_transform<T>(j, q[(size_t)i]);
    const Motion<T> s = detail::local_axis<T>(j);
    const Motion<T> vj = s * qd[(size_t)i];
    v[(size_t)i] = inverse_transform_motion(xpc[(size_t)i], p < 0 ? Motion<T>() : v[(size_t)p]) + vj;
    a[(size_t)i] = inverse_transform_motion(xpc[(size_t)i], p < 0 ? abase : a[(size_t)p]) + s * qdd[(size_t)i] +
                   cross_motion(v[(size_t)i], vj);
    const Mat6<T> I = m.inertias[(size_t)i].as<T>();
    f[(size_t)i] = apply(I, a[(size_t)i]) + cross_force(v[(size_t)i], apply(I, v[(size_t)i]));
    if (!fext.empty()) {
      world[(size_t)i] = p < 0 ? xpc[(size_t)i] : world[(size_t)p] * xpc[(size_t)i];
      f[(size_t)i] = f[(size_t)i] - inverse_transform_force(world[(size_t)i], fext.w[(size_t)i]);
    }
  }
  std::vector<T> tau((size_t)n);
  for (int i = n - 1; i >= 0; --i) {
    const Joint& j = m.joints[(size_t)i];
    tau[(size_t)i] = dot(f[(size_t)i], detail::local_axis<T>(j));
    if (j.parent >= 0) f[(size_t)j.parent] = f[(size_t)j.parent] + transform_force(xpc[(size_t)i], f[(size_t)i]);
  }
  return tau;
}

// dynamics.hpp:337-350: C = Uᵀ I ; lower = U ⊙ (C S)·Sᵀ ; M = L + Lᵀ − diag L.
template <class T>
Dense<T> crba_from_workspace(const Model& m, Workspace<T>& ws) {
  const int n = m.dof();
  ws.C.assign((size_t)n, Mat6<T>());
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (m.U(i, j) != 0.0) ws.C[(size_t)j] = ws.C[(size_t)j] + ws.I[(size_t)i];
  std::vector<Force<T>> cs((size_t)n);
  for (int i = 0; i < n; ++i) cs[(size_t)i] = apply(ws.C[(size_t)i], ws.S[(size_t)i]);
  Dense<T> M(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j)
      if (m.U(i, j) != 0.0) {
        const T l = dot(cs[(size_t)i], ws.S[(size_t)j]);
        M(i, j) = l;
        M(j, i) = l;
      }
  return M;
}

template <class T>
Dense<T> crba(const Model& m, const std::vector<T>& q, Workspace<T>* wsp = nullptr) {
  Workspace<T> local;
  Workspace<T>& ws = wsp ? *wsp : local;
  prepare_world_arrays(m, forward_kinematics(m, q), ws);
  return crba_from_workspace(m, ws);
}

// dynamics.hpp:369-400
template <class T>
Dense<T> crba_loop(const Model& m, const std::vector<T>& q) {
  detail::check_size(m, q.size(), "configuration vector");
  const int n = m.dof();
  std::vector<Xform<T>> xpc((size_t)n);
  std::vector<Mat6<T>> ic((size_t)n);
  for (int i = 0; i < n; ++i) {
    xpc[(size_t)i] = detail::local_transform<T>(m.joints[(size_t)i], q[(size_t)i]);
    ic[(size_t)i] = m.inertias[(size_t)i].as<T>();
  }
  for (int i = n - 1; i >= 0; --i) {
    const int p = m.joints[(size_t)i].parent;
    if (p >= 0) ic[(size_t)p] = ic[(size_t)p] + transform_inertia(xpc[(size_t)i], ic[(size_t)i]);
  }
  Dense<T> M(n, n);
  for (int i = 0; i < n; ++i) {
    const Motion<T> si = detail::local_axis<T>(m.joints[(size_t)i]);
    Force<T> f = apply(ic[(size_t)i], si);
    M(i, i) = dot(f, si);
    int j = i;
    while (m.joints[(size_t)j].parent >= 0) {
      f = transform_force(xpc[(size_t)j], f);
      j = m.joints[(size_t)j].parent;
      const T v = dot(f, detail::local_axis<T>(m.joints[(size_t)j]));
      M(i, j) = v;
      M(j, i) = v;
    }
  }
  return M;
}

// dynamics.hpp:402-416
template <class T>
std::vector<T> gravity_vector(const Model& m, const std::vector<T>& q, const Gravity& g = Gravity::standard()) {
  const std::vector<T> z((size_t)m.dof(), T(0));
  return rnea<T>(m, q, z, z, g);
}
template <class T>
std::vector<T> coriolis_vector(const Model& m, const std::vector<T>& q, const std::vector<T>& qd) {
  const std::vector<T> z((size_t)m.dof(), T(0));
  return rnea<T>(m, q, qd, z, Gravity::zero());
}

// dynamics.hpp:418-444: q̈ = M⁻¹(τ − bias) via LLT; SingularInertiaError if not PD.
template <class T>
std::vector<T> forward_dynamics(const Model& m, const std::vector<T>& q, const std::vector<T>& qd,
                                const std::vector<T>& tau, const Gravity& g = Gravity::standard(),
                                const ExtForces<T>& fext = ExtForces<T>()) {
  detail::check_size(m, tau.size(), "tau");
  const int n = m.dof();
  if (n == 0) return {};
  Workspace<T> ws;
  prepare_world_arrays(m, forward_kinematics(m, q), ws);
  const std::vector<T> z((size_t)n, T(0));
  const std::vector<T> bias = rnea_from_workspace(m, ws, qd, z, g, fext);
  Dense<T> M = crba_from_workspace(m, ws);
  if (!llt_factor(M))
    throw SingularInertiaError(
        "forward_dynamics: mass matrix is not positive definite (zero-inertia degree of freedom?)");
  Dense<T> rhs(n, 1);
  for (int i = 0; i < n; ++i) rhs(i, 0) = tau[(size_t)i] - bias[(size_t)i];
  llt_solve(M, rhs);
  return rhs.d;
}

// Articulated-body algorithm (Featherstone, RBDA Table 7.1) in local
// coordinates — NOT in the reference; see the file header.
template <class T>
std::vector<T> aba_loop(const Model& m, const std::vector<T>& q, const std::vector<T>& qd, const std::vector<T>& tau,
                        const Gravity& g = Gravity::standard(), const ExtForces<T>& fext = ExtForces<T>()) {
  detail::check_size(m, q.size(), "configuration vector");
  detail::check_size(m, qd.size(), "qd");
  detail::check_size(m, tau.size(), "tau");
  detail::check_fext(m, fext);
  const int n = m.dof();
  std::vector<Xform<T>> xpc((size_t)n), world((size_t)n);
  std::vector<Motion<T>> v((size_t)n), c((size_t)n), a((size_t)n), S((size_t)n);
  std::vector<Mat6<T>> IA((size_t)n);
  std::vector<Force<T>> pA((size_t)n), U((size_t)n);
  std::vector<T> D((size_t)n), u((size_t)n), qdd((size_t)n);
  for (int i = 0; i < n; ++i) {
    const Joint& j = m.joints[(size_t)i];
    const int p = j.parent;
    xpc[(size_t)i] = detail::local_transform<T>(j, q[(size_t)i]);
    S[(size_t)i] = detail::local_axis<T>(j);
    const Motion<T> vj = S[(size_t)i] * qd[(size_t)i];
    v[(size_t)i] = (p < 0 ? Motion<T>() : inverse_transform_motion(xpc[(size_t)i], v[(size_t)p])) + vj;
    c[(size_t)i] = cross_motion(v[(size_t)i], vj);
    IA[(size_t)i] = m.inertias[(size_t)i].as<T>();
    pA[(size_t)i] = cross_force(v[(size_t)i], apply(IA[(size_t)i], v[(size_t)i]));
    if (!fext.empty()) {
      world[(size_t)i] = p < 0 ? xpc[(size_t)i] : world[(size_t)p] * xpc[(size_t)i];
      pA[(size_t)i] = pA[(size_t)i] - inverse_transform_force(world[(size_t)i], fext.w[(size_t)i]);
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    const Motion<T>& s = S[(size_t)i];
    U[(size_t)i] = apply(IA[(size_t)i], s);
    D[(size_t)i] = dot(U[(size_t)i], s);
    u[(size_t)i] = tau[(size_t)i] - dot(pA[(size_t)i], s);
    const int p = m.joints[(size_t)i].parent;
    if (p < 0) continue;
    Mat6<T> Ia = IA[(size_t)i];
    const T dinv = T(1) / D[(size_t)i];
    for (int r = 0; r < 6; ++r)
      for (int cc = 0; cc < 6; ++cc) Ia(r, cc) = Ia(r, cc) - U[(size_t)i][r] * U[(size_t)i][cc] * dinv;
    const Force<T> pa = pA[(size_t)i] + apply(Ia, c[(size_t)i]) + U[(size_t)i] * (u[(size_t)i] * dinv);
    IA[(size_t)p] = IA[(size_t)p] + transform_inertia(xpc[(size_t)i], Ia);
    pA[(size_t)p] = pA[(size_t)p] + transform_force(xpc[(size_t)i], pa);
  }
  Motion<T> abase;
  abase.lin = g.lin.as<T>();
  for (int i = 0; i < n; ++i) {
    const int p = m.joints[(size_t)i].parent;
    const Motion<T> ap = inverse_transform_motion(xpc[(size_t)i], p < 0 ? abase : a[(size_t)p]) + c[(size_t)i];
    qdd[(size_t)i] = (u[(size_t)i] - dot(U[(size_t)i], ap)) / D[(size_t)i];
    a[(size_t)i] = ap + S[(size_t)i] * qdd[(size_t)i];
  }
  return qdd;
}

// ================================================================ control
// control.hpp:12-42
struct TaskGains {
  double kp[6] = {0, 0, 0, 0, 0, 0}, kd[6] = {0, 0, 0, 0, 0, 0};
  static TaskGains uniform(double p, double d = 0.0) {
    TaskGains g;
    for (int i = 0; i < 6; ++i) {
      g.kp[i] = p;
      g.kd[i] = d;
    }
    return g;
  }
};
struct TaskTarget {
  std::string frame;
  Xform<double> pose;
  Motion<double> twist_ff, accel_ff;
  TaskGains gains;
  void validate() const {
    for (int i = 0; i < 6; ++i)
      if (gains.kp[i] < 0.0 || gains.kd[i] < 0.0) throw Error("task gains must be nonnegative");
  }
};
struct PostureGains {
  double kp = 0, kd = 0;
};

// control.hpp:45-68 (acos form, branches at 1e-9 and π − 1e-6)
inline V3<double> rotation_log(const M3<double>& r) {
  const double tr = r(0, 0) + r(1, 1) + r(2, 2);
  const V3<double> anti(r(2, 1) - r(1, 2), r(0, 2) - r(2, 0), r(1, 0) - r(0, 1));
  const double ca = std::clamp(0.5 * (tr - 1.0), -1.0, 1.0);
  const double ang = std::acos(ca);
  if (ang < 1e-9) return anti * 0.5;
  if (ang > M_PI - 1e-6) {
    M3<double> s = 0.5 * (r + M3<double>::identity());
    int k = 0;
    for (int i = 1; i < 3; ++i)
      if (s(i, i) > s(k, k)) k = i;
    V3<double> axis = V3<double>(s(0, k), s(1, k), s(2, k)) * (1.0 / std::sqrt(std::max(s(k, k), 1e-12)));
    axis = axis * (1.0 / norm3(axis));
    if (dot3(anti, axis) < 0.0) axis = -axis;
    return axis * ang;
  }
  return anti * (0.5 * ang / std::sin(ang));
}

// control.hpp:73-77
inline Motion<double> pose_error(const Xform<double>& target, const Xform<double>& cur) {
  return {rotation_log(target.R * transpose(cur.R)), target.p - cur.p};
}

// control.hpp:81-97
inline std::vector<double> diff_ik_step(const Model& m, const std::vector<double>& q, const TaskTarget& t,
                                        double damping) {
  if (damping <= 0.0) throw Error("diff_ik_step: damping must be positive");
  t.validate();
  const Frames<double> w = forward_kinematics(m, q);
  const Dense<double> J = geometric_jacobian(m, w, t.frame);
  const Motion<double> err = pose_error(t.pose, frame_transform(m, w, t.frame));
  Dense<double> rhs(6, 1), g(6, 6);
  for (int r = 0; r < 6; ++r) rhs(r, 0) = t.gains.kp[r] * err[r] + t.twist_ff[r];
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      double s = 0;
      for (int k = 0; k < m.dof(); ++k) s += J(r, k) * J(c, k);
      g(r, c) = s + (r == c ? damping * damping : 0.0);
    }
  llt_factor(g);
  llt_solve(g, rhs);
  std::vector<double> out((size_t)m.dof(), 0.0);
  for (int k = 0; k < m.dof(); ++k)
    for (int r = 0; r < 6; ++r) out[(size_t)k] += J(r, k) * rhs(r, 0);
  return out;
}

struct OscResult {
  std::vector<double> tau;
  double Lambda[36];  // (J M⁻¹ Jᵀ + εI)⁻¹, column-major
};

// control.hpp:108-155 (Khatib OSC), plus Λ returned for the batched API.
inline OscResult osc_step_full(const Model& m, const std::vector<double>& q, const std::vector<double>& qd,
                               const TaskTarget& t, const std::vector<double>& posture, const PostureGains& pg,
                               const Gravity& g = Gravity::standard(), double eps = 1e-6) {
  t.validate();
  const int n = m.dof();
  detail::check_size(m, qd.size(), "qd");
  detail::check_size(m, posture.size(), "posture");
  const Frames<double> w = forward_kinematics(m, q);
  Workspace<double> ws;
  prepare_world_arrays(m, w, ws);
  Dense<double> M = crba_from_workspace(m, ws);
  const std::vector<double> z((size_t)n, 0.0);
  const std::vector<double> bias = rnea_from_workspace(m, ws, qd, z, g, ExtForces<double>());
  const Dense<double> J = geometric_jacobian(m, w, t.frame);
  const Motion<double> err = pose_error(t.pose, frame_transform(m, w, t.frame));
  if (!llt_factor(M)) throw SingularInertiaError("osc_step: mass matrix is not positive definite");
  Dense<double> minv_jt(n, 6);  // M⁻¹ Jᵀ
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < 6; ++c) minv_jt(r, c) = J(c, r);
  llt_solve(M, minv_jt);
  Dense<double> gram(6, 6);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += J(r, k) * minv_jt(k, c);
      gram(r, c) = s;
    }
  Dense<double> greg = gram;
  for (int i = 0; i < 6; ++i) greg(i, i) += eps;
  Dense<double> task(6, 1);
  for (int r = 0; r < 6; ++r) {
    double jqd = 0;
    for (int k = 0; k < n; ++k) jqd += J(r, k) * qd[(size_t)k];
    task(r, 0) = t.gains.kp[r] * err[r] - t.gains.kd[r] * jqd + t.accel_ff[r];
  }
  Dense<double> greg_l = greg;
  llt_factor(greg_l);
  Dense<double> F = task;
  llt_solve(greg_l, F);
  // J̄ᵀ = gram⁻¹ (M⁻¹Jᵀ)ᵀ, falling back to the regularized factor.
  Dense<double> gram_l = gram;
  const bool ok = llt_factor(gram_l);
  Dense<double> jbar_t(6, n);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < n; ++c) jbar_t(r, c) = minv_jt(c, r);
  llt_solve(ok ? gram_l : greg_l, jbar_t);
  std::vector<double> tp((size_t)n);
  for (int i = 0; i < n; ++i) tp[(size_t)i] = pg.kp * (posture[(size_t)i] - q[(size_t)i]) - pg.kd * qd[(size_t)i];
  double jb_tp[6];
  for (int r = 0; r < 6; ++r) {
    double s = 0;
    for (int k = 0; k < n; ++k) s += jbar_t(r, k) * tp[(size_t)k];
    jb_tp[r] = s;
  }
  OscResult out;
  out.tau.assign((size_t)n, 0.0);
  for (int k = 0; k < n; ++k) {
    double a = 0, b = 0;
    for (int r = 0; r < 6; ++r) {
      a += J(r, k) * F(r, 0);
      b += J(r, k) * jb_tp[r];
    }
    out.tau[(size_t)k] = a + tp[(size_t)k] - b + bias[(size_t)k];
  }
  // Λ = greg⁻¹
  Dense<double> lam(6, 6);
  for (int i = 0; i < 6; ++i) lam(i, i) = 1.0;
  llt_solve(greg_l, lam);
  for (int i = 0; i < 36; ++i) out.Lambda[i] = lam.d[(size_t)i];
  return out;
}

inline std::vector<double> osc_step(const Model& m, const std::vector<double>& q, const std::vector<double>& qd,
                                    const TaskTarget& t, const std::vector<double>& posture, const PostureGains& pg,
                                    const Gravity& g = Gravity::standard(), double eps = 1e-6) {
  return osc_step_full(m, q, qd, t, posture, pg, g, eps).tau;
}

}  // namespace orc
