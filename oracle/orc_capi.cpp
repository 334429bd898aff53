// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_spatial.hpp header).
//
// Flat C entry points over the oracle so Python tests / bench.py's
// cpu_baseline leg can drive it with ctypes.  Every batch entry point takes
// SoA column-major buffers (element (i, k) at k*N + i, exactly Eigen's
// column-major N x K used by StateBatch and batch_crba, batch.hpp:15-19,
// 147-148) and runs through orc::batch_eval (batch.hpp:82-125).
#include <algorithm>
#include <ctime>
#include <vector>
#include <cstring>
#include <string>

#include "orc_batch.hpp"
#include "orc_count.hpp"
#include "orc_dual.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ParseError*>(&e)) return 2;
  if (dynamic_cast<const UnknownFrameError*>(&e)) return 4;
  if (dynamic_cast<const ModelError*>(&e)) return 3;
  if (dynamic_cast<const DimensionError*>(&e)) return 1;
  if (dynamic_cast<const UnsupportedFeatureError*>(&e)) return 5;
  if (dynamic_cast<const UnsupportedStructureError*>(&e)) return 6;
  if (dynamic_cast<const SingularInertiaError*>(&e)) return 7;
  return 99;
}

Gravity grav(const double* g3) {
  Gravity g;
  if (g3) g.lin = V3<double>(g3[0], g3[1], g3[2]);
  return g;
}

template <class T>
std::vector<T> plane_row(const double* a, int64_t N, int n, int64_t i) {
  std::vector<T> r((size_t)n);
  for (int j = 0; j < n; ++j) r[(size_t)j] = T(a[j * N + i]);
  return r;
}

template <class T>
ExtForces<T> fext_row(const double* f, int64_t N, int n, int64_t i) {
  if (!f) return ExtForces<T>();
  ExtForces<T> e(n);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < 6; ++k) e.w[(size_t)j].at(k) = T(f[(j * 6 + k) * N + i]);
  return e;
}

const Model& M(void* h) { return *static_cast<Model*>(h); }

void put_xform(double* out, int64_t N, int64_t i, int base, const Xform<double>& x) {
  // R column-major (Eigen Mat3 storage), then p.
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) out[(base + c * 3 + r) * N + i] = x.R(r, c);
  for (int r = 0; r < 3; ++r) out[(base + 9 + r) * N + i] = x.p[r];
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void* orc_model_builtin(const char* name) {
  try {
    return new Model(robots::by_name(name));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void* orc_model_from_urdf(const char* text) {
  try {
    return new Model(urdf::load_model_from_string(text));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

int orc_model_from_urdf_status(const char* text, void** out) {
  try {
    *out = new Model(urdf::load_model_from_string(text));
    return 0;
  } catch (const std::exception& e) {
    *out = nullptr;
    return fail(e);
  }
}

void* orc_model_floating(void* h) {
  try {
    return new Model(floating_base(M(h)));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void orc_model_free(void* h) { delete static_cast<Model*>(h); }
int orc_model_dof(void* h) { return M(h).dof(); }
double orc_model_total_mass(void* h) { return M(h).total_mass; }
int orc_model_max_depth(void* h) { return M(h).max_depth; }
int orc_model_is_serial(void* h) { return M(h).serial ? 1 : 0; }
int orc_model_warning_count(void* h) { return (int)M(h).warnings.size(); }

// parents[n], types[n] (0 revolute, 1 prismatic), axes[n*3], offsets[n*12]
// (R row-major 9, p 3), inertias[n*36] (row-major), mask[n*n] (row-major).
void orc_model_arrays(void* h, int* parents, int* types, double* axes, double* offsets, double* inertias,
                      double* mask) {
  const Model& m = M(h);
  const int n = m.dof();
  for (int i = 0; i < n; ++i) {
    const Joint& j = m.joints[(size_t)i];
    if (parents) parents[i] = j.parent;
    if (types) types[i] = j.type == JointType::Revolute ? 0 : 1;
    for (int k = 0; k < 3; ++k) {
      if (axes) axes[i * 3 + k] = j.axis[k];
      if (offsets) offsets[i * 12 + 9 + k] = j.offset.p[k];
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        if (offsets) offsets[i * 12 + r * 3 + c] = j.offset.R(r, c);
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c)
        if (inertias) inertias[i * 36 + r * 6 + c] = m.inertias[(size_t)i](r, c);
  }
  if (mask)
    for (size_t k = 0; k < m.mask.size(); ++k) mask[k] = m.mask[k];
}

int orc_model_joint_name(void* h, int i, char* buf, int len) {
  const std::string& s = M(h).joints[(size_t)i].name;
  std::snprintf(buf, (size_t)len, "%s", s.c_str());
  return (int)s.size();
}

int orc_model_frame_count(void* h) { return (int)M(h).frames.size(); }
// Frame k: name into buf, joint index returned via *joint, offset as R row-major + p.
int orc_model_frame(void* h, int k, char* buf, int len, int* joint, double* off12) {
  const Frame& f = M(h).frames[(size_t)k];
  std::snprintf(buf, (size_t)len, "%s", f.name.c_str());
  *joint = f.joint;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) off12[r * 3 + c] = f.offset.R(r, c);
    off12[9 + r] = f.offset.p[r];
  }
  return 0;
}

int orc_frame_id(void* h, const char* name) {
  try {
    return M(h).frame_id(name);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// batch.hpp:48-75; any of qdd / tau may be null (with_qdd / with_tau false).
void orc_random_states(void* h, int64_t N, uint64_t seed, double* q, double* qd, double* qdd, double* tau) {
  StateBatch b = random_states(M(h), (int)N, seed, qdd != nullptr, tau != nullptr);
  std::memcpy(q, b.q.data(), b.q.size() * sizeof(double));
  std::memcpy(qd, b.qd.data(), b.qd.size() * sizeof(double));
  if (qdd) std::memcpy(qdd, b.qdd.data(), b.qdd.size() * sizeof(double));
  if (tau) std::memcpy(tau, b.tau.data(), b.tau.size() * sizeof(double));
}

// variant 0: vectorized mask form (dynamics.hpp:222-248); 1: rnea_loop.
// f32 != 0 evaluates in single precision (inputs rounded to float).
int orc_batch_rnea(void* h, int64_t N, const double* q, const double* qd, const double* qdd, const double* g3,
                   const double* fext, double* tau, int threads, int variant, int f32) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    const Gravity g = grav(g3);
    batch_eval((int)N,
               [&](int i) {
                 std::vector<double> r;
                 if (f32) {
                   auto a = plane_row<float>(q, N, n, i), b = plane_row<float>(qd, N, n, i),
                        c = plane_row<float>(qdd, N, n, i);
                   auto t = variant ? rnea_loop<float>(m, a, b, c, g, fext_row<float>(fext, N, n, i))
                                    : rnea<float>(m, a, b, c, g, fext_row<float>(fext, N, n, i));
                   r.assign(t.begin(), t.end());
                 } else {
                   auto a = plane_row<double>(q, N, n, i), b = plane_row<double>(qd, N, n, i),
                        c = plane_row<double>(qdd, N, n, i);
                   r = variant ? rnea_loop<double>(m, a, b, c, g, fext_row<double>(fext, N, n, i))
                               : rnea<double>(m, a, b, c, g, fext_row<double>(fext, N, n, i));
                 }
                 for (int j = 0; j < n; ++j) tau[j * N + i] = r[(size_t)j];
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// M column-major n x n per instance: plane c*n + r.  variant 0 vectorized, 1 loop.
int orc_batch_crba(void* h, int64_t N, const double* q, double* Mout, int threads, int variant, int f32) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    batch_eval((int)N,
               [&](int i) {
                 if (f32) {
                   auto a = plane_row<float>(q, N, n, i);
                   Dense<float> mm = variant ? crba_loop<float>(m, a) : crba<float>(m, a);
                   for (int k = 0; k < n * n; ++k) Mout[k * N + i] = mm.d[(size_t)k];
                 } else {
                   auto a = plane_row<double>(q, N, n, i);
                   Dense<double> mm = variant ? crba_loop<double>(m, a) : crba<double>(m, a);
                   for (int k = 0; k < n * n; ++k) Mout[k * N + i] = mm.d[(size_t)k];
                 }
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Forward dynamics. variant 0: reference LLT path (dynamics.hpp:421-444);
// 1: aba_loop.  status[i] = 0 ok, 7 singular (SingularInertiaError).
int orc_batch_fd(void* h, int64_t N, const double* q, const double* qd, const double* tau, const double* g3,
                 const double* fext, double* qdd, int* status, int threads, int variant) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    const Gravity g = grav(g3);
    batch_eval((int)N,
               [&](int i) {
                 auto a = plane_row<double>(q, N, n, i), b = plane_row<double>(qd, N, n, i),
                      c = plane_row<double>(tau, N, n, i);
                 int st = 0;
                 std::vector<double> r((size_t)n, 0.0);
                 try {
                   r = variant ? aba_loop<double>(m, a, b, c, g, fext_row<double>(fext, N, n, i))
                               : forward_dynamics<double>(m, a, b, c, g, fext_row<double>(fext, N, n, i));
                 } catch (const SingularInertiaError&) {
                   st = 7;
                 }
                 for (int j = 0; j < n; ++j) qdd[j * N + i] = r[(size_t)j];
                 if (status) status[i] = st;
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// All joint world transforms: plane (j*12 + k), k 0..8 = R column-major, 9..11 = p.
int orc_batch_fk(void* h, int64_t N, const double* q, double* out, int threads, int scan) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    batch_eval((int)N,
               [&](int i) {
                 auto a = plane_row<double>(q, N, n, i);
                 Frames<double> w = scan ? forward_kinematics_scan<double>(m, a) : forward_kinematics<double>(m, a);
                 for (int j = 0; j < n; ++j) put_xform(out, N, i, j * 12, w[(size_t)j]);
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Frame pose (12 planes) and 6 x n Jacobian (plane c*6 + r).
int orc_batch_jacobian(void* h, int64_t N, const double* q, const char* frame, double* pose, double* J,
                       int threads) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    (void)m.frame(frame);
    batch_eval((int)N,
               [&](int i) {
                 auto a = plane_row<double>(q, N, n, i);
                 Frames<double> w = forward_kinematics<double>(m, a);
                 if (pose) put_xform(pose, N, i, 0, frame_transform<double>(m, w, frame));
                 if (J) {
                   Dense<double> jj = geometric_jacobian<double>(m, w, frame);
                   for (int k = 0; k < 6 * n; ++k) J[k * N + i] = jj.d[(size_t)k];
                 }
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// OSC (control.hpp:108-155).  target12 = R row-major + p; kp/kd/accel_ff 6
// each (angular first); posture n values shared by the batch.
int orc_batch_osc(void* h, int64_t N, const double* q, const double* qd, const char* frame, const double* target12,
                  const double* kp, const double* kd, const double* accel_ff, const double* posture, double pkp,
                  double pkd, const double* g3, double eps, double* tau, double* lambda, int* status, int threads) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    TaskTarget t;
    t.frame = frame;
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) t.pose.R(r, c) = target12[r * 3 + c];
      t.pose.p[r] = target12[9 + r];
    }
    for (int k = 0; k < 6; ++k) {
      t.gains.kp[k] = kp[k];
      t.gains.kd[k] = kd[k];
      t.accel_ff.at(k) = accel_ff ? accel_ff[k] : 0.0;
    }
    (void)m.frame(frame);
    const std::vector<double> post(posture, posture + n);
    const PostureGains pg{pkp, pkd};
    const Gravity g = grav(g3);
    batch_eval((int)N,
               [&](int i) {
                 auto a = plane_row<double>(q, N, n, i), b = plane_row<double>(qd, N, n, i);
                 int st = 0;
                 OscResult r;
                 r.tau.assign((size_t)n, 0.0);
                 for (double& x : r.Lambda) x = 0.0;
                 try {
                   r = osc_step_full(m, a, b, t, post, pg, g, eps);
                 } catch (const SingularInertiaError&) {
                   st = 7;
                 }
                 for (int j = 0; j < n; ++j) tau[j * N + i] = r.tau[(size_t)j];
                 if (lambda)
                   for (int k = 0; k < 36; ++k) lambda[k * N + i] = r.Lambda[k];
                 if (status) status[i] = st;
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Forward-mode JVP (autodiff.hpp:41-52: the algorithm run on the Dual scalar
// of dual.hpp) of op 0 forward_kinematics (all frames, fk layout), 1 rnea,
// 2 crba, 3 forward dynamics, on inputs seeded with tangents (NULL = 0).
// variant: 0 the reference's vectorized / LLT path, 1 the loop path
// (rnea_loop, crba_loop, aba_loop).  out / dout: values / tangents.
int orc_batch_jvp(void* h, int op, int64_t N, const double* q, const double* qd, const double* x2, const double* dq,
                  const double* dqd, const double* dx2, const double* g3, const double* fext, double* out,
                  double* dout, int* status, int threads, int variant) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    const Gravity g = grav(g3);
    auto seed = [&](const double* x, const double* dx, int64_t i) {
      std::vector<Dual> r((size_t)n);
      for (int j = 0; j < n; ++j) r[(size_t)j] = Dual(x ? x[j * N + i] : 0.0, dx ? dx[j * N + i] : 0.0);
      return r;
    };
    auto put = [&](int k, int64_t i, const Dual& v) {
      if (out) out[k * N + i] = v.value;
      if (dout) dout[k * N + i] = v.tangent;
    };
    batch_eval((int)N,
               [&](int i) {
                 const std::vector<Dual> a = seed(q, dq, i);
                 if (op == 0) {
                   const Frames<Dual> w = forward_kinematics<Dual>(m, a);
                   for (int j = 0; j < n; ++j) {
                     for (int c = 0; c < 3; ++c)
                       for (int r = 0; r < 3; ++r) put(j * 12 + c * 3 + r, i, w[(size_t)j].R(r, c));
                     for (int r = 0; r < 3; ++r) put(j * 12 + 9 + r, i, w[(size_t)j].p[r]);
                   }
                 } else if (op == 2) {
                   const Dense<Dual> mm = variant ? crba_loop<Dual>(m, a) : crba<Dual>(m, a);
                   for (int k = 0; k < n * n; ++k) put(k, i, mm.d[(size_t)k]);
                 } else {
                   const std::vector<Dual> b = seed(qd, dqd, i), c = seed(x2, dx2, i);
                   const ExtForces<Dual> f = fext_row<Dual>(fext, N, n, i);
                   std::vector<Dual> r((size_t)n, Dual(0.0));
                   int st = 0;
                   if (op == 1) {
                     r = variant ? rnea_loop<Dual>(m, a, b, c, g, f) : rnea<Dual>(m, a, b, c, g, f);
                   } else {
                     try {
                       r = variant ? aba_loop<Dual>(m, a, b, c, g, f) : forward_dynamics<Dual>(m, a, b, c, g, f);
                     } catch (const SingularInertiaError&) {
                       st = 7;
                       r.assign((size_t)n, Dual(0.0));
                     }
                     if (status) status[i] = st;
                   }
                   for (int j = 0; j < n; ++j) put(j, i, r[(size_t)j]);
                 }
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// diff_ik_step per instance (control.hpp:79-97); err (6 planes, may be NULL) = pose_error.
int orc_batch_diffik(void* h, int64_t N, const double* q, const char* frame, const double* target12,
                     const double* kp, const double* twist_ff, double damping, double* qdot, double* err,
                     int threads) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    TaskTarget t;
    t.frame = frame;
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) t.pose.R(r, c) = target12[r * 3 + c];
      t.pose.p[r] = target12[9 + r];
    }
    for (int k = 0; k < 6; ++k) {
      t.gains.kp[k] = kp[k];
      t.twist_ff.at(k) = twist_ff ? twist_ff[k] : 0.0;
    }
    (void)m.frame(frame);
    (void)diff_ik_step(m, std::vector<double>((size_t)n, 0.0), t, damping);  // argument checks up front
    batch_eval((int)N,
               [&](int i) {
                 const auto a = plane_row<double>(q, N, n, i);
                 const std::vector<double> v = diff_ik_step(m, a, t, damping);
                 for (int j = 0; j < n; ++j) qdot[j * N + i] = v[(size_t)j];
                 if (err) {
                   const Frames<double> w = forward_kinematics(m, a);
                   const Motion<double> e = pose_error(t.pose, frame_transform(m, w, t.frame));
                   for (int k = 0; k < 6; ++k) err[k * N + i] = e[k];
                 }
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// manipulability(geometric_jacobian(frame)) per instance (kinematics.hpp:138-153).
int orc_batch_manip(void* h, int64_t N, const double* q, const char* frame, double* w_out, int threads) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    (void)m.frame(frame);
    const std::string f = frame;
    batch_eval((int)N,
               [&](int i) {
                 const Frames<double> w = forward_kinematics(m, plane_row<double>(q, N, n, i));
                 w_out[i] = manipulability(geometric_jacobian(m, w, f));
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// jvp_scalar (autodiff.hpp:52-62) of manipulability(geometric_jacobian(frame))
// per instance: the JVP the reference's lie_derivative (control.hpp:157-163)
// takes of h = manipulability ∘ J along a direction dq.
int orc_batch_manip_jvp(void* h, int64_t N, const double* q, const double* dq, const char* frame, double* w_out,
                        double* dw_out, int threads) {
  try {
    const Model& m = M(h);
    const int n = m.dof();
    (void)m.frame(frame);
    const std::string f = frame;
    batch_eval((int)N,
               [&](int i) {
                 std::vector<Dual> a((size_t)n);
                 for (int j = 0; j < n; ++j) a[(size_t)j] = Dual(q[j * N + i], dq ? dq[j * N + i] : 0.0);
                 const Frames<Dual> w = forward_kinematics<Dual>(m, a);
                 const Dual v = manipulability(geometric_jacobian(m, w, f));
                 w_out[i] = v.value;
                 dw_out[i] = v.tangent;
               },
               threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Frozen algorithmic op counts per evaluation (orc_count.hpp).  algo:
// 0 rnea_loop, 1 crba_loop, 2 aba_loop, 3 forward_kinematics, 4 rnea (mask
// form), 5 forward_dynamics (CRBA + bias + LLT), 6 crba (mask form).
// out[0..4] = add, mul, div, sqrt, trig; returns flops (add+mul+div).
extern "C++" {
template <class S>
static int count_algo(const Model& m, int algo) {
  const int n = m.dof();
  std::vector<S> q((size_t)n), qd((size_t)n), qdd((size_t)n);
  for (int i = 0; i < n; ++i) {  // generic, non-zero, non-unit state
    q[(size_t)i] = S(0.1 * (i + 1) + 0.0123);
    qd[(size_t)i] = S(0.2 - 0.03 * i + 0.0071);
    qdd[(size_t)i] = S(0.05 * i - 0.1 + 0.0037);
  }
  switch (algo) {
    case 0: (void)rnea_loop<S>(m, q, qd, qdd); break;
    case 1: (void)crba_loop<S>(m, q); break;
    case 2: (void)aba_loop<S>(m, q, qd, qdd); break;
    case 3: (void)forward_kinematics<S>(m, q); break;
    case 4: (void)rnea<S>(m, q, qd, qdd); break;
    case 5: (void)forward_dynamics<S>(m, q, qd, qdd); break;
    case 6: (void)crba<S>(m, q); break;
    default: return -1;
  }
  return 0;
}
}  // extern "C++"

// algo + 100: structure-aware count (orc_count.hpp `Sparse`).
double orc_count_flops(void* h, int algo, double* out) {
  const Model& m = M(h);
  op_count() = OpCount();
  const int rc = algo >= 100 ? count_algo<Sparse>(m, algo - 100) : count_algo<Counted>(m, algo);
  if (rc) return -1;
  const OpCount c = op_count();
  if (out) {
    out[0] = (double)c.add;
    out[1] = (double)c.mul;
    out[2] = (double)c.div;
    out[3] = (double)c.sqrt;
    out[4] = (double)c.trig;
  }
  return (double)c.flops();
}

// BASELINE config 1: single-state RNEA latency of the reference path (the
// mask-vectorised rnea, dynamics.hpp:250-267) as PAPER.md:312 measures it —
// CLOCK_MONOTONIC around each call, `iters` calls on one seeded random state
// (batch.hpp:48-75 draw order), median in nanoseconds.  Test infrastructure:
// bench.py's CPU leg only.
double orc_rnea_latency_ns(void* h, int iters, uint64_t seed) {
  const Model& m = M(h);
  const int n = m.dof();
  std::vector<double> q(n), qd(n), qdd(n);
  orc_random_states(h, 1, seed, q.data(), qd.data(), qdd.data(), nullptr);
  std::vector<double> ns((size_t)std::max(iters, 1));
  volatile double sink = 0;
  for (size_t k = 0; k < ns.size(); ++k) {
    timespec a, b;
    clock_gettime(CLOCK_MONOTONIC, &a);
    const std::vector<double> t = rnea<double>(m, q, qd, qdd, Gravity::standard(), ExtForces<double>());
    clock_gettime(CLOCK_MONOTONIC, &b);
    sink = sink + t[0];
    ns[k] = (double)(b.tv_sec - a.tv_sec) * 1e9 + (double)(b.tv_nsec - a.tv_nsec);
  }
  std::nth_element(ns.begin(), ns.begin() + ns.size() / 2, ns.end());
  return ns[ns.size() / 2];
}

}  // extern "C"
