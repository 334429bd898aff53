// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A tiny self-registering test harness (doctest is not available: the
// reference's vendor/ directory is absent, proj/.gitignore:2) plus the
// fixtures of proj/tests/helpers.hpp restated over the oracle types.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "../orc_batch.hpp"

namespace port {

struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* s, const char* n, void (*f)()) { registry().push_back({s, n, f}); }
};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}

#define PT_CAT2(a, b) a##b
#define PT_CAT(a, b) PT_CAT2(a, b)
#define TEST(suite, name)                                                      \
  static void PT_CAT(pt_fn_, __LINE__)();                                      \
  static ::port::Reg PT_CAT(pt_reg_, __LINE__)(suite, name, &PT_CAT(pt_fn_, __LINE__)); \
  static void PT_CAT(pt_fn_, __LINE__)()

#define CHECK(cond)                                                                  \
  do {                                                                               \
    ++::port::checks();                                                              \
    if (!(cond)) {                                                                   \
      ++::port::failures();                                                          \
      std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                                \
  } while (0)

#define CHECK_THROWS(expr, Type)                                                     \
  do {                                                                               \
    ++::port::checks();                                                              \
    bool pt_ok = false;                                                              \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const Type&) {                                                          \
      pt_ok = true;                                                                  \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!pt_ok) {                                                                    \
      ++::port::failures();                                                          \
      std::printf("    CHECK_THROWS failed %s:%d: %s !-> %s\n", __FILE__, __LINE__, #expr, #Type); \
    }                                                                                \
  } while (0)

// ----------------------------------------------------------- helpers.hpp:15-150
using Rng = std::mt19937_64;
using orc::Dense;
using orc::Force;
using orc::M3;
using orc::Mat6;
using orc::Motion;
using orc::V3;
using orc::Xform;
using Vec = std::vector<double>;

inline double uniform(Rng& r, double lo = -1.0, double hi = 1.0) {
  return std::uniform_real_distribution<double>(lo, hi)(r);
}
inline V3<double> random_vec3(Rng& r, double s = 1.0) {
  const double a = uniform(r), b = uniform(r), c = uniform(r);
  return V3<double>(a, b, c) * s;
}
inline Vec random_vector(Rng& r, int n, double s = M_PI) {
  Vec v((size_t)n);
  for (int i = 0; i < n; ++i) v[(size_t)i] = uniform(r, -s, s);
  return v;
}
inline V3<double> normalized(const V3<double>& v) { return v * (1.0 / orc::norm3(v)); }
inline M3<double> random_rotation(Rng& r) {
  const V3<double> ax = normalized(random_vec3(r));
  return orc::axis_angle_rotation<double>(ax, uniform(r, -M_PI, M_PI));
}
inline M3<double> test_rotation(double a) {
  return orc::axis_angle_rotation<double>(normalized(V3<double>(1, 2, 3)), a);
}
inline Xform<double> random_transform(Rng& r, double ts = 1.0) {
  Xform<double> x;
  x.R = random_rotation(r);
  x.p = random_vec3(r, ts);
  return x;
}
inline Motion<double> random_motion(Rng& r) {
  Motion<double> m;
  m.ang = random_vec3(r);
  m.lin = random_vec3(r);
  return m;
}
inline Force<double> random_force(Rng& r) {
  Force<double> f;
  f.mom = random_vec3(r);
  f.frc = random_vec3(r);
  return f;
}
inline M3<double> random_m3(Rng& r) {
  M3<double> a;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a(i, j) = uniform(r);
  return a;
}
inline Mat6<double> random_inertia(Rng& r) {
  const double mass = uniform(r, 0.1, 5.0);
  const V3<double> com = random_vec3(r, 0.3);
  const M3<double> a = random_m3(r);
  const M3<double> rot = a * orc::transpose(a) + 0.05 * M3<double>::identity();
  return orc::inertia_from_params(mass, com, rot);
}

// helpers.hpp:67-72: max|a-b| / max(1, max|a|, max|b|).
inline double rel_err(const Vec& a, const Vec& b) {
  double s = 1e-30, d = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    s = std::max({s, std::abs(a[i]), std::abs(b[i])});
    d = std::max(d, std::abs(a[i] - b[i]));
  }
  return d / std::max(1.0, s);
}
inline Vec flat(const M3<double>& m) {
  Vec v;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) v.push_back(m(r, c));
  return v;
}
inline Vec flat(const V3<double>& m) { return {m[0], m[1], m[2]}; }
inline Vec flat(const Motion<double>& m) { return {m[0], m[1], m[2], m[3], m[4], m[5]}; }
inline Vec flat(const Force<double>& m) { return {m[0], m[1], m[2], m[3], m[4], m[5]}; }
inline Vec flat(const Mat6<double>& m) {
  Vec v;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) v.push_back(m(r, c));
  return v;
}
inline Vec flat(const Dense<double>& m) { return m.d; }
template <class A, class B>
double rel(const A& a, const B& b) {
  return rel_err(flat(a), flat(b));
}
inline double rel(const Vec& a, const Vec& b) { return rel_err(a, b); }

// helpers.hpp:76-92 dense oracles
inline Mat6<double> motion_cross_operator(const Motion<double>& v) {
  Mat6<double> op;
  const M3<double> w = orc::skew(v.ang), l = orc::skew(v.lin);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      op(r, c) = w(r, c);
      op(r + 3, c) = l(r, c);
      op(r + 3, c + 3) = w(r, c);
    }
  return op;
}
inline Mat6<double> motion_transform_operator(const Xform<double>& x) { return orc::motion_operator(x); }
inline Vec mat6_vec(const Mat6<double>& m, const Vec& v) {
  Vec o(6, 0.0);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) o[(size_t)r] += m(r, c) * v[(size_t)c];
  return o;
}

// 4x4 homogeneous FK oracle (helpers.hpp:96-120).
struct H4 {
  double a[4][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}};
};
inline H4 homogeneous(const M3<double>& r, const V3<double>& p) {
  H4 h;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) h.a[i][j] = r(i, j);
    h.a[i][3] = p[i];
  }
  return h;
}
inline H4 mul(const H4& x, const H4& y) {
  H4 o;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += x.a[i][k] * y.a[k][j];
      o.a[i][j] = s;
    }
  return o;
}
inline M3<double> rot_of(const H4& h) {
  M3<double> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = h.a[i][j];
  return r;
}
inline V3<double> pos_of(const H4& h) { return V3<double>(h.a[0][3], h.a[1][3], h.a[2][3]); }
inline std::vector<H4> naive_fk(const orc::Model& m, const Vec& q) {
  std::vector<H4> w((size_t)m.dof());
  for (int i = 0; i < m.dof(); ++i) {
    const orc::Joint& j = m.joints[(size_t)i];
    H4 motion;
    if (j.type == orc::JointType::Revolute)
      motion = homogeneous(orc::axis_angle_rotation<double>(j.axis, q[(size_t)i]), V3<double>());
    else
      motion = homogeneous(M3<double>::identity(), j.axis * q[(size_t)i]);
    const H4 loc = mul(homogeneous(j.offset.R, j.offset.p), motion);
    w[(size_t)i] = j.parent < 0 ? loc : mul(w[(size_t)j.parent], loc);
  }
  return w;
}

// helpers.hpp:124-150 random_tree (zero-padded names keep creation order).
inline orc::Description random_tree(Rng& r, int n, double branchiness = 0.5) {
  orc::Description d;
  d.name = "random_tree";
  {
    const double mass = uniform(r, 0.5, 2.0);
    const V3<double> com = random_vec3(r, 0.1);
    const double s = uniform(r, 0.01, 0.1);
    d.add_link("link0", mass, com, s * M3<double>::identity());
  }
  for (int i = 1; i <= n; ++i) {
    const std::string link = "link" + std::to_string(i);
    const M3<double> a = random_m3(r);
    const double mass = uniform(r, 0.2, 3.0);
    const V3<double> com = random_vec3(r, 0.15);
    d.add_link(link, mass, com, 0.05 * (a * orc::transpose(a) + 0.02 * M3<double>::identity()));
    int parent = i - 1;
    if (uniform(r, 0.0, 1.0) < branchiness && i > 1) parent = (int)uniform(r, 0.0, (double)i - 1e-9);
    const orc::JointType t = uniform(r, 0.0, 1.0) < 0.8 ? orc::JointType::Revolute : orc::JointType::Prismatic;
    char nm[16];
    std::snprintf(nm, sizeof nm, "j%03d", i);
    const Xform<double> x = random_transform(r, 0.4);
    const V3<double> ax = normalized(random_vec3(r));
    d.add_joint(nm, t, "link" + std::to_string(parent), link, x, ax);
  }
  return d;
}

inline Vec zeros(int n) { return Vec((size_t)n, 0.0); }
inline Vec basis(int n, int i) {
  Vec v((size_t)n, 0.0);
  v[(size_t)i] = 1.0;
  return v;
}
inline Vec col(const Dense<double>& m, int c) {
  Vec v((size_t)m.rows);
  for (int r = 0; r < m.rows; ++r) v[(size_t)r] = m(r, c);
  return v;
}

}  // namespace port
