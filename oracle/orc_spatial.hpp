// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Eigen-free CPU restatement of the reference `vecdyn` spatial algebra
// (reference: proj/core/include/vecdyn/spatial.hpp, errors.hpp).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
// this code; the product library (paper_2604_04310_b200/) never links it.
//
// Conventions follow the reference exactly: 6-vectors are angular-first
// (spatial.hpp:41-46), transforms are (R, p) mapping child -> parent
// coordinates x_parent = R x + p (spatial.hpp:129-131), inertias are dense
// 6x6 about the body-frame origin (spatial.hpp:162-163).
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace orc {

// ---------------------------------------------------------------- errors
// errors.hpp:9-61 — same hierarchy, same meaning.
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct ModelError : Error {
  using Error::Error;
};
struct UnknownFrameError : ModelError {
  using ModelError::ModelError;
};
struct ParseError : Error {
  ParseError(const std::string& msg, int l, int c)
      : Error(msg + " (line " + std::to_string(l) + ", column " + std::to_string(c) + ")"),
        line(l),
        column(c) {}
  int line;
  int column;
};
struct UnsupportedFeatureError : Error {
  using Error::Error;
};
struct UnsupportedStructureError : Error {
  using Error::Error;
};
struct SingularInertiaError : Error {
  using Error::Error;
};

// ---------------------------------------------------------------- 3-D
template <class T>
struct V3 {
  T e[3] = {T(0), T(0), T(0)};
  V3() = default;
  V3(T a, T b, T c) { e[0] = a; e[1] = b; e[2] = c; }
  T& operator[](int i) { return e[i]; }
  const T& operator[](int i) const { return e[i]; }
  template <class U>
  V3<U> as() const { return V3<U>(U(e[0]), U(e[1]), U(e[2])); }
};

template <class T> V3<T> operator+(const V3<T>& a, const V3<T>& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
template <class T> V3<T> operator-(const V3<T>& a, const V3<T>& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
template <class T> V3<T> operator-(const V3<T>& a) { return {-a[0], -a[1], -a[2]}; }
template <class T> V3<T> operator*(const V3<T>& a, const T& s) { return {a[0] * s, a[1] * s, a[2] * s}; }
template <class T> V3<T> operator*(const T& s, const V3<T>& a) { return {s * a[0], s * a[1], s * a[2]}; }
template <class T> T dot3(const V3<T>& a, const V3<T>& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
template <class T> V3<T> cross3(const V3<T>& a, const V3<T>& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline double norm3(const V3<double>& a) { return std::sqrt(dot3(a, a)); }

// Row-major 3x3.
template <class T>
struct M3 {
  T a[3][3] = {{T(0), T(0), T(0)}, {T(0), T(0), T(0)}, {T(0), T(0), T(0)}};
  T& operator()(int r, int c) { return a[r][c]; }
  const T& operator()(int r, int c) const { return a[r][c]; }
  static M3 identity() {
    M3 m;
    m(0, 0) = m(1, 1) = m(2, 2) = T(1);
    return m;
  }
  template <class U>
  M3<U> as() const {
    M3<U> m;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) m(r, c) = U(a[r][c]);
    return m;
  }
};

template <class T> V3<T> operator*(const M3<T>& m, const V3<T>& v) {
  V3<T> o;
  for (int r = 0; r < 3; ++r) o[r] = m(r, 0) * v[0] + m(r, 1) * v[1] + m(r, 2) * v[2];
  return o;
}
template <class T> M3<T> operator*(const M3<T>& x, const M3<T>& y) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = x(r, 0) * y(0, c) + x(r, 1) * y(1, c) + x(r, 2) * y(2, c);
  return o;
}
template <class T> M3<T> operator+(const M3<T>& x, const M3<T>& y) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = x(r, c) + y(r, c);
  return o;
}
template <class T> M3<T> operator-(const M3<T>& x, const M3<T>& y) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = x(r, c) - y(r, c);
  return o;
}
template <class T> M3<T> operator*(const T& s, const M3<T>& x) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = s * x(r, c);
  return o;
}
template <class T> M3<T> transpose(const M3<T>& x) {
  M3<T> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = x(c, r);
  return o;
}
// spatial.hpp:30-39
template <class T> M3<T> skew(const V3<T>& v) {
  M3<T> m;
  m(0, 1) = -v[2]; m(0, 2) = v[1];
  m(1, 0) = v[2];  m(1, 2) = -v[0];
  m(2, 0) = -v[1]; m(2, 1) = v[0];
  return m;
}
inline double max_abs(const M3<double>& m) {
  double s = 0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) s = std::max(s, std::abs(m(r, c)));
  return s;
}
inline double det3(const M3<double>& m) {
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) -
         m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
         m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}

// ---------------------------------------------------------------- 6-D
// SpatialMotionT / SpatialForceT, spatial.hpp:43-127.
template <class T>
struct Motion {
  V3<T> ang, lin;
  T operator[](int i) const { return i < 3 ? ang[i] : lin[i - 3]; }
  T& at(int i) { return i < 3 ? ang[i] : lin[i - 3]; }
};
template <class T>
struct Force {
  V3<T> mom, frc;
  T operator[](int i) const { return i < 3 ? mom[i] : frc[i - 3]; }
  T& at(int i) { return i < 3 ? mom[i] : frc[i - 3]; }
};
template <class T> Motion<T> operator+(const Motion<T>& a, const Motion<T>& b) { return {a.ang + b.ang, a.lin + b.lin}; }
template <class T> Motion<T> operator-(const Motion<T>& a, const Motion<T>& b) { return {a.ang - b.ang, a.lin - b.lin}; }
template <class T> Motion<T> operator*(const Motion<T>& a, const T& s) { return {a.ang * s, a.lin * s}; }
template <class T> Force<T> operator+(const Force<T>& a, const Force<T>& b) { return {a.mom + b.mom, a.frc + b.frc}; }
template <class T> Force<T> operator-(const Force<T>& a, const Force<T>& b) { return {a.mom - b.mom, a.frc - b.frc}; }
template <class T> Force<T> operator*(const Force<T>& a, const T& s) { return {a.mom * s, a.frc * s}; }

// SpatialTransformT, spatial.hpp:132-160.
template <class T>
struct Xform {
  M3<T> R = M3<T>::identity();
  V3<T> p;
  static Xform identity() { return Xform(); }
  template <class U>
  Xform<U> as() const { return {R.template as<U>(), p.template as<U>()}; }
};
// Composition (a ∘ b): b expressed in a's local frame.
template <class T> Xform<T> operator*(const Xform<T>& a, const Xform<T>& b) { return {a.R * b.R, a.R * b.p + a.p}; }
template <class T> Xform<T> inverse(const Xform<T>& x) {
  M3<T> rt = transpose(x.R);
  return {rt, -(rt * x.p)};
}

// Dense 6x6, angular-first blocks.  SpatialInertiaT spatial.hpp:164-196.
template <class T>
struct Mat6 {
  T a[6][6];
  Mat6() {
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) a[r][c] = T(0);
  }
  T& operator()(int r, int c) { return a[r][c]; }
  const T& operator()(int r, int c) const { return a[r][c]; }
  template <class U>
  Mat6<U> as() const {
    Mat6<U> m;
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) m(r, c) = U(a[r][c]);
    return m;
  }
};
template <class T> Mat6<T> operator+(const Mat6<T>& x, const Mat6<T>& y) {
  Mat6<T> o;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) o(r, c) = x(r, c) + y(r, c);
  return o;
}
template <class T> Mat6<T> mul6(const Mat6<T>& x, const Mat6<T>& y) {
  Mat6<T> o;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      T s = T(0);
      for (int k = 0; k < 6; ++k) s = s + x(r, k) * y(k, c);
      o(r, c) = s;
    }
  return o;
}
template <class T> Mat6<T> transpose6(const Mat6<T>& x) {
  Mat6<T> o;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) o(r, c) = x(c, r);
  return o;
}
// I * v (inertia applied to a motion gives a force), spatial.hpp:179-182.
template <class T> Force<T> apply(const Mat6<T>& m, const Motion<T>& v) {
  Force<T> f;
  for (int r = 0; r < 6; ++r) {
    T s = T(0);
    for (int k = 0; k < 6; ++k) s = s + m(r, k) * v[k];
    f.at(r) = s;
  }
  return f;
}

// spatial.hpp:204-208
template <class T> Motion<T> cross_motion(const Motion<T>& v, const Motion<T>& m) {
  return {cross3(v.ang, m.ang), cross3(v.ang, m.lin) + cross3(v.lin, m.ang)};
}
// spatial.hpp:212-216
template <class T> Force<T> cross_force(const Motion<T>& v, const Force<T>& f) {
  return {cross3(v.ang, f.mom) + cross3(v.lin, f.frc), cross3(v.ang, f.frc)};
}
// spatial.hpp:219-222
template <class T> T dot(const Force<T>& f, const Motion<T>& m) { return dot3(f.mom, m.ang) + dot3(f.frc, m.lin); }
// spatial.hpp:225-230
template <class T> Motion<T> transform_motion(const Xform<T>& X, const Motion<T>& m) {
  V3<T> w = X.R * m.ang;
  return {w, X.R * m.lin + cross3(X.p, w)};
}
// spatial.hpp:233-238
template <class T> Motion<T> inverse_transform_motion(const Xform<T>& X, const Motion<T>& m) {
  M3<T> rt = transpose(X.R);
  return {rt * m.ang, rt * (m.lin - cross3(X.p, m.ang))};
}
// spatial.hpp:241-246
template <class T> Force<T> transform_force(const Xform<T>& X, const Force<T>& f) {
  V3<T> fr = X.R * f.frc;
  return {X.R * f.mom + cross3(X.p, fr), fr};
}
// spatial.hpp:249-254
template <class T> Force<T> inverse_transform_force(const Xform<T>& X, const Force<T>& f) {
  M3<T> rt = transpose(X.R);
  return {rt * (f.mom - cross3(X.p, f.frc)), rt * f.frc};
}
// Y = [[R, 0], [p× R, R]]: the motion operator of X.  spatial.hpp:259-267 uses
// I' = Y I Yᵀ with Y built exactly this way.
template <class T> Mat6<T> motion_operator(const Xform<T>& X) {
  Mat6<T> y;
  M3<T> pr = skew(X.p) * X.R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      y(r, c) = X.R(r, c);
      y(r + 3, c + 3) = X.R(r, c);
      y(r + 3, c) = pr(r, c);
    }
  return y;
}
// transform_inertia, spatial.hpp:259-267.  NOTE the reference places skew(p)R
// in the *top-right* block of Y (spatial.hpp:264), i.e. Y is the force
// operator [[R, p×R],[0, R]]; I' = Y I Yᵀ is the congruence that maps an
// inertia about the child origin to one about the parent origin.
template <class T> Mat6<T> transform_inertia(const Xform<T>& X, const Mat6<T>& I) {
  Mat6<T> y;
  M3<T> pr = skew(X.p) * X.R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      y(r, c) = X.R(r, c);
      y(r + 3, c + 3) = X.R(r, c);
      y(r, c + 3) = pr(r, c);
    }
  return mul6(mul6(y, I), transpose6(y));
}

// Symmetric 3x3 eigenvalues (cyclic Jacobi); used only for the PSD check of
// inertia_from_params (spatial.hpp:287-290 uses SelfAdjointEigenSolver).
inline double min_eigen_sym3(M3<double> a) {
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = std::abs(a(0, 1)) + std::abs(a(0, 2)) + std::abs(a(1, 2));
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a(p, q) == 0.0) continue;
        double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- A J
          double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // A <- Jᵀ A
          double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
      }
  }
  return std::min({a(0, 0), a(1, 1), a(2, 2)});
}

// spatial.hpp:277-298
inline Mat6<double> inertia_from_params(double mass, const V3<double>& com, const M3<double>& Ic) {
  if (mass < 0.0) throw ModelError("inertia_from_params: negative mass " + std::to_string(mass));
  const double scale = std::max(1.0, max_abs(Ic));
  if (max_abs(Ic - transpose(Ic)) > 1e-9 * scale)
    throw ModelError("inertia_from_params: rotational inertia is not symmetric");
  if (min_eigen_sym3(Ic) < -1e-9 * scale)
    throw ModelError("inertia_from_params: rotational inertia is not positive semidefinite");
  const M3<double> cx = skew(com);
  const M3<double> top = Ic + mass * (cx * transpose(cx));
  const M3<double> tr = mass * cx;
  Mat6<double> m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      m(r, c) = top(r, c);
      m(r, c + 3) = tr(r, c);
      m(r + 3, c) = tr(c, r);
    }
  m(3, 3) = m(4, 4) = m(5, 5) = mass;
  return m;
}

// spatial.hpp:302-308 (Rodrigues).  Generic in the scalar.
template <class T> M3<T> axis_angle_rotation(const V3<double>& axis, const T& angle) {
  using std::cos;
  using std::sin;
  const M3<T> k = skew(axis.as<T>());
  const M3<T> kk = k * k;
  const T s = sin(angle), c1 = T(1) - cos(angle);
  M3<T> out = M3<T>::identity();
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out(r, c) = out(r, c) + s * k(r, c) + c1 * kk(r, c);
  return out;
}

}  // namespace orc
