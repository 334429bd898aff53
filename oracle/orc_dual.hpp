// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Forward-mode dual scalar, restating proj/core/include/vecdyn/dual.hpp:14-180
// (value + one directional derivative; comparisons act on values only).  The
// oracle's algorithms are generic over the scalar exactly like the
// reference's, so instantiating them with Dual gives the reference's JVPs
// (autodiff.hpp:41-56).  The Eigen NumTraits block of dual.hpp:186-196 has no
// counterpart here (the oracle's own Dense/LLT are scalar-generic).
#pragma once

#include <cmath>

namespace orc {

struct Dual {
  double value = 0.0;
  double tangent = 0.0;
  Dual() = default;
  Dual(double v) : value(v) {}  // NOLINT: implicit lift of constants (dual.hpp:19)
  Dual(double v, double t) : value(v), tangent(t) {}
  Dual& operator+=(const Dual& o) {
    value += o.value;
    tangent += o.tangent;
    return *this;
  }
  Dual& operator-=(const Dual& o) {
    value -= o.value;
    tangent -= o.tangent;
    return *this;
  }
  Dual& operator*=(const Dual& o) {  // dual.hpp:32-36
    tangent = tangent * o.value + value * o.tangent;
    value *= o.value;
    return *this;
  }
  Dual& operator/=(const Dual& o) {  // dual.hpp:37-41
    tangent = (tangent * o.value - value * o.tangent) / (o.value * o.value);
    value /= o.value;
    return *this;
  }
  explicit operator double() const { return value; }
};

// dual.hpp:44-73
inline Dual operator+(const Dual& a, const Dual& b) { return {a.value + b.value, a.tangent + b.tangent}; }
inline Dual operator-(const Dual& a, const Dual& b) { return {a.value - b.value, a.tangent - b.tangent}; }
inline Dual operator-(const Dual& a) { return {-a.value, -a.tangent}; }
inline Dual operator+(const Dual& a) { return a; }
inline Dual operator*(const Dual& a, const Dual& b) {
  return {a.value * b.value, a.tangent * b.value + a.value * b.tangent};
}
inline Dual operator/(const Dual& a, const Dual& b) {
  return {a.value / b.value, (a.tangent * b.value - a.value * b.tangent) / (b.value * b.value)};
}
inline Dual operator+(const Dual& a, double b) { return {a.value + b, a.tangent}; }
inline Dual operator+(double a, const Dual& b) { return {a + b.value, b.tangent}; }
inline Dual operator-(const Dual& a, double b) { return {a.value - b, a.tangent}; }
inline Dual operator-(double a, const Dual& b) { return {a - b.value, -b.tangent}; }
inline Dual operator*(const Dual& a, double b) { return {a.value * b, a.tangent * b}; }
inline Dual operator*(double a, const Dual& b) { return {a * b.value, a * b.tangent}; }
inline Dual operator/(const Dual& a, double b) { return {a.value / b, a.tangent / b}; }
inline Dual operator/(double a, const Dual& b) { return {a / b.value, -a * b.tangent / (b.value * b.value)}; }

// dual.hpp:75-95 (values only)
inline bool operator==(const Dual& a, const Dual& b) { return a.value == b.value; }
inline bool operator!=(const Dual& a, const Dual& b) { return a.value != b.value; }
inline bool operator<(const Dual& a, const Dual& b) { return a.value < b.value; }
inline bool operator>(const Dual& a, const Dual& b) { return a.value > b.value; }
inline bool operator<=(const Dual& a, const Dual& b) { return a.value <= b.value; }
inline bool operator>=(const Dual& a, const Dual& b) { return a.value >= b.value; }

// dual.hpp:97-180 (the subset the algorithms use, plus the common ones)
inline Dual sin(const Dual& x) { return {std::sin(x.value), std::cos(x.value) * x.tangent}; }
inline Dual cos(const Dual& x) { return {std::cos(x.value), -std::sin(x.value) * x.tangent}; }
inline Dual sqrt(const Dual& x) {
  const double s = std::sqrt(x.value);
  return {s, x.tangent / (2.0 * s)};
}
inline Dual acos(const Dual& x) { return {std::acos(x.value), -x.tangent / std::sqrt(1.0 - x.value * x.value)}; }
inline Dual exp(const Dual& x) {
  const double e = std::exp(x.value);
  return {e, e * x.tangent};
}
inline Dual abs(const Dual& x) { return x.value < 0.0 ? -x : x; }
inline Dual fabs(const Dual& x) { return abs(x); }
inline bool isfinite(const Dual& x) { return std::isfinite(x.value) && std::isfinite(x.tangent); }

}  // namespace orc
