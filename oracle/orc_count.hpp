// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Op-counting scalar (a Dual-style scalar, cf. proj/core/include/vecdyn/dual.hpp:14-42):
// instantiating the oracle's recursive algorithms (rnea_loop, crba_loop,
// aba_loop, forward_kinematics) with it freezes their ALGORITHMIC flop count
// per evaluation — the implementation-independent numerator of the roofline
// (SURVEY §8d).  Every +, −, ×, ÷ is one flop; sqrt and sin/cos are counted
// separately (transcendental calls).
#pragma once

#include <cmath>
#include <cstdint>

namespace orc {

struct OpCount {
  uint64_t add = 0, mul = 0, div = 0, sqrt = 0, trig = 0;
  uint64_t flops() const { return add + mul + div; }
};
inline OpCount& op_count() {
  static thread_local OpCount c;
  return c;
}

struct Counted {
  double v = 0.0;
  Counted() = default;
  Counted(double x) : v(x) {}  // NOLINT: implicit like a scalar
  explicit operator double() const { return v; }
};
inline Counted operator+(Counted a, Counted b) { ++op_count().add; return Counted(a.v + b.v); }
inline Counted operator-(Counted a, Counted b) { ++op_count().add; return Counted(a.v - b.v); }
inline Counted operator*(Counted a, Counted b) { ++op_count().mul; return Counted(a.v * b.v); }
inline Counted operator/(Counted a, Counted b) { ++op_count().div; return Counted(a.v / b.v); }
inline Counted operator-(Counted a) { return Counted(-a.v); }
inline Counted& operator+=(Counted& a, Counted b) { return a = a + b; }
inline Counted& operator-=(Counted& a, Counted b) { return a = a - b; }
inline bool operator>(Counted a, Counted b) { return a.v > b.v; }
inline bool operator<(Counted a, Counted b) { return a.v < b.v; }
inline bool operator<=(Counted a, Counted b) { return a.v <= b.v; }
inline bool operator>=(Counted a, Counted b) { return a.v >= b.v; }
inline bool operator==(Counted a, Counted b) { return a.v == b.v; }
inline bool operator!=(Counted a, Counted b) { return a.v != b.v; }
inline Counted sqrt(Counted a) { ++op_count().sqrt; return Counted(std::sqrt(a.v)); }
inline Counted sin(Counted a) { ++op_count().trig; return Counted(std::sin(a.v)); }
inline Counted cos(Counted a) { ++op_count().trig; return Counted(std::cos(a.v)); }

// Structure-aware variant: an operation with an exactly-zero operand (x·0,
// x + 0) or a unit factor (x·±1) is not counted — the flops that remain are
// those of the recursion on the robot's actual structure (axis-aligned joints,
// permutation-like offsets, sparse inertias).  Evaluated at generic non-zero
// states, so only STRUCTURAL zeros/units are discounted.
struct Sparse {
  double v = 0.0;
  Sparse() = default;
  Sparse(double x) : v(x) {}  // NOLINT
  explicit operator double() const { return v; }
};
inline bool trivial_mul(double a) { return a == 0.0 || a == 1.0 || a == -1.0; }
inline Sparse operator+(Sparse a, Sparse b) {
  if (a.v != 0.0 && b.v != 0.0) ++op_count().add;
  return Sparse(a.v + b.v);
}
inline Sparse operator-(Sparse a, Sparse b) {
  if (a.v != 0.0 && b.v != 0.0) ++op_count().add;
  return Sparse(a.v - b.v);
}
inline Sparse operator*(Sparse a, Sparse b) {
  if (!trivial_mul(a.v) && !trivial_mul(b.v)) ++op_count().mul;
  return Sparse(a.v * b.v);
}
inline Sparse operator/(Sparse a, Sparse b) {
  if (b.v != 1.0 && b.v != -1.0 && a.v != 0.0) ++op_count().div;
  return Sparse(a.v / b.v);
}
inline Sparse operator-(Sparse a) { return Sparse(-a.v); }
inline Sparse& operator+=(Sparse& a, Sparse b) { return a = a + b; }
inline Sparse& operator-=(Sparse& a, Sparse b) { return a = a - b; }
inline bool operator>(Sparse a, Sparse b) { return a.v > b.v; }
inline bool operator<(Sparse a, Sparse b) { return a.v < b.v; }
inline bool operator<=(Sparse a, Sparse b) { return a.v <= b.v; }
inline bool operator>=(Sparse a, Sparse b) { return a.v >= b.v; }
inline bool operator==(Sparse a, Sparse b) { return a.v == b.v; }
inline bool operator!=(Sparse a, Sparse b) { return a.v != b.v; }
inline Sparse sqrt(Sparse a) { ++op_count().sqrt; return Sparse(std::sqrt(a.v)); }
inline Sparse sin(Sparse a) { ++op_count().trig; return Sparse(std::sin(a.v)); }
inline Sparse cos(Sparse a) { ++op_count().trig; return Sparse(std::cos(a.v)); }

}  // namespace orc
