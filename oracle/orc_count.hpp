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

}  // namespace orc
