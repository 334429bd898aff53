// C++ host API (include/vecdyn_b200/vecdyn.hpp) used the way a reference
// vecdyn user would: builtin robots, random_states, batch_* on host buffers.
// Checks the FD∘ID roundtrip (test_dynamics.cpp:335-351), CRBA symmetry and
// the error mapping; exit code 0 on success.
#include <cmath>
#include <cstdio>

#include "vecdyn_b200/vecdyn.hpp"

int main() {
  using namespace vecdyn;
  int bad = 0;
  for (const char* name : {"chain7", "tree29"}) {
    const RobotModel model = robots::by_name(name);
    StateBatch b = random_states(model, 20000, 2604, true, false);
    const std::vector<double> tau = batch_rnea(model, b);
    StateBatch fd = b;
    fd.tau = tau;
    const std::vector<double> qdd = batch_forward_dynamics(model, fd);
    const int n = model.dof();
    double worst = 0;
    int counted = 0;
    for (int64_t i = 0; i < b.N; ++i) {
      if (n == 29 && std::abs(std::cos(b.q[4 * b.N + i])) < 0.05) continue;  // Euler-stack gimbal lock
      double num = 0, den = 1;
      for (int j = 0; j < n; ++j) {
        num = std::max(num, std::abs(qdd[j * b.N + i] - b.qdd[j * b.N + i]));
        den = std::max(den, std::abs(b.qdd[j * b.N + i]));
      }
      worst = std::max(worst, num / den);
      ++counted;
    }
    const std::vector<double> M = batch_crba(model, b);
    double asym = 0;
    for (int64_t i = 0; i < b.N; i += 97)
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) asym = std::max(asym, std::abs(M[(c * n + r) * b.N + i] - M[(r * n + c) * b.N + i]));
    // crba_pattern: every entry outside it (and its mirror) is an exact zero of M
    const auto [rows, cols] = model.crba_pattern();
    std::vector<char> keep((size_t)n * n, 0);
    for (size_t k = 0; k < rows.size(); ++k) keep[(size_t)cols[k] * n + rows[k]] = keep[(size_t)rows[k] * n + cols[k]] = 1;
    for (int64_t i = 0; i < b.N; i += 97)
      for (int e = 0; e < n * n; ++e)
        if (!keep[(size_t)e] && M[(size_t)e * b.N + i] != 0.0) ++bad;
    if (rows.size() != (n == 7 ? 28u : 242u)) ++bad;
    std::printf("%s: FD(ID) roundtrip max rel err %.3e over %d states, CRBA asymmetry %.1e\n", name, worst, counted, asym);
    if (!(worst <= 1e-8) || asym != 0.0) ++bad;
  }
  try {
    (void)robots::chain7().frame_index("nope");
    ++bad;
  } catch (const UnknownFrameError&) {
  }
  try {
    (void)urdf::load_model_from_string("<a>\n  <b>\n  </c>\n</a>");
    ++bad;
  } catch (const ParseError& e) {
    if (e.line != 3 || e.column != 3) ++bad;
  }
  std::printf(bad ? "FAIL\n" : "OK\n");
  return bad;
}
