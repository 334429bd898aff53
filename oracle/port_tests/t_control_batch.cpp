// ORACLE — TEST INFRASTRUCTURE ONLY.
// The reference has no tests for control.hpp / batch.hpp; these
// implement the examples SPEC.md states for them,
// plus the ABA-vs-LLT cross-check for the oracle's aba_loop.
#include "harness.hpp"

using namespace port;
using namespace orc;

namespace {
Dense<double> solve_spd(Dense<double> A, Dense<double> B) {
  llt_factor(A);
  llt_solve(A, B);
  return B;
}
}  // namespace

TEST("control", "rotation_log inverts axis_angle_rotation (incl. near 0 and pi)") {
  Rng rng(300);
  for (int t = 0; t < 200; ++t) {
    const V3<double> ax = normalized(random_vec3(rng));
    const double ang = t == 0 ? 0.0 : t == 1 ? M_PI - 1e-8 : uniform(rng, 0.0, M_PI - 1e-3);
    const V3<double> w = rotation_log(axis_angle_rotation<double>(ax, ang));
    CHECK(rel(w, ax * ang) < 1e-7);
  }
}

TEST("control", "osc at rest on target with zero posture torque is pure gravity compensation") {
  Rng rng(301);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const std::string fr = m->dof() == 7 ? "ee" : "l_palm";
    for (int t = 0; t < 20; ++t) {
      const Vec q = random_vector(rng, m->dof());
      TaskTarget tg;
      tg.frame = fr;
      tg.pose = frame_transform<double>(*m, forward_kinematics<double>(*m, q), fr);
      tg.gains = TaskGains::uniform(100, 20);
      const Vec tau = osc_step(*m, q, zeros(m->dof()), tg, q, PostureGains{10, 2});
      CHECK(rel(tau, gravity_vector<double>(*m, q)) < 1e-9);
    }
  }
}

TEST("control", "osc null-space projector is dynamically consistent") {
  Rng rng(302);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    const std::string fr = n == 7 ? "ee" : "l_palm";
    for (int t = 0; t < 20; ++t) {
      const Vec q = random_vector(rng, n);
      const Vec tp = random_vector(rng, n, 5.0);
      const auto w = forward_kinematics<double>(*m, q);
      const Dense<double> J = geometric_jacobian<double>(*m, w, fr);
      const Dense<double> M = crba<double>(*m, q);
      Dense<double> Jt(n, 6);
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < 6; ++c) Jt(r, c) = J(c, r);
      const Dense<double> MiJt = solve_spd(M, Jt);
      Dense<double> gram(6, 6);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c)
          for (int k = 0; k < n; ++k) gram(r, c) += J(r, k) * MiJt(k, c);
      Dense<double> MiJt_T(6, n);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < n; ++c) MiJt_T(r, c) = MiJt(c, r);
      const Dense<double> jbar_t = solve_spd(gram, MiJt_T);
      Dense<double> proj(n, 1);  // (1 - Jᵀ J̄ᵀ) τ_post
      double jb[6] = {0, 0, 0, 0, 0, 0};
      for (int r = 0; r < 6; ++r)
        for (int k = 0; k < n; ++k) jb[r] += jbar_t(r, k) * tp[(size_t)k];
      for (int k = 0; k < n; ++k) {
        double s = 0;
        for (int r = 0; r < 6; ++r) s += J(r, k) * jb[r];
        proj(k, 0) = tp[(size_t)k] - s;
      }
      const Dense<double> mp = solve_spd(M, proj);
      Vec task(6, 0.0);
      for (int r = 0; r < 6; ++r)
        for (int k = 0; k < n; ++k) task[(size_t)r] += J(r, k) * mp(k, 0);
      double mx = 0, sc = 1;
      for (double x : task) mx = std::max(mx, std::abs(x));
      for (double x : tp) sc = std::max(sc, std::abs(x));
      CHECK(mx / sc < 1e-8);
    }
  }
}

TEST("control", "osc with zero gains, posture, velocity and gravity gives zero torque") {
  const Model m = robots::chain7();
  Rng rng(303);
  const Vec q = random_vector(rng, 7);
  TaskTarget tg;
  tg.frame = "ee";
  tg.pose = frame_transform<double>(m, forward_kinematics<double>(m, q), "ee");
  const Vec tau = osc_step(m, q, zeros(7), tg, zeros(7), PostureGains{0, 0}, Gravity::zero());
  double mx = 0;
  for (double x : tau) mx = std::max(mx, std::abs(x));
  CHECK(mx < 1e-12);
}

TEST("control", "diff_ik at target with zero feedforward is zero") {
  const Model m = robots::chain7();
  Rng rng(304);
  const Vec q = random_vector(rng, 7);
  TaskTarget tg;
  tg.frame = "ee";
  tg.pose = frame_transform<double>(m, forward_kinematics<double>(m, q), "ee");
  tg.gains = TaskGains::uniform(1.0);
  const Vec qd = diff_ik_step(m, q, tg, 1e-2);
  double mx = 0;
  for (double x : qd) mx = std::max(mx, std::abs(x));
  CHECK(mx < 1e-12);
  CHECK_THROWS(diff_ik_step(m, q, tg, 0.0), Error);
}

TEST("batch", "random_states is reproducible and uniform on [-pi, pi]") {
  const Model m = robots::chain7();
  const StateBatch a = random_states(m, 300, 5, true, true), b = random_states(m, 300, 5, true, true);
  CHECK(a.q == b.q);
  CHECK(a.tau == b.tau);
  double lo = 1e9, hi = -1e9;
  for (double x : a.q) {
    lo = std::min(lo, x);
    hi = std::max(hi, x);
  }
  CHECK(lo >= -M_PI && hi <= M_PI && lo < -3.0 && hi > 3.0);
  const StateBatch c = random_states(m, 300, 6);
  CHECK(a.q != c.q);
  CHECK(c.tau.empty());
}

TEST("batch", "batched outputs are bitwise equal at all worker counts") {
  const Model m = robots::tree29();
  const StateBatch b = random_states(m, 257, 17);
  const int n = m.dof();
  std::vector<Vec> outs;
  for (int workers : {1, 3, 8}) {
    Vec out((size_t)b.N * n);
    batch_eval(b.N,
               [&](int i) {
                 const Vec t = rnea<double>(m, b.row(b.q, i), b.row(b.qd, i), b.row(b.qdd, i));
                 for (int j = 0; j < n; ++j) out[(size_t)j * b.N + i] = t[(size_t)j];
               },
               workers);
    outs.push_back(out);
  }
  CHECK(outs[0] == outs[1]);
  CHECK(outs[0] == outs[2]);
  // N = 1 equals the direct call
  const Vec direct = rnea<double>(m, b.row(b.q, 0), b.row(b.qd, 0), b.row(b.qdd, 0));
  bool same = true;
  for (int j = 0; j < n; ++j) same &= outs[0][(size_t)j * b.N] == direct[(size_t)j];
  CHECK(same);
}

TEST("aba", "aba_loop agrees with the LLT forward dynamics") {
  Rng rng(305);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    for (int t = 0; t < 100; ++t) {
      const Vec q = random_vector(rng, n), qd = random_vector(rng, n), tau = random_vector(rng, n);
      const Vec a = aba_loop<double>(*m, q, qd, tau), b = forward_dynamics<double>(*m, q, qd, tau);
      // Normwise backward error |M q̈ + bias − τ| / (|M| |q̈| + |τ − bias|) of
      // both solutions, and forward agreement away from the Euler-stack
      // gimbal lock of tree29 (base_ry = q[4] near ±π/2, model.hpp:160-162).
      const Dense<double> M = crba<double>(*m, q);
      const Vec bias = rnea<double>(*m, q, qd, zeros(n));
      for (const Vec* sol : {&a, &b}) {
        double res = 0, mn = 0, xn = 0, rn = 0;
        for (int i = 0; i < n; ++i) {
          double s = bias[(size_t)i] - tau[(size_t)i];
          for (int k = 0; k < n; ++k) {
            s += M(i, k) * (*sol)[(size_t)k];
            mn = std::max(mn, std::abs(M(i, k)));
          }
          res = std::max(res, std::abs(s));
          xn = std::max(xn, std::abs((*sol)[(size_t)i]));
          rn = std::max(rn, std::abs(tau[(size_t)i] - bias[(size_t)i]));
        }
        CHECK(res / (mn * xn + rn) < 1e-13);
      }
      if (n == 7 || std::abs(std::cos(q[4])) > 0.05) CHECK(rel(a, b) < 1e-9);
    }
  }
  {  // random trees with external forces and arbitrary gravity
    Rng r2(306);
    for (int t = 0; t < 20; ++t) {
      const Model m = build_model(random_tree(r2, 11, 0.5));
      const int n = m.dof();
      const Vec q = random_vector(r2, n), qd = random_vector(r2, n), qdd = random_vector(r2, n);
      ExtForces<double> f(n);
      for (int i = 0; i < n; ++i) f.w[(size_t)i] = random_force(r2);
      const Gravity g{random_vec3(r2, 5.0)};
      const Vec tau = rnea<double>(m, q, qd, qdd, g, f);
      CHECK(rel(aba_loop<double>(m, q, qd, tau, g, f), qdd) < 1e-8);
    }
  }
}
