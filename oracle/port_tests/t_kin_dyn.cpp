// ORACLE — TEST INFRASTRUCTURE ONLY.
// Port of proj/tests/test_kinematics.cpp and test_dynamics.cpp onto the
// oracle restatement (same seeds and tolerances; Eigen-only checks rewritten
// with the oracle's own dense helpers).
#include "harness.hpp"

using namespace port;
using namespace orc;

namespace {
Vec fd_twist(const Model& m, const Vec& q, const Vec& qd, const std::string& frame, double h) {  // :21-38
  Vec qp = q, qm = q;
  for (size_t i = 0; i < q.size(); ++i) {
    qp[i] += h * qd[i];
    qm[i] -= h * qd[i];
  }
  const Xform<double> p = frame_transform<double>(m, forward_kinematics<double>(m, qp), frame);
  const Xform<double> mi = frame_transform<double>(m, forward_kinematics<double>(m, qm), frame);
  const Xform<double> c = frame_transform<double>(m, forward_kinematics<double>(m, q), frame);
  const M3<double> dr = (1.0 / (2.0 * h)) * (p.R - mi.R);
  const M3<double> w = dr * transpose(c.R);
  Vec t(6);
  t[0] = 0.5 * (w(2, 1) - w(1, 2));
  t[1] = 0.5 * (w(0, 2) - w(2, 0));
  t[2] = 0.5 * (w(1, 0) - w(0, 1));
  for (int k = 0; k < 3; ++k) t[(size_t)(3 + k)] = (p.p[k] - mi.p[k]) / (2.0 * h);
  return t;
}
Vec jac_times(const Dense<double>& J, const Vec& v) {
  Vec o(6, 0.0);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < J.cols; ++c) o[(size_t)r] += J(r, c) * v[(size_t)c];
  return o;
}
Model pendulum(double mass, double len) {  // test_dynamics.cpp:18-25
  Description d;
  d.add_link("base");
  d.add_link("bob", mass, V3<double>(len, 0, 0), M3<double>());
  d.add_joint("pivot", JointType::Revolute, "base", "bob", Xform<double>(), {0, 0, 1});
  return build_model(d);
}
const Gravity kPendulumG = Gravity::from_field(V3<double>(0, -9.81, 0));
Model vertical_prismatic(double mass) {  // test_dynamics.cpp:29-36
  Description d;
  d.add_link("base");
  d.add_link("slider", mass, V3<double>(), M3<double>());
  d.add_joint("lift", JointType::Prismatic, "base", "slider", Xform<double>(), {0, 0, 1});
  return build_model(d);
}
}  // namespace

// ---------------------------------------------------------------- kinematics
TEST("kinematics", "FK matches the naive homogeneous-matrix oracle") {  // :42-56
  Rng rng(100);
  for (int t = 0; t < 20; ++t) {
    const Model m = build_model(random_tree(rng, 7, 0.3));
    const Vec q = random_vector(rng, m.dof());
    const auto w = forward_kinematics<double>(m, q);
    const auto o = naive_fk(m, q);
    for (int i = 0; i < m.dof(); ++i) {
      CHECK(rel(w[(size_t)i].R, rot_of(o[(size_t)i])) < 1e-13);
      CHECK(rel(w[(size_t)i].p, pos_of(o[(size_t)i])) < 1e-13);
    }
  }
}

TEST("kinematics", "all-zero q on identity-offset chain gives identity transforms") {  // :58-75
  Description d;
  d.add_link("l0", 1.0, V3<double>(), 0.01 * M3<double>::identity());
  for (int i = 1; i <= 4; ++i) {
    d.add_link("l" + std::to_string(i), 1.0, V3<double>(), 0.01 * M3<double>::identity());
    d.add_joint("j" + std::to_string(i), JointType::Revolute, "l" + std::to_string(i - 1), "l" + std::to_string(i),
                Xform<double>(), {0, 0, 1});
  }
  const Model m = build_model(d);
  const auto w = forward_kinematics<double>(m, zeros(m.dof()));
  for (int i = 0; i < m.dof(); ++i) {
    CHECK(rel(w[(size_t)i].R, M3<double>::identity()) == 0.0);
    CHECK(norm3(w[(size_t)i].p) == 0.0);
  }
}

TEST("kinematics", "single revolute z joint at pi/2 maps x to y") {  // :77-88
  Description d;
  d.add_link("base");
  d.add_link("spinner", 1.0, V3<double>(), 0.01 * M3<double>::identity());
  d.add_joint("j", JointType::Revolute, "base", "spinner", Xform<double>(), {0, 0, 1});
  const Model m = build_model(d);
  const auto w = forward_kinematics<double>(m, Vec{M_PI / 2});
  CHECK(rel(w[0].R * V3<double>(1, 0, 0), V3<double>(0, 1, 0)) < 1e-15);
}

TEST("kinematics", "FK rotations stay orthonormal on deep chains") {  // :90-103
  Rng rng(101);
  const Model m = build_model(random_tree(rng, 16, 0.0));
  for (int t = 0; t < 50; ++t) {
    const auto w = forward_kinematics<double>(m, random_vector(rng, m.dof()));
    for (int i = 0; i < m.dof(); ++i)
      CHECK(max_abs(transpose(w[(size_t)i].R) * w[(size_t)i].R - M3<double>::identity()) < 1e-10);
  }
}

TEST("kinematics", "scan FK equals sequential FK on serial chains, n = 1..16") {  // :105-120
  Rng rng(102);
  for (int n = 1; n <= 16; ++n) {
    const Model m = build_model(random_tree(rng, n, 0.0));
    CHECK(m.serial);
    for (int t = 0; t < 25; ++t) {
      const Vec q = random_vector(rng, n);
      const auto a = forward_kinematics<double>(m, q), b = forward_kinematics_scan<double>(m, q);
      for (int i = 0; i < n; ++i) {
        CHECK(rel(a[(size_t)i].R, b[(size_t)i].R) < 1e-12);
        CHECK(rel(a[(size_t)i].p, b[(size_t)i].p) < 1e-12);
      }
    }
  }
}

TEST("kinematics", "scan FK rejects branched trees") {  // :122-131
  Rng rng(103);
  Model b = build_model(random_tree(rng, 8, 0.9));
  while (b.serial) b = build_model(random_tree(rng, 8, 0.9));
  CHECK_THROWS(forward_kinematics_scan<double>(b, random_vector(rng, b.dof())), UnsupportedStructureError);
}

TEST("kinematics", "frame transforms") {  // :133-171
  const Model m = robots::chain7();
  {
    Rng rng(104);
    const auto w = forward_kinematics<double>(m, random_vector(rng, m.dof()));
    const Xform<double> l4 = frame_transform<double>(m, w, "link4");
    const int idx = m.joint_index("joint4");
    CHECK(rel(l4.R, w[(size_t)idx].R) == 0.0);
    CHECK(rel(l4.p, w[(size_t)idx].p) == 0.0);
  }
  {
    H4 prod;
    for (int i = 0; i < m.dof(); ++i) prod = mul(prod, homogeneous(m.joints[(size_t)i].offset.R, m.joints[(size_t)i].offset.p));
    prod = mul(prod, homogeneous(m.frame("ee").offset.R, m.frame("ee").offset.p));
    const Xform<double> tool = frame_transform<double>(m, forward_kinematics<double>(m, zeros(7)), "ee");
    CHECK(rel(tool.R, rot_of(prod)) < 1e-14);
    CHECK(rel(tool.p, pos_of(prod)) < 1e-14);
  }
  {
    Rng rng(105);
    const Xform<double> b1 = frame_transform<double>(m, forward_kinematics<double>(m, random_vector(rng, 7)), "base_link");
    const Xform<double> b2 = frame_transform<double>(m, forward_kinematics<double>(m, random_vector(rng, 7)), "base_link");
    CHECK(rel(b1.R, b2.R) == 0.0);
    CHECK(rel(b1.p, b2.p) == 0.0);
  }
  CHECK_THROWS(frame_transform<double>(m, forward_kinematics<double>(m, zeros(7)), "nope"), UnknownFrameError);
}

TEST("kinematics", "geometric jacobian") {  // :173-226
  {
    Rng rng(106);
    const Model chain = robots::chain7();
    const Model tree = build_model(random_tree(rng, 12, 0.5));
    for (const Model* m : {&chain, &tree}) {
      const std::string frame = m->dof() == 7 ? "ee" : m->frames.back().name;
      for (int t = 0; t < 25; ++t) {
        const Vec q = random_vector(rng, m->dof());
        const Vec qd = random_vector(rng, m->dof(), 1.0);
        const Dense<double> J = geometric_jacobian<double>(*m, forward_kinematics<double>(*m, q), frame);
        CHECK(rel(jac_times(J, qd), fd_twist(*m, q, qd, frame, 1e-6)) < 1e-5);
      }
    }
  }
  {
    Rng rng(107);
    Model tree = build_model(random_tree(rng, 12, 0.8));
    while (tree.serial) tree = build_model(random_tree(rng, 12, 0.8));
    const std::string frame = tree.frames.back().name;
    const int target = tree.frame(frame).joint;
    const Dense<double> J =
        geometric_jacobian<double>(tree, forward_kinematics<double>(tree, random_vector(rng, tree.dof())), frame);
    for (int j = 0; j < tree.dof(); ++j) {
      double nrm = 0;
      for (int r = 0; r < 6; ++r) nrm += J(r, j) * J(r, j);
      if (tree.U(target, j) == 0.0) CHECK(nrm == 0.0);
      else CHECK(nrm > 0.0);
    }
  }
  {
    Description d;
    d.add_link("base");
    d.add_link("rod", 1.0, V3<double>(0.25, 0, 0), 0.01 * M3<double>::identity());
    d.add_joint("j", JointType::Revolute, "base", "rod", Xform<double>(), {0, 0, 1});
    d.add_link("tip");
    Xform<double> x;
    x.p = V3<double>(0.5, 0, 0);
    d.add_joint("tip_mount", JointType::Fixed, "rod", "tip", x);
    const Model m = build_model(d);
    const Dense<double> J = geometric_jacobian<double>(m, forward_kinematics<double>(m, zeros(1)), "tip");
    CHECK(rel(col(J, 0), Vec{0, 0, 1, 0, 0.5, 0}) < 1e-15);
  }
}

TEST("kinematics", "manipulability") {  // :228-260
  CHECK(manipulability<double>(Dense<double>(6, 7)) == 0.0);
  Dense<double> J(6, 8);
  for (int i = 0; i < 6; ++i) J(i, i) = 1.0;
  CHECK(std::abs(manipulability<double>(J) - 1.0) < 1e-12);
  Dense<double> ones(6, 3);
  for (double& x : ones.d) x = 1.0;
  CHECK(manipulability<double>(ones) == 0.0);
}

// ---------------------------------------------------------------- dynamics
TEST("dynamics", "prepare_world_arrays") {  // :192-216
  {
    const Model m = pendulum(1.0, 0.5);
    Workspace<double> ws;
    prepare_world_arrays(m, forward_kinematics<double>(m, Vec{1.234}), ws);
    CHECK(rel(ws.S[0], Motion<double>{V3<double>(0, 0, 1), V3<double>()}) < 1e-15);
  }
  {
    Rng rng(200);
    const Model m = build_model(random_tree(rng, 10, 0.4));
    Workspace<double> ws;
    prepare_world_arrays(m, forward_kinematics<double>(m, random_vector(rng, m.dof())), ws);
    for (int i = 0; i < m.dof(); ++i)
      if (m.joints[(size_t)i].type == JointType::Prismatic) {
        CHECK(norm3(ws.S[(size_t)i].ang) == 0.0);
        CHECK(std::abs(norm3(ws.S[(size_t)i].lin) - 1.0) < 1e-12);
      }
  }
}

TEST("dynamics", "rnea zero state with zero gravity gives zero torque") {  // :218-228
  const Model m = robots::chain7();
  Rng rng(201);
  const Vec q = random_vector(rng, 7), z = zeros(7);
  const Vec tau = rnea<double>(m, q, z, z, Gravity::zero());
  double mx = 0;
  for (double x : tau) mx = std::max(mx, std::abs(x));
  CHECK(mx < 1e-14);
  CHECK(rel(rnea_loop<double>(m, q, z, z, Gravity::zero()), tau) < 1e-14);
}

TEST("dynamics", "pendulum gravity torque is m g L cos q") {  // :230-247
  const double mass = 1.7, len = 0.6;
  const Model m = pendulum(mass, len);
  for (double a : {0.0, 0.3, -1.2, M_PI / 3, 2.9}) {
    const double want = mass * 9.81 * len * std::cos(a);
    const Vec tau = rnea<double>(m, Vec{a}, zeros(1), zeros(1), kPendulumG);
    CHECK(std::abs(tau[0] - want) < 1e-10 * std::max(1.0, std::abs(want)));
  }
  CHECK(std::abs(gravity_vector<double>(m, Vec{M_PI / 2}, kPendulumG)[0]) < 1e-10);
}

TEST("dynamics", "vertical prismatic joint") {  // :249-260
  const Model m = vertical_prismatic(2.5);
  CHECK(std::abs(gravity_vector<double>(m, zeros(1))[0] - 2.5 * 9.81) < 1e-14 * 2.5 * 9.81);
  CHECK(std::abs(forward_dynamics<double>(m, zeros(1), zeros(1), zeros(1))[0] + 9.81) < 1e-12);
}

TEST("dynamics", "vectorized and loop dynamics agree to 1e-9 over random states") {  // :262-281
  Rng rng(202);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    double wr = 0, wc = 0;
    for (int t = 0; t < 250; ++t) {
      const Vec q = random_vector(rng, n), qd = random_vector(rng, n), qdd = random_vector(rng, n);
      wr = std::max(wr, rel(rnea<double>(*m, q, qd, qdd), rnea_loop<double>(*m, q, qd, qdd)));
      wc = std::max(wc, rel(crba<double>(*m, q), crba_loop<double>(*m, q)));
    }
    CHECK(wr < 1e-9);
    CHECK(wc < 1e-9);
  }
}

TEST("dynamics", "vectorized and loop dynamics agree on random trees with external forces") {  // :283-299
  Rng rng(203);
  for (int t = 0; t < 20; ++t) {
    const Model m = build_model(random_tree(rng, 11, 0.5));
    const int n = m.dof();
    const Vec q = random_vector(rng, n), qd = random_vector(rng, n), qdd = random_vector(rng, n);
    ExtForces<double> f(n);
    for (int i = 0; i < n; ++i) f.w[(size_t)i] = random_force(rng);
    const Gravity g{random_vec3(rng, 5.0)};
    CHECK(rel(rnea<double>(m, q, qd, qdd, g, f), rnea_loop<double>(m, q, qd, qdd, g, f)) < 1e-9);
  }
}

TEST("dynamics", "crba identities") {  // :301-369
  Rng rng(204);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    for (int t = 0; t < 20; ++t) {
      const Vec q = random_vector(rng, n);
      const Dense<double> M = crba<double>(*m, q);
      for (int i = 0; i < n; ++i)
        CHECK(rel(col(M, i), rnea<double>(*m, q, zeros(n), basis(n, i), Gravity::zero())) < 1e-9);
    }
  }
  {
    const double mass = 1.3, len = 0.4;
    const Model m = pendulum(mass, len);
    const Dense<double> M = crba<double>(m, Vec{0.77});
    CHECK(std::abs(M(0, 0) - m.inertias[0](2, 2)) < 1e-14 * std::abs(M(0, 0)));
    CHECK(std::abs(M(0, 0) - mass * len * len) < 1e-14 * std::abs(M(0, 0)));
  }
  for (const Model* m : {&chain, &tree}) {
    for (int t = 0; t < 50; ++t) {
      Dense<double> M = crba<double>(*m, random_vector(rng, m->dof()));
      Dense<double> Mt(M.rows, M.cols);
      for (int r = 0; r < M.rows; ++r)
        for (int c = 0; c < M.cols; ++c) Mt(r, c) = M(c, r);
      CHECK(rel(M, Mt) < 1e-10);
      CHECK(llt_factor(M));
    }
  }
  for (int t = 0; t < 200; ++t) {  // PD at many states (LLT success == all eigenvalues > 0)
    Dense<double> M = crba<double>(tree, random_vector(rng, tree.dof()));
    CHECK(llt_factor(M));
  }
  {
    const Vec q = random_vector(rng, tree.dof());
    const Dense<double> M = crba<double>(tree, q), Ml = crba_loop<double>(tree, q);
    int decoupled = 0;
    for (int i = 0; i < tree.dof(); ++i)
      for (int j = 0; j < tree.dof(); ++j)
        if (tree.U(i, j) == 0.0 && tree.U(j, i) == 0.0) {
          CHECK(M(i, j) == 0.0);
          CHECK(Ml(i, j) == 0.0);
          ++decoupled;
        }
    CHECK(decoupled > 0);
  }
}

TEST("dynamics", "energy identity ties rnea velocities to the crba mass matrix") {  // :397-422
  Rng rng(206);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    for (int t = 0; t < 100; ++t) {
      const Vec q = random_vector(rng, n), qd = random_vector(rng, n);
      Workspace<double> ws;
      rnea<double>(*m, q, qd, zeros(n), Gravity::zero(), ExtForces<double>(), &ws);
      double es = 0;
      for (int i = 0; i < n; ++i) es += 0.5 * dot(apply(ws.I[(size_t)i], ws.V[(size_t)i]), ws.V[(size_t)i]);
      const Dense<double> M = crba_from_workspace(*m, ws);
      double em = 0;
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) em += 0.5 * qd[(size_t)r] * M(r, c) * qd[(size_t)c];
      CHECK(std::abs(es - em) / std::max(1.0, std::abs(em)) < 1e-10);
    }
  }
}

TEST("dynamics", "coriolis vector") {  // :424-443
  Rng rng(207);
  const Model m = robots::chain7();
  const Vec c0 = coriolis_vector<double>(m, random_vector(rng, 7), zeros(7));
  double mx = 0;
  for (double x : c0) mx = std::max(mx, std::abs(x));
  CHECK(mx < 1e-14);
  for (int t = 0; t < 25; ++t) {
    const Vec q = random_vector(rng, 7), qd = random_vector(rng, 7);
    Vec qd2 = qd;
    for (double& x : qd2) x *= 2.0;
    Vec c1 = coriolis_vector<double>(m, q, qd);
    for (double& x : c1) x *= 4.0;
    CHECK(rel(coriolis_vector<double>(m, q, qd2), c1) < 1e-12);
  }
}

TEST("dynamics", "equation-of-motion decomposition") {  // :445-485
  Rng rng(208);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    for (int t = 0; t < 25; ++t) {
      const Vec q = random_vector(rng, n), qd = random_vector(rng, n), qdd = random_vector(rng, n);
      ExtForces<double> f(n);
      for (int i = 0; i < n; ++i)
        if (uniform(rng) > 0.3) f.w[(size_t)i] = random_force(rng);
      const Vec gamma = rnea<double>(*m, q, qd, qdd, Gravity::standard(), f);
      const Dense<double> M = crba<double>(*m, q);
      const Vec c = coriolis_vector<double>(*m, q, qd), g = gravity_vector<double>(*m, q);
      Workspace<double> ws;
      prepare_world_arrays(*m, forward_kinematics<double>(*m, q), ws);
      Vec rec((size_t)n, 0.0);
      for (int j = 0; j < n; ++j) {
        double ext = 0;
        for (int i = 0; i < n; ++i)
          if (m->U(i, j) != 0.0) ext += dot(f.w[(size_t)i], ws.S[(size_t)j]);
        double mq = 0;
        for (int k = 0; k < n; ++k) mq += M(j, k) * qdd[(size_t)k];
        rec[(size_t)j] = mq + c[(size_t)j] + g[(size_t)j] - ext;
      }
      CHECK(rel(gamma, rec) < 1e-9);
    }
  }
}

TEST("dynamics", "forward dynamics") {  // :487-535
  Rng rng(209);
  const Model chain = robots::chain7(), tree = robots::tree29();
  for (const Model* m : {&chain, &tree}) {
    const int n = m->dof();
    for (int t = 0; t < 25; ++t) {
      const Vec q = random_vector(rng, n), qd = random_vector(rng, n), qdd = random_vector(rng, n);
      const Vec tau = rnea<double>(*m, q, qd, qdd);
      CHECK(rel(forward_dynamics<double>(*m, q, qd, tau), qdd) < 1e-8);
    }
  }
  {
    const Vec q = random_vector(rng, 7), qd = random_vector(rng, 7), qdd = random_vector(rng, 7);
    ExtForces<double> f(7);
    const V3<double> pt = random_vec3(rng), fr = random_vec3(rng, 20.0);
    f.add_at_point(6, pt, fr);
    const Vec tau = rnea<double>(chain, q, qd, qdd, Gravity::standard(), f);
    CHECK(rel(forward_dynamics<double>(chain, q, qd, tau, Gravity::standard(), f), qdd) < 1e-8);
  }
  {
    const Vec r = forward_dynamics<double>(chain, zeros(7), zeros(7), zeros(7), Gravity::zero());
    double mx = 0;
    for (double x : r) mx = std::max(mx, std::abs(x));
    CHECK(mx < 1e-12);
  }
  {
    Description d;
    d.add_link("base");
    d.add_link("ghost", 0.0, V3<double>(), M3<double>());
    d.add_joint("j", JointType::Revolute, "base", "ghost", Xform<double>(), {0, 0, 1});
    const Model m = build_model(d);
    CHECK_THROWS(forward_dynamics<double>(m, zeros(1), zeros(1), zeros(1)), SingularInertiaError);
  }
}

TEST("dynamics", "dimension mismatches are rejected") {  // :537-548
  const Model m = robots::chain7();
  const Vec good = zeros(7), bad = zeros(6);
  CHECK_THROWS(rnea<double>(m, bad, good, good), DimensionError);
  CHECK_THROWS(rnea<double>(m, good, bad, good), DimensionError);
  CHECK_THROWS(rnea_loop<double>(m, good, good, bad), DimensionError);
  CHECK_THROWS(crba<double>(m, bad), DimensionError);
  CHECK_THROWS(rnea<double>(m, good, good, good, Gravity::standard(), ExtForces<double>(3)), DimensionError);
}

TEST("dynamics", "single precision instantiation stays within 1e-4 of double") {  // :550-565
  Rng rng(210);
  const Model m = robots::chain7();
  for (int t = 0; t < 10; ++t) {
    const Vec q = random_vector(rng, 7), qd = random_vector(rng, 7), qdd = random_vector(rng, 7);
    const std::vector<float> qf(q.begin(), q.end()), qdf(qd.begin(), qd.end()), qddf(qdd.begin(), qdd.end());
    const std::vector<float> tf = rnea<float>(m, qf, qdf, qddf);
    CHECK(rel(Vec(tf.begin(), tf.end()), rnea<double>(m, q, qd, qdd)) < 1e-4);
    const Dense<float> Mf = crba<float>(m, qf);
    CHECK(rel(Vec(Mf.d.begin(), Mf.d.end()), crba<double>(m, q).d) < 1e-4);
  }
}

TEST("dynamics", "0-dof model yields empty results") {  // :567-576
  Description d;
  d.add_link("base");
  d.add_link("tool");
  d.add_joint("mount", JointType::Fixed, "base", "tool", Xform<double>());
  const Model m = build_model(d);
  CHECK(rnea<double>(m, Vec(), Vec(), Vec()).empty());
  CHECK(crba<double>(m, Vec()).d.empty());
}
