// ORACLE — TEST INFRASTRUCTURE ONLY.
// Port of the reference suites proj/tests/test_spatial.cpp, test_model.cpp and
// test_urdf.cpp onto the oracle restatement (same seeds, same tolerances).
#include <fstream>
#include <sstream>

#include "harness.hpp"

using namespace port;
using namespace orc;

namespace {
Mat6<double> force_operator(const Xform<double>& x) {  // inverse-transpose of the motion operator
  Mat6<double> op;
  const M3<double> pr = skew(x.p) * x.R;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      op(r, c) = x.R(r, c);
      op(r + 3, c + 3) = x.R(r, c);
      op(r, c + 3) = pr(r, c);
    }
  return op;
}
Vec neg(Vec v) {
  for (double& x : v) x = -x;
  return v;
}
}  // namespace

// ---------------------------------------------------------------- test_spatial.cpp
TEST("spatial", "cross_motion matches the dense 6x6 operator") {  // :11-19
  Rng rng(42);
  for (int t = 0; t < 100; ++t) {
    const Motion<double> v = random_motion(rng), m = random_motion(rng);
    CHECK(rel(flat(cross_motion(v, m)), mat6_vec(motion_cross_operator(v), flat(m))) < 1e-14);
  }
}

TEST("spatial", "self-cross and zero-cross vanish") {  // :21-27
  Rng rng(1);
  const Motion<double> v = random_motion(rng);
  const Vec c = flat(cross_motion(v, v));
  double nrm = 0;
  for (double x : c) nrm += x * x;
  CHECK(std::sqrt(nrm) < 1e-15);
  const Vec z = flat(cross_force(Motion<double>(), random_force(rng)));
  CHECK(rel(z, zeros(6)) == 0.0);
}

TEST("spatial", "cross_force matches minus the transposed motion operator") {  // :29-37
  Rng rng(43);
  for (int t = 0; t < 100; ++t) {
    const Motion<double> v = random_motion(rng);
    const Force<double> f = random_force(rng);
    CHECK(rel(flat(cross_force(v, f)), neg(mat6_vec(transpose6(motion_cross_operator(v)), flat(f)))) < 1e-14);
  }
}

TEST("spatial", "adjoint identity <v x* f, m> + <f, v x m> = 0") {  // :39-49
  Rng rng(44);
  for (int t = 0; t < 200; ++t) {
    const Motion<double> v = random_motion(rng), m = random_motion(rng);
    const Force<double> f = random_force(rng);
    const double lhs = dot(cross_force(v, f), m) + dot(f, cross_motion(v, m));
    CHECK(std::abs(lhs) / std::max(1.0, std::abs(dot(f, cross_motion(v, m)))) < 1e-12);
  }
}

TEST("spatial", "transforms match the dense Plücker operators") {  // :51-71
  Rng rng(45);
  for (int t = 0; t < 100; ++t) {
    const Xform<double> x = random_transform(rng);
    const Mat6<double> xm = motion_transform_operator(x), xf = force_operator(x);
    const Mat6<double> xm_inv = motion_transform_operator(inverse(x)), xf_inv = force_operator(inverse(x));
    const Motion<double> m = random_motion(rng);
    CHECK(rel(flat(transform_motion(x, m)), mat6_vec(xm, flat(m))) < 1e-12);
    CHECK(rel(flat(inverse_transform_motion(x, m)), mat6_vec(xm_inv, flat(m))) < 1e-12);
    const Force<double> f = random_force(rng);
    CHECK(rel(flat(transform_force(x, f)), mat6_vec(xf, flat(f))) < 1e-12);
    CHECK(rel(flat(inverse_transform_force(x, f)), mat6_vec(xf_inv, flat(f))) < 1e-12);
    const Mat6<double> I = random_inertia(rng);
    CHECK(rel(transform_inertia(x, I), mul6(mul6(xf, I), transpose6(xf))) < 1e-12);
  }
}

TEST("spatial", "identity transform is a no-op") {  // :73-80
  Rng rng(46);
  const Motion<double> m = random_motion(rng);
  CHECK(rel(transform_motion(Xform<double>::identity(), m), m) == 0.0);
  const Mat6<double> I = random_inertia(rng);
  CHECK(rel(transform_inertia(Xform<double>::identity(), I), I) < 1e-15);
}

TEST("spatial", "kinetic energy and power are frame invariant") {  // :92-111
  Rng rng(47);
  for (int t = 0; t < 200; ++t) {
    const Xform<double> x = random_transform(rng);
    const Motion<double> v = random_motion(rng);
    const Force<double> f = random_force(rng);
    const Mat6<double> I = random_inertia(rng);
    const double e0 = 0.5 * dot(apply(I, v), v);
    const Motion<double> v2 = transform_motion(x, v);
    const double e1 = 0.5 * dot(apply(transform_inertia(x, I), v2), v2);
    CHECK(std::abs(e0 - e1) / std::max(1.0, std::abs(e0)) < 1e-12);
    const double p0 = dot(f, v), p1 = dot(transform_force(x, f), v2);
    CHECK(std::abs(p0 - p1) / std::max(1.0, std::abs(p0)) < 1e-12);
  }
}

TEST("spatial", "transform composition") {  // :126-138
  Rng rng(49);
  for (int t = 0; t < 50; ++t) {
    const Xform<double> a = random_transform(rng), b = random_transform(rng);
    const Motion<double> m = random_motion(rng);
    CHECK(rel(transform_motion(a * b, m), transform_motion(a, transform_motion(b, m))) < 1e-13);
    const Xform<double> rt = (a * b) * inverse(a * b);
    CHECK(rel(rt.R, M3<double>::identity()) < 1e-13);
    CHECK(norm3(rt.p) < 1e-13);
  }
}

TEST("spatial", "inertia_from_params") {  // :140-173
  CHECK(rel(inertia_from_params(0.0, V3<double>(0.3, 0.1, -0.2), M3<double>()), Mat6<double>()) == 0.0);
  Mat6<double> pm;
  pm(3, 3) = pm(4, 4) = pm(5, 5) = 2.5;
  CHECK(rel(inertia_from_params(2.5, V3<double>(), M3<double>()), pm) == 0.0);
  Rng rng(50);
  for (int t = 0; t < 50; ++t) {
    const double mass = uniform(rng, 0.1, 4.0);
    const V3<double> com = random_vec3(rng);
    const Mat6<double> I = inertia_from_params(mass, com, M3<double>());
    Motion<double> v;
    v.ang = random_vec3(rng);
    const double e = 0.5 * dot(apply(I, v), v);
    const V3<double> wc = cross3(v.ang, com);
    const double want = 0.5 * mass * dot3(wc, wc);
    CHECK(std::abs(e - want) < 1e-12 * std::max(1.0, want));
  }
  CHECK_THROWS(inertia_from_params(-1.0, V3<double>(), M3<double>()), ModelError);
  M3<double> asym = M3<double>::identity();
  asym(0, 1) = 0.5;
  CHECK_THROWS(inertia_from_params(1.0, V3<double>(), asym), ModelError);
}

// ---------------------------------------------------------------- test_model.cpp
namespace {
std::vector<double> closure(const std::vector<int>& parents) {
  const size_t n = parents.size();
  std::vector<double> u(n * n, 0.0);
  for (size_t i = 0; i < n; ++i)
    for (int j = (int)i; j >= 0; j = parents[(size_t)j]) u[i * n + (size_t)j] = 1.0;
  return u;
}
Description two_link_chain() {  // test_model.cpp:30-43
  Description d;
  d.name = "two_link";
  d.add_link("base", 1.5, V3<double>(0, 0, 0.05), 0.02 * M3<double>::identity());
  d.add_link("l1", 1.0, V3<double>(0.1, 0, 0), 0.01 * M3<double>::identity());
  d.add_link("l2", 0.8, V3<double>(0.1, 0, 0), 0.01 * M3<double>::identity());
  Xform<double> a, b;
  a.p = V3<double>(0, 0, 0.1);
  b.p = V3<double>(0.3, 0, 0);
  d.add_joint("a", JointType::Revolute, "base", "l1", a, {0, 0, 1});
  d.add_joint("b", JointType::Revolute, "l1", "l2", b, {0, 1, 0});
  return d;
}
}  // namespace

TEST("model", "ancestor mask examples") {  // :47-76
  CHECK(build_ancestor_mask({-1, 0, 1}) == (std::vector<double>{1, 0, 0, 1, 1, 0, 1, 1, 1}));
  CHECK(build_ancestor_mask({-1, 0, 0}) == (std::vector<double>{1, 0, 0, 1, 1, 0, 1, 0, 1}));
  CHECK(build_ancestor_mask({-1}) == (std::vector<double>{1}));
  CHECK(build_ancestor_mask({-1, -1, 1}) == (std::vector<double>{1, 0, 0, 0, 1, 0, 0, 1, 1}));
  CHECK_THROWS(build_ancestor_mask({-1, 2, 1}), ModelError);
  CHECK_THROWS(build_ancestor_mask({0}), ModelError);
  CHECK_THROWS(build_ancestor_mask({-1, -2}), ModelError);
}

TEST("model", "ancestor mask equals brute-force transitive closure on random trees") {  // :78-107
  Rng rng(123);
  for (int t = 0; t < 50; ++t) {
    const int n = 1 + (int)uniform(rng, 0.0, 31.0);
    std::vector<int> parents((size_t)n);
    parents[0] = -1;
    for (int i = 1; i < n; ++i)
      parents[(size_t)i] = uniform(rng, 0.0, 1.0) < 0.05 ? -1 : (int)uniform(rng, 0.0, (double)i - 1e-9);
    const std::vector<double> mask = build_ancestor_mask(parents);
    CHECK(mask == closure(parents));
    // sat((A + 1)^n) reaches the same closure.
    std::vector<double> a((size_t)n * n, 0.0), pw((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) {
      a[(size_t)i * n + i] = 1.0;
      pw[(size_t)i * n + i] = 1.0;
      if (parents[(size_t)i] >= 0) a[(size_t)i * n + parents[(size_t)i]] = 1.0;
    }
    for (int k = 0; k < n; ++k) {
      std::vector<double> nx((size_t)n * n, 0.0);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int l = 0; l < n; ++l) nx[(size_t)i * n + j] += pw[(size_t)i * n + l] * a[(size_t)l * n + j];
      pw = nx;
    }
    bool same = true;
    for (size_t k = 0; k < pw.size(); ++k) same &= ((pw[k] > 0.0) ? 1.0 : 0.0) == mask[k];
    CHECK(same);
  }
}

TEST("model", "build_model fuses fixed joints") {  // :109-139
  Description d;
  d.add_link("base");
  d.add_link("l1", 1.0, V3<double>(), 0.01 * M3<double>::identity());
  d.add_link("l2", 0.5, V3<double>(0.05, 0, 0), 0.005 * M3<double>::identity());
  d.add_link("l3", 0.7, V3<double>(), 0.002 * M3<double>::identity());
  Xform<double> x1{test_rotation(0.3), V3<double>(0, 0, 0.2)};
  Xform<double> xf{test_rotation(-0.8), V3<double>(0.1, 0.05, 0)};
  Xform<double> x2{test_rotation(1.1), V3<double>(0, 0.2, 0)};
  d.add_joint("j1", JointType::Revolute, "base", "l1", x1, {0, 0, 1});
  d.add_joint("jf", JointType::Fixed, "l1", "l2", xf);
  d.add_joint("j2", JointType::Revolute, "l2", "l3", x2, {0, 1, 0});
  const Model m = build_model(d);
  CHECK(m.dof() == 2);
  const Xform<double> want = xf * x2;
  CHECK(rel(m.joints[1].offset.R, want.R) < 1e-15);
  CHECK(rel(m.joints[1].offset.p, want.p) < 1e-15);
  const Mat6<double> folded =
      inertia_from_params(1.0, V3<double>(), 0.01 * M3<double>::identity()) +
      transform_inertia(xf, inertia_from_params(0.5, V3<double>(0.05, 0, 0), 0.005 * M3<double>::identity()));
  CHECK(rel(m.inertias[0], folded) < 1e-14);
  CHECK(m.has_frame("l2"));
  CHECK(m.frame("l2").joint == 0);
  CHECK(rel(m.frame("l2").offset.R, xf.R) < 1e-15);
}

TEST("model", "fusing fixed joints never changes FK of surviving frames") {  // :141-178
  Rng rng(321);
  for (int t = 0; t < 20; ++t) {
    Description d = random_tree(rng, 10, 0.4);
    int fixed = 0;
    for (auto& j : d.joints)
      if (uniform(rng, 0.0, 1.0) < 0.3) {
        j.type = JointType::Fixed;
        ++fixed;
      }
    Description unfused = d;
    for (auto& j : unfused.joints)
      if (j.type == JointType::Fixed) {
        j.type = JointType::Revolute;
        j.axis = V3<double>(0, 0, 1);
      }
    const Model a = build_model(d), b = build_model(unfused);
    CHECK(a.dof() == b.dof() - fixed);
    const Vec q = random_vector(rng, a.dof());
    Vec qb = zeros(b.dof());
    for (int i = 0; i < a.dof(); ++i) qb[(size_t)b.joint_index(a.joints[(size_t)i].name)] = q[(size_t)i];
    const auto fa = forward_kinematics<double>(a, q);
    const auto fb = forward_kinematics<double>(b, qb);
    for (int i = 0; i < a.dof(); ++i) {
      const int o = b.joint_index(a.joints[(size_t)i].name);
      CHECK(rel(fa[(size_t)i].R, fb[(size_t)o].R) < 1e-12);
      CHECK(rel(fa[(size_t)i].p, fb[(size_t)o].p) < 1e-12);
    }
  }
}

TEST("model", "only fixed joints leaves a 0-dof model with working FK") {  // :180-195
  Description d;
  d.add_link("base");
  d.add_link("tool");
  const Xform<double> x{test_rotation(0.5), V3<double>(1, 2, 3)};
  d.add_joint("mount", JointType::Fixed, "base", "tool", x);
  const Model m = build_model(d);
  CHECK(m.dof() == 0);
  const auto w = forward_kinematics<double>(m, Vec());
  const Xform<double> tool = frame_transform<double>(m, w, "tool");
  CHECK(rel(tool.R, x.R) < 1e-15);
  CHECK(rel(tool.p, x.p) < 1e-15);
  CHECK(w.empty());
}

TEST("model", "out-of-order joint listing builds the same model") {  // :197-212
  Description d = two_link_chain(), s = d;
  std::swap(s.joints[0], s.joints[1]);
  std::swap(s.links[0], s.links[2]);
  const Model a = build_model(d), b = build_model(s);
  CHECK(a.dof() == b.dof());
  for (int i = 0; i < a.dof(); ++i) {
    CHECK(a.joints[(size_t)i].name == b.joints[(size_t)i].name);
    CHECK(a.joints[(size_t)i].parent == b.joints[(size_t)i].parent);
    CHECK(rel(a.inertias[(size_t)i], b.inertias[(size_t)i]) == 0.0);
  }
  CHECK(a.mask == b.mask);
}

TEST("model", "structural errors") {  // :214-262
  {
    Description d = two_link_chain();
    d.add_link("l1");
    CHECK_THROWS(build_model(d), ModelError);
    Description d2 = two_link_chain();
    d2.add_joint("a", JointType::Fixed, "l2", "base2", Xform<double>());
    CHECK_THROWS(build_model(d2), ModelError);
  }
  {
    Description d = two_link_chain();
    d.add_link("orphan1");
    d.add_link("orphan2");
    d.add_joint("oj", JointType::Revolute, "orphan1", "orphan2", Xform<double>(), {0, 0, 1});
    CHECK_THROWS(build_model(d), ModelError);
  }
  {
    Description d = two_link_chain();
    d.add_joint("back", JointType::Revolute, "l2", "base", Xform<double>(), {0, 0, 1});
    CHECK_THROWS(build_model(d), ModelError);
  }
  {
    Description d = two_link_chain();
    d.joints[0].axis = V3<double>(0, 0, 2.0);
    CHECK_THROWS(build_model(d), ModelError);
  }
  {
    Description d;
    d.add_link("base");
    d.add_link("middle");
    d.add_link("tip", 0.5, V3<double>(), 0.01 * M3<double>::identity());
    d.add_joint("j1", JointType::Revolute, "base", "middle", Xform<double>(), {0, 0, 1});
    d.add_joint("j2", JointType::Revolute, "middle", "tip", Xform<double>(), {0, 1, 0});
    CHECK_THROWS(build_model(d), ModelError);
  }
  {
    Description d;
    d.add_link("base");
    d.add_link("middle", 0.0, V3<double>(), M3<double>());
    d.add_link("tip", 0.5, V3<double>(), 0.01 * M3<double>::identity());
    d.add_joint("j1", JointType::Revolute, "base", "middle", Xform<double>(), {0, 0, 1});
    d.add_joint("j2", JointType::Revolute, "middle", "tip", Xform<double>(), {0, 1, 0});
    CHECK(!build_model(d).warnings.empty());
  }
}

TEST("model", "floating base") {  // :264-301
  const Model fixed = build_model(two_link_chain());
  const Model fl = floating_base(fixed);
  CHECK(fl.dof() == fixed.dof() + 6);
  CHECK(fl.joints[0].type == JointType::Prismatic);
  CHECK(fl.joints[3].type == JointType::Revolute);
  CHECK(rel(fl.joints[3].axis, V3<double>(0, 0, 1)) == 0.0);
  CHECK(rel(fl.joints[5].axis, V3<double>(1, 0, 0)) == 0.0);
  {
    Rng rng(7);
    const Vec q = random_vector(rng, fixed.dof());
    Vec qf = zeros(fl.dof());
    for (int i = 0; i < fixed.dof(); ++i) qf[(size_t)(i + 6)] = q[(size_t)i];
    const auto a = forward_kinematics<double>(fixed, q), b = forward_kinematics<double>(fl, qf);
    for (int i = 0; i < fixed.dof(); ++i) {
      CHECK(rel(a[(size_t)i].R, b[(size_t)(i + 6)].R) < 1e-15);
      CHECK(rel(a[(size_t)i].p, b[(size_t)(i + 6)].p) < 1e-15);
    }
  }
  {
    Rng rng(8);
    const Vec q = random_vector(rng, fl.dof());
    const Vec g = gravity_vector<double>(fl, q);
    CHECK(std::abs(g[0]) < 1e-12);
    CHECK(std::abs(g[1]) < 1e-12);
    CHECK(std::abs(g[2] - fl.total_mass * 9.81) < 1e-12 * std::max(1.0, fl.total_mass * 9.81));
  }
  CHECK(!fl.warnings.empty());
}

TEST("model", "max depth and serial flag") {  // :303-316
  const Model chain = build_model(two_link_chain());
  CHECK(chain.serial);
  CHECK(chain.max_depth == 2);
  Description b = two_link_chain();
  b.add_link("l3", 0.3, V3<double>(), 0.01 * M3<double>::identity());
  b.add_joint("c", JointType::Revolute, "l1", "l3", Xform<double>(), {1, 0, 0});
  const Model tree = build_model(b);
  CHECK(!tree.serial);
  CHECK(tree.max_depth == 2);
  CHECK(tree.dof() == 3);
}

// ---------------------------------------------------------------- test_urdf.cpp
namespace {
const char* kMinimal = R"(<?xml version="1.0"?>
<robot name="mini">
  <link name="base"/>
  <link name="arm">
    <inertial>
      <origin xyz="0.1 0 0" rpy="0 0 0"/>
      <mass value="1.5"/>
      <inertia ixx="0.01" ixy="0" ixz="0" iyy="0.01" iyz="0" izz="0.02"/>
    </inertial>
  </link>
  <joint name="shoulder" type="revolute">
    <parent link="base"/>
    <child link="arm"/>
    <origin xyz="0 0 0.5" rpy="0 0 0"/>
    <axis xyz="0 0 1"/>
    <limit lower="-1.0" upper="1.0" effort="10" velocity="2"/>
  </joint>
</robot>
)";

bool same_doc(const urdf::Document& a, const urdf::Document& b) {  // test_urdf.cpp:47-86
  if (a.robot_name != b.robot_name || a.links.size() != b.links.size() || a.joints.size() != b.joints.size())
    return false;
  for (size_t i = 0; i < a.links.size(); ++i) {
    const auto &x = a.links[i], &y = b.links[i];
    if (x.name != y.name || x.inertial.present != y.inertial.present) return false;
    if (x.inertial.present &&
        (x.inertial.mass != y.inertial.mass || flat(x.inertial.xyz) != flat(y.inertial.xyz) ||
         flat(x.inertial.rpy) != flat(y.inertial.rpy) || flat(x.inertial.inertia) != flat(y.inertial.inertia)))
      return false;
  }
  for (size_t i = 0; i < a.joints.size(); ++i) {
    const auto &x = a.joints[i], &y = b.joints[i];
    if (x.name != y.name || x.type != y.type || x.parent_link != y.parent_link || x.child_link != y.child_link ||
        flat(x.xyz) != flat(y.xyz) || flat(x.rpy) != flat(y.rpy) || x.limits.has_value() != y.limits.has_value())
      return false;
    if (x.type != urdf::JType::Fixed && flat(x.axis) != flat(y.axis)) return false;
    if (x.limits && (x.limits->lower != y.limits->lower || x.limits->upper != y.limits->upper ||
                     x.limits->effort != y.limits->effort || x.limits->velocity != y.limits->velocity))
      return false;
  }
  return true;
}
std::string replaced(std::string s, const std::string& what, const std::string& with) {
  s.replace(s.find(what), what.size(), with);
  return s;
}
}  // namespace

TEST("urdf", "xml reader basics") {  // :90-100
  const xml::Element r =
      xml::parse("<a x=\"1\">\n  <!-- comment -->\n  <b y=\"&lt;&amp;&gt;\"/>\n  text\n  <b y=\"2\"><c/></b>\n</a>");
  CHECK(r.name == "a");
  CHECK(*r.attr("x") == "1");
  CHECK(r.children.size() == 2);
  CHECK(*r.children[0].attr("y") == "<&>");
  CHECK(r.children[1].child("c") != nullptr);
  CHECK(r.children_named("b").size() == 2);
}

TEST("urdf", "xml errors carry line and column") {  // :102-124
  bool caught = false;
  try {
    xml::parse("<a>\n  <b>\n  </c>\n</a>");
  } catch (const ParseError& e) {
    caught = true;
    CHECK(e.line == 3);
    CHECK(e.column == 3);
  }
  CHECK(caught);
  CHECK_THROWS(xml::parse("<a><b></b>"), ParseError);
  CHECK_THROWS(xml::parse("<a x=\"&bogus;\"/>"), ParseError);
  CHECK_THROWS(xml::parse("<!DOCTYPE robot><robot/>"), ParseError);
  CHECK_THROWS(xml::parse("<a x=\"1\" x=\"2\"/>"), ParseError);
}

TEST("urdf", "rpy_to_rotation") {  // :126-146
  CHECK(rel(urdf::rpy_to_rotation(0, 0, 0), M3<double>::identity()) == 0.0);
  CHECK(rel(urdf::rpy_to_rotation(0, 0, M_PI / 2) * V3<double>(1, 0, 0), V3<double>(0, 1, 0)) < 1e-15);
  Rng rng(11);
  for (int t = 0; t < 50; ++t) {
    const double r = uniform(rng, -M_PI, M_PI), p = uniform(rng, -M_PI, M_PI), y = uniform(rng, -M_PI, M_PI);
    const M3<double> want = axis_angle_rotation<double>({0, 0, 1}, y) * axis_angle_rotation<double>({0, 1, 0}, p) *
                            axis_angle_rotation<double>({1, 0, 0}, r);
    CHECK(rel(urdf::rpy_to_rotation(r, p, y), want) < 1e-14);
  }
}

TEST("urdf", "minimal document builds a 1-dof model") {  // :148-157
  const urdf::Document doc = urdf::parse_urdf(kMinimal);
  CHECK(doc.robot_name == "mini");
  CHECK(doc.warnings.empty());
  const Model m = build_model(urdf::to_description(doc));
  CHECK(m.dof() == 1);
  CHECK(m.joints[0].limits.has_value());
  CHECK(m.joints[0].limits->effort == 10.0);
  CHECK(std::abs(m.inertias[0](5, 5) - 1.5) < 1e-12);
}

TEST("urdf", "chain7 asset: 7 moving dofs, serial chain") {  // :159-175
  const urdf::Document doc = urdf::parse_urdf(robots::asset_text("chain7.urdf"));
  int moving = 0;
  for (const auto& j : doc.joints) moving += j.type != urdf::JType::Fixed;
  CHECK(moving == 7);
  const Model m = build_model(urdf::to_description(doc));
  CHECK(m.dof() == 7);
  CHECK(m.serial);
  CHECK(m.has_frame("ee"));
  CHECK(!doc.warnings.empty());
}

TEST("urdf", "humanoid asset: 23 moving dofs, branched") {  // :177-185
  const Model m = robots::humanoid23();
  CHECK(m.dof() == 23);
  CHECK(!m.serial);
  CHECK(m.has_frame("l_palm"));
  CHECK(m.has_frame("head"));
  CHECK(floating_base(m).dof() == 29);
}

TEST("urdf", "parse-serialize roundtrip is idempotent on recognized fields") {  // :187-202
  const urdf::Document a = urdf::parse_urdf(kMinimal);
  CHECK(same_doc(a, urdf::parse_urdf(urdf::serialize_urdf(a))));
  for (const char* f : {"chain7.urdf", "humanoid23.urdf"}) {
    const urdf::Document d = urdf::parse_urdf(robots::asset_text(f));
    CHECK(same_doc(d, urdf::parse_urdf(urdf::serialize_urdf(d))));
  }
}

TEST("urdf", "document errors") {  // :204-271
  const std::string t = kMinimal;
  CHECK_THROWS(urdf::parse_urdf(replaced(t, "revolute", "planar")), UnsupportedFeatureError);
  CHECK_THROWS(urdf::parse_urdf(replaced(t, "revolute", "floating")), UnsupportedFeatureError);
  {
    const Model m = build_model(urdf::to_description(urdf::parse_urdf(replaced(t, "revolute", "continuous"))));
    CHECK(m.dof() == 1);
    CHECK(m.joints[0].type == JointType::Revolute);
  }
  CHECK_THROWS(urdf::parse_urdf(R"(<robot name="c">
          <link name="a"/><link name="b"/>
          <joint name="j1" type="fixed"><parent link="a"/><child link="b"/></joint>
          <joint name="j2" type="fixed"><parent link="b"/><child link="a"/></joint>
        </robot>)"),
               ModelError);
  CHECK_THROWS(urdf::parse_urdf(R"(<robot name="d">
          <link name="a"/>
          <joint name="j" type="fixed"><parent link="a"/><child link="ghost"/></joint>
        </robot>)"),
               ModelError);
  {
    const char* text = R"(<robot name="m">
      <link name="base"/>
      <link name="mid"/>
      <link name="tip">
        <inertial><mass value="1"/>
          <inertia ixx="0.1" ixy="0" ixz="0" iyy="0.1" iyz="0" izz="0.1"/>
        </inertial>
      </link>
      <joint name="j1" type="revolute">
        <parent link="base"/><child link="mid"/><axis xyz="0 1 0"/>
      </joint>
      <joint name="j2" type="revolute">
        <parent link="mid"/><child link="tip"/><axis xyz="0 1 0"/>
      </joint>
    </robot>)";
    bool named = false;
    try {
      build_model(urdf::to_description(urdf::parse_urdf(text)));
    } catch (const ModelError& e) {
      named = std::string(e.what()).find("mid") != std::string::npos;
    }
    CHECK(named);
  }
  {
    urdf::Document d = urdf::parse_urdf(kMinimal);
    d.links[1].inertial.inertia(0, 1) = 0.5;
    CHECK_THROWS(urdf::to_description(d), ModelError);
  }
  CHECK_THROWS(urdf::parse_urdf(replaced(t, "1.5", "abc")), ParseError);
}

TEST("urdf", "unrecognized elements are skipped with warnings") {  // :273-284
  const urdf::Document d = urdf::parse_urdf(R"(<robot name="w">
    <link name="a">
      <visual><geometry><box size="1 1 1"/></geometry></visual>
    </link>
    <transmission name="t"/>
  </robot>)");
  CHECK(d.warnings.size() == 2);
  if (d.warnings.size() == 2) {
    CHECK(d.warnings[0].find("visual") != std::string::npos);
    CHECK(d.warnings[1].find("transmission") != std::string::npos);
  }
}
