// Host model layer: see vd_host.hpp.
#include "vd_host.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <fstream>
#include <functional>
#include <set>
#include <sstream>

// The two robot assets are compiled into the library, as the reference embeds
// them at configure time (proj/core/CMakeLists.txt:3-9, embedded_assets.hpp.in).
#ifndef VD_ASSET_DIR
#error "VD_ASSET_DIR must point at the repository's assets/ directory"
#endif
__asm__(
    ".section .rodata\n"
    ".global vd_asset_chain7\n"
    "vd_asset_chain7:\n"
    ".incbin \"" VD_ASSET_DIR "/chain7.urdf\"\n"
    ".byte 0\n"
    ".global vd_asset_humanoid23\n"
    "vd_asset_humanoid23:\n"
    ".incbin \"" VD_ASSET_DIR "/humanoid23.urdf\"\n"
    ".byte 0\n"
    ".previous\n");
extern "C" const char vd_asset_chain7[];
extern "C" const char vd_asset_humanoid23[];

namespace vdh {

// ================================================================ linear algebra
Mat3 mat3_identity() { return {1, 0, 0, 0, 1, 0, 0, 0, 1}; }
Mat3 mat3_mul(const Mat3& a, const Mat3& b) {
  Mat3 o{};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o[r * 3 + c] = a[r * 3] * b[c] + a[r * 3 + 1] * b[3 + c] + a[r * 3 + 2] * b[6 + c];
  return o;
}
Vec3 mat3_vec(const Mat3& a, const Vec3& v) {
  return {a[0] * v[0] + a[1] * v[1] + a[2] * v[2], a[3] * v[0] + a[4] * v[1] + a[5] * v[2],
          a[6] * v[0] + a[7] * v[1] + a[8] * v[2]};
}
Mat3 mat3_transpose(const Mat3& a) { return {a[0], a[3], a[6], a[1], a[4], a[7], a[2], a[5], a[8]}; }
Pose compose(const Pose& a, const Pose& b) {
  Pose o;
  o.R = mat3_mul(a.R, b.R);
  const Vec3 t = mat3_vec(a.R, b.p);
  o.p = {t[0] + a.p[0], t[1] + a.p[1], t[2] + a.p[2]};
  return o;
}

namespace {

double max_abs9(const Mat3& m) {
  double s = 0;
  for (double x : m) s = std::max(s, std::abs(x));
  return s;
}
Mat3 skew(const Vec3& v) { return {0, -v[2], v[1], v[2], 0, -v[0], -v[1], v[0], 0}; }

// Smallest eigenvalue of a symmetric 3x3 (closed-form trigonometric solution).
double min_eig_sym(const Mat3& a) {
  const double p1 = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
  if (p1 == 0.0) return std::min({a[0], a[4], a[8]});
  const double q = (a[0] + a[4] + a[8]) / 3.0;
  const double p2 = (a[0] - q) * (a[0] - q) + (a[4] - q) * (a[4] - q) + (a[8] - q) * (a[8] - q) + 2.0 * p1;
  const double p = std::sqrt(p2 / 6.0);
  Mat3 b;
  for (int i = 0; i < 9; ++i) b[i] = (a[i] - (i % 4 == 0 ? q : 0.0)) / p;
  const double detb = b[0] * (b[4] * b[8] - b[5] * b[7]) - b[1] * (b[3] * b[8] - b[5] * b[6]) +
                      b[2] * (b[3] * b[7] - b[4] * b[6]);
  const double r = std::clamp(detb / 2.0, -1.0, 1.0);
  const double phi = std::acos(r) / 3.0;
  return q + 2.0 * p * std::cos(phi + 2.0 * M_PI / 3.0);
}

// inertia_from_params, spatial.hpp:277-298.
Mat6 spatial_inertia(double mass, const Vec3& c, const Mat3& Ic) {
  if (mass < 0.0) throw Failure(kModel, "inertia_from_params: negative mass " + std::to_string(mass));
  const double scale = std::max(1.0, max_abs9(Ic));
  Mat3 asym;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) asym[r * 3 + k] = Ic[r * 3 + k] - Ic[k * 3 + r];
  if (max_abs9(asym) > 1e-9 * scale) throw Failure(kModel, "inertia_from_params: rotational inertia is not symmetric");
  if (min_eig_sym(Ic) < -1e-9 * scale)
    throw Failure(kModel, "inertia_from_params: rotational inertia is not positive semidefinite");
  const Mat3 cx = skew(c);
  const Mat3 cct = mat3_mul(cx, mat3_transpose(cx));
  Mat6 m{};
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) {
      m[r * 6 + k] = Ic[r * 3 + k] + mass * cct[r * 3 + k];
      m[r * 6 + k + 3] = mass * cx[r * 3 + k];
      m[(r + 3) * 6 + k] = mass * cx[k * 3 + r];
    }
  m[21] = m[28] = m[35] = mass;
  return m;
}

// transform_inertia, spatial.hpp:259-267: Y I Yᵀ with Y = [[R, p×R], [0, R]].
Mat6 shift_inertia(const Pose& x, const Mat6& I) {
  Mat6 y{};
  const Mat3 pr = mat3_mul(skew(x.p), x.R);
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) {
      y[r * 6 + k] = x.R[r * 3 + k];
      y[(r + 3) * 6 + k + 3] = x.R[r * 3 + k];
      y[r * 6 + k + 3] = pr[r * 3 + k];
    }
  Mat6 t{}, o{};
  for (int r = 0; r < 6; ++r)
    for (int k = 0; k < 6; ++k) {
      double s = 0;
      for (int l = 0; l < 6; ++l) s += y[r * 6 + l] * I[l * 6 + k];
      t[r * 6 + k] = s;
    }
  for (int r = 0; r < 6; ++r)
    for (int k = 0; k < 6; ++k) {
      double s = 0;
      for (int l = 0; l < 6; ++l) s += t[r * 6 + l] * y[k * 6 + l];
      o[r * 6 + k] = s;
    }
  return o;
}

bool is_rotation(const Mat3& r) {  // spatial.hpp:270-273
  const Mat3 rtr = mat3_mul(mat3_transpose(r), r);
  double e = 0;
  for (int i = 0; i < 9; ++i) e = std::max(e, std::abs(rtr[i] - (i % 4 == 0 ? 1.0 : 0.0)));
  const double det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[1] * (r[3] * r[8] - r[5] * r[6]) +
                     r[2] * (r[3] * r[7] - r[4] * r[6]);
  return e <= 1e-9 && std::abs(det - 1.0) <= 1e-9;
}

// ================================================================ XML (xml.cpp semantics)
struct XNode {
  std::string tag;
  std::vector<std::pair<std::string, std::string>> attrs;
  std::vector<XNode> kids;
  int line = 0, col = 0;
  const std::string* get(const char* k) const {
    for (const auto& a : attrs)
      if (a.first == k) return &a.second;
    return nullptr;
  }
  const XNode* first(const char* t) const {
    for (const XNode& c : kids)
      if (c.tag == t) return &c;
    return nullptr;
  }
};

class XmlScanner {
 public:
  explicit XmlScanner(std::string_view t) : t_(t) {}

  XNode document() {
    prolog(true);
    if (end()) die("document has no root element");
    XNode root = node();
    prolog(false);
    if (!end()) die("content after the root element");
    return root;
  }

 private:
  std::string_view t_;
  size_t k_ = 0;
  int ln_ = 1, cl_ = 1;

  bool end() const { return k_ >= t_.size(); }
  bool sees(std::string_view s) const { return t_.compare(k_, s.size(), s) == 0; }
  char take() {
    const char c = t_[k_++];
    if (c == '\n') {
      ++ln_;
      cl_ = 1;
    } else {
      ++cl_;
    }
    return c;
  }
  void skip(size_t m) {
    for (size_t i = 0; i < m && !end(); ++i) take();
  }
  [[noreturn]] void die(const std::string& m) const { throw Failure(kParse, m, ln_, cl_); }
  void blanks() {
    while (!end() && std::isspace((unsigned char)t_[k_])) take();
  }
  static bool head(char c) { return std::isalpha((unsigned char)c) || c == '_' || c == ':'; }
  static bool body(char c) { return head(c) || std::isdigit((unsigned char)c) || c == '-' || c == '.'; }
  std::string ident() {
    if (end() || !head(t_[k_])) die("expected a name");
    std::string s;
    while (!end() && body(t_[k_])) s += take();
    return s;
  }
  void must(char c) {
    if (end() || t_[k_] != c) die(std::string("expected '") + c + "'");
    take();
  }
  void until(std::string_view stop, const char* what) {
    const int l = ln_, c = cl_;
    while (!end()) {
      if (sees(stop)) {
        skip(stop.size());
        return;
      }
      take();
    }
    throw Failure(kParse, std::string("unterminated ") + what, l, c);
  }
  std::string reference() {
    const int l = ln_, c = cl_;
    take();
    std::string e;
    while (!end() && t_[k_] != ';') {
      e += take();
      if (e.size() > 10) throw Failure(kParse, "malformed entity reference", l, c);
    }
    if (end()) throw Failure(kParse, "unterminated entity reference", l, c);
    take();
    if (e == "amp") return "&";
    if (e == "lt") return "<";
    if (e == "gt") return ">";
    if (e == "quot") return "\"";
    if (e == "apos") return "'";
    if (!e.empty() && e[0] == '#') {
      const bool hex = e.size() > 1 && (e[1] == 'x' || e[1] == 'X');
      unsigned long cp;
      try {
        cp = std::stoul(e.substr(hex ? 2 : 1), nullptr, hex ? 16 : 10);
      } catch (const std::invalid_argument&) {
        throw Failure(kParse, "malformed character reference", l, c);
      } catch (const std::out_of_range&) {
        throw Failure(kParse, "character reference out of range", l, c);
      }
      if (cp == 0 || cp > 0x10FFFF) throw Failure(kParse, "character reference out of range", l, c);
      std::string u;
      if (cp < 0x80) {
        u += char(cp);
      } else if (cp < 0x800) {
        u += char(0xC0 | (cp >> 6));
        u += char(0x80 | (cp & 0x3F));
      } else if (cp < 0x10000) {
        u += char(0xE0 | (cp >> 12));
        u += char(0x80 | ((cp >> 6) & 0x3F));
        u += char(0x80 | (cp & 0x3F));
      } else {
        u += char(0xF0 | (cp >> 18));
        u += char(0x80 | ((cp >> 12) & 0x3F));
        u += char(0x80 | ((cp >> 6) & 0x3F));
        u += char(0x80 | (cp & 0x3F));
      }
      return u;
    }
    throw Failure(kParse, "unknown entity '&" + e + ";'", l, c);
  }
  std::string value() {
    if (end() || (t_[k_] != '"' && t_[k_] != '\'')) die("expected a quoted attribute value");
    const char q = take();
    std::string v;
    for (;;) {
      if (end()) die("unterminated attribute value");
      const char c = t_[k_];
      if (c == q) {
        take();
        return v;
      }
      if (c == '<') die("'<' is not allowed in attribute values");
      v += (c == '&') ? reference() : std::string(1, take());
    }
  }
  void prolog(bool first) {
    for (;;) {
      blanks();
      if (sees("<!--")) {
        skip(4);
        until("-->", "comment");
      } else if (sees("<?")) {
        skip(2);
        until("?>", "processing instruction");
      } else if (first && sees("<!DOCTYPE")) {
        die("DOCTYPE declarations are not supported");
      } else {
        return;
      }
    }
  }
  XNode node() {
    XNode x;
    x.line = ln_;
    x.col = cl_;
    must('<');
    x.tag = ident();
    for (;;) {
      blanks();
      if (end()) die("unterminated start tag <" + x.tag + ">");
      if (t_[k_] == '>') {
        take();
        inner(x);
        return x;
      }
      if (sees("/>")) {
        skip(2);
        return x;
      }
      std::string k = ident();
      blanks();
      must('=');
      blanks();
      std::string v = value();
      for (const auto& a : x.attrs)
        if (a.first == k) die("duplicate attribute '" + k + "'");
      x.attrs.emplace_back(std::move(k), std::move(v));
    }
  }
  void inner(XNode& x) {
    for (;;) {
      if (end()) die("missing end tag </" + x.tag + ">");
      if (sees("</")) {
        const int l = ln_, c = cl_;
        skip(2);
        const std::string closing = ident();
        if (closing != x.tag)
          throw Failure(kParse, "mismatched end tag </" + closing + ">; expected </" + x.tag + ">", l, c);
        blanks();
        must('>');
        return;
      }
      if (sees("<!--")) {
        skip(4);
        until("-->", "comment");
      } else if (sees("<![CDATA[")) {
        skip(9);
        until("]]>", "CDATA section");
      } else if (sees("<?")) {
        skip(2);
        until("?>", "processing instruction");
      } else if (t_[k_] == '<') {
        x.kids.push_back(node());
      } else if (t_[k_] == '&') {
        reference();
      } else {
        take();
      }
    }
  }
};

// ================================================================ URDF (urdf.cpp semantics)
[[noreturn]] void urdf_fail(const XNode& e, const std::string& m) { throw Failure(kParse, m, e.line, e.col); }

double to_number(const XNode& e, const std::string& s, const char* what) {
  size_t used = 0;
  double v = 0;
  try {
    v = std::stod(s, &used);
  } catch (const std::exception&) {
    urdf_fail(e, std::string("invalid number '") + s + "' in " + what);
  }
  while (used < s.size() && std::isspace((unsigned char)s[used])) ++used;
  if (used != s.size()) urdf_fail(e, std::string("invalid number '") + s + "' in " + what);
  return v;
}
Vec3 to_vec3(const XNode& e, const std::string& s, const char* what) {
  std::istringstream in(s);
  Vec3 v{};
  std::string tok;
  for (int i = 0; i < 3; ++i) {
    if (!(in >> tok)) urdf_fail(e, std::string("expected 3 numbers in ") + what + ", got '" + s + "'");
    v[i] = to_number(e, tok, what);
  }
  if (in >> tok) urdf_fail(e, std::string("expected 3 numbers in ") + what + ", got '" + s + "'");
  return v;
}
double attr_number(const XNode& e, const char* a) {
  const std::string* v = e.get(a);
  if (!v) urdf_fail(e, "<" + e.tag + "> is missing the '" + a + "' attribute");
  return to_number(e, *v, a);
}
Mat3 rpy_matrix(const Vec3& rpy) {  // urdf.cpp:14-31
  const double cr = std::cos(rpy[0]), sr = std::sin(rpy[0]);
  const double cp = std::cos(rpy[1]), sp = std::sin(rpy[1]);
  const double cy = std::cos(rpy[2]), sy = std::sin(rpy[2]);
  const Mat3 rx{1, 0, 0, 0, cr, -sr, 0, sr, cr};
  const Mat3 ry{cp, 0, sp, 0, 1, 0, -sp, 0, cp};
  const Mat3 rz{cy, -sy, 0, sy, cy, 0, 0, 0, 1};
  return mat3_mul(mat3_mul(rz, ry), rx);
}
void read_origin(const XNode& e, Vec3* xyz, Vec3* rpy) {
  const XNode* o = e.first("origin");
  if (!o) return;
  if (const std::string* v = o->get("xyz")) *xyz = to_vec3(*o, *v, "origin xyz");
  if (const std::string* v = o->get("rpy")) *rpy = to_vec3(*o, *v, "origin rpy");
}

}  // namespace

int Model::frame_index(std::string_view name) const {
  auto it = frame_of.find(std::string(name));
  if (it == frame_of.end()) throw Failure(kUnknownFrame, "unknown frame '" + std::string(name) + "'");
  return it->second;
}

Description parse_urdf_text(std::string_view text) {
  const XNode root = XmlScanner(text).document();
  if (root.tag != "robot")
    throw Failure(kParse, "root element must be <robot>, found <" + root.tag + ">", root.line, root.col);
  Description d;
  if (const std::string* n = root.get("name")) d.name = *n;
  std::set<std::string> link_names, joint_names, child_names;
  for (const XNode& c : root.kids) {
    if (c.tag == "link") {  // urdf.cpp:95-132
      const std::string* nm = c.get("name");
      if (!nm) urdf_fail(c, "<link> is missing the 'name' attribute");
      LinkDesc l;
      l.name = *nm;
      for (const XNode& sub : c.kids) {
        if (sub.tag != "inertial") continue;
        Vec3 xyz{0, 0, 0}, rpy{0, 0, 0};
        read_origin(sub, &xyz, &rpy);
        const XNode* ms = sub.first("mass");
        if (!ms) urdf_fail(sub, "link '" + l.name + "' inertial is missing <mass>");
        const double mass = attr_number(*ms, "value");
        const XNode* in = sub.first("inertia");
        if (!in) urdf_fail(sub, "link '" + l.name + "' inertial is missing <inertia>");
        const double ixx = attr_number(*in, "ixx"), ixy = attr_number(*in, "ixy"), ixz = attr_number(*in, "ixz");
        const double iyy = attr_number(*in, "iyy"), iyz = attr_number(*in, "iyz"), izz = attr_number(*in, "izz");
        const Mat3 I{ixx, ixy, ixz, ixy, iyy, iyz, ixz, iyz, izz};
        // to_description (urdf.cpp:342-357): symmetrize, rotate by the inertial rpy.
        Mat3 sym;
        for (int r = 0; r < 3; ++r)
          for (int k = 0; k < 3; ++k) sym[r * 3 + k] = 0.5 * (I[r * 3 + k] + I[k * 3 + r]);
        const Mat3 rr = rpy_matrix(rpy);
        l.has_inertial = true;
        l.mass = mass;
        l.com = xyz;
        l.inertia = mat3_mul(mat3_mul(rr, sym), mat3_transpose(rr));
      }
      d.links.push_back(l);
    } else if (c.tag == "joint") {  // urdf.cpp:134-200
      const std::string* nm = c.get("name");
      if (!nm) urdf_fail(c, "<joint> is missing the 'name' attribute");
      JointDesc j;
      j.name = *nm;
      j.axis = {1, 0, 0};  // URDF default (urdf.hpp:30)
      const std::string* ty = c.get("type");
      if (!ty) urdf_fail(c, "joint '" + j.name + "' is missing the 'type' attribute");
      if (*ty == "revolute" || *ty == "continuous") j.kind = Kind::Revolute;
      else if (*ty == "prismatic") j.kind = Kind::Prismatic;
      else if (*ty == "fixed") j.kind = Kind::Fixed;
      else if (*ty == "planar" || *ty == "floating")
        throw Failure(kUnsupportedFeature, "joint '" + j.name + "' has unsupported type '" + *ty + "'");
      else urdf_fail(c, "joint '" + j.name + "' has unknown type '" + *ty + "'");
      const XNode* pa = c.first("parent");
      const XNode* ch = c.first("child");
      if (!pa || !pa->get("link")) urdf_fail(c, "joint '" + j.name + "' is missing <parent link=...>");
      if (!ch || !ch->get("link")) urdf_fail(c, "joint '" + j.name + "' is missing <child link=...>");
      j.parent = *pa->get("link");
      j.child = *ch->get("link");
      Vec3 xyz{0, 0, 0}, rpy{0, 0, 0};
      read_origin(c, &xyz, &rpy);
      j.origin.R = rpy_matrix(rpy);
      j.origin.p = xyz;
      if (const XNode* ax = c.first("axis"))
        if (const std::string* v = ax->get("xyz")) j.axis = to_vec3(*ax, *v, "axis xyz");
      if (const XNode* lim = c.first("limit")) {
        j.has_limits = true;
        const char* keys[4] = {"lower", "upper", "effort", "velocity"};
        const char* what[4] = {"limit lower", "limit upper", "limit effort", "limit velocity"};
        for (int k = 0; k < 4; ++k)
          if (const std::string* v = lim->get(keys[k])) j.limits[k] = to_number(*lim, *v, what[k]);
      }
      d.joints.push_back(j);
    }
  }
  // validate_structure, urdf.cpp:202-239
  for (const LinkDesc& l : d.links)
    if (!link_names.insert(l.name).second) throw Failure(kModel, "duplicate link name '" + l.name + "'");
  for (const JointDesc& j : d.joints) {
    if (!joint_names.insert(j.name).second) throw Failure(kModel, "duplicate joint name '" + j.name + "'");
    if (!link_names.count(j.parent))
      throw Failure(kModel, "joint '" + j.name + "' references unknown parent link '" + j.parent + "'");
    if (!link_names.count(j.child))
      throw Failure(kModel, "joint '" + j.name + "' references unknown child link '" + j.child + "'");
    if (!child_names.insert(j.child).second)
      throw Failure(kModel, "link '" + j.child + "' is the child of more than one joint");
  }
  int roots = 0;
  for (const LinkDesc& l : d.links) roots += child_names.count(l.name) ? 0 : 1;
  if (roots != 1)
    throw Failure(kModel, "document must have exactly one root link, found " + std::to_string(roots) +
                              (roots == 0 ? " (joint graph contains a cycle)" : ""));
  // to_description's asymmetry check (urdf.cpp:343-349) cannot fire on parsed
  // text: the tensor is assembled symmetric from its six attributes.
  return d;
}

// ================================================================ builder (model.cpp)
Model build(const Description& d) {
  std::map<std::string, int> link_of;
  for (size_t i = 0; i < d.links.size(); ++i)
    if (!link_of.emplace(d.links[i].name, (int)i).second)
      throw Failure(kModel, "duplicate link name '" + d.links[i].name + "'");
  std::vector<std::vector<int>> below(d.links.size());
  std::vector<int> in_joint(d.links.size(), -1);
  std::set<std::string> seen;
  for (size_t j = 0; j < d.joints.size(); ++j) {
    const JointDesc& s = d.joints[j];
    if (!seen.insert(s.name).second) throw Failure(kModel, "duplicate joint name '" + s.name + "'");
    auto pi = link_of.find(s.parent), ci = link_of.find(s.child);
    if (pi == link_of.end())
      throw Failure(kModel, "joint '" + s.name + "' references unknown parent link '" + s.parent + "'");
    if (ci == link_of.end())
      throw Failure(kModel, "joint '" + s.name + "' references unknown child link '" + s.child + "'");
    if (in_joint[(size_t)ci->second] >= 0)
      throw Failure(kModel, "link '" + s.child + "' is the child of more than one joint");
    in_joint[(size_t)ci->second] = (int)j;
    below[(size_t)pi->second].push_back((int)j);
  }
  for (auto& v : below)  // canonical order: joint name (model.cpp:115-120)
    std::sort(v.begin(), v.end(), [&](int a, int b) { return d.joints[(size_t)a].name < d.joints[(size_t)b].name; });
  int root = -1;
  for (size_t i = 0; i < d.links.size(); ++i) {
    if (in_joint[i] >= 0) continue;
    if (root >= 0)
      throw Failure(kModel, "model has multiple root links ('" + d.links[(size_t)root].name + "' and '" +
                                d.links[i].name + "')");
    root = (int)i;
  }
  if (root < 0) throw Failure(kModel, "model has no root link (joint graph contains a cycle)");
  for (size_t i = 0; i < d.links.size(); ++i) {
    if (d.links[i].has_inertial || (int)i == root) continue;
    const int pj = in_joint[i];
    const bool moved = pj >= 0 && d.joints[(size_t)pj].kind != Kind::Fixed;
    const bool carries =
        std::any_of(below[i].begin(), below[i].end(), [&](int j) { return d.joints[(size_t)j].kind != Kind::Fixed; });
    if (moved && carries)
      throw Failure(kModel, "link '" + d.links[i].name + "' has no inertial but carries a moving child joint");
  }

  Model m;
  std::vector<char> reached(d.links.size(), 0);
  std::function<void(int, int, const Pose&)> visit = [&](int link, int mover, const Pose& rel) {
    reached[(size_t)link] = 1;
    const LinkDesc& L = d.links[(size_t)link];
    if (m.frame_of.count(L.name)) throw Failure(kModel, "duplicate frame name '" + L.name + "'");
    m.frame_of[L.name] = (int)m.frames.size();
    m.frames.push_back({L.name, mover, rel});
    if (mover >= 0) {
      const Mat6 li = L.has_inertial ? spatial_inertia(L.mass, L.com, L.inertia) : Mat6{};
      const Mat6 moved = shift_inertia(rel, li);
      for (int k = 0; k < 36; ++k) m.bodies[(size_t)mover].inertia[k] += moved[k];
      m.total_mass += L.mass;
    }
    for (int j : below[(size_t)link]) {
      const JointDesc& s = d.joints[(size_t)j];
      if (!is_rotation(s.origin.R)) throw Failure(kModel, "joint '" + s.name + "' origin rotation is not orthonormal");
      const int child = link_of.at(s.child);
      if (s.kind == Kind::Fixed) {
        visit(child, mover, compose(rel, s.origin));
        continue;
      }
      const double nrm = std::sqrt(s.axis[0] * s.axis[0] + s.axis[1] * s.axis[1] + s.axis[2] * s.axis[2]);
      if (std::abs(nrm - 1.0) > 1e-9)
        throw Failure(kModel, "joint '" + s.name + "' axis has norm " + std::to_string(nrm) + "; expected a unit vector");
      Body b;
      b.name = s.name;
      b.kind = s.kind;
      b.parent = mover;
      b.offset = compose(rel, s.origin);
      b.axis = {s.axis[0] / nrm, s.axis[1] / nrm, s.axis[2] / nrm};
      b.depth = mover >= 0 ? m.bodies[(size_t)mover].depth + 1 : 1;
      m.bodies.push_back(b);
      visit(child, (int)m.bodies.size() - 1, Pose{});
    }
  };
  visit(root, -1, Pose{});
  for (size_t i = 0; i < d.links.size(); ++i)
    if (!reached[i])
      throw Failure(kModel, "link '" + d.links[i].name + "' is not connected to the root link '" +
                                d.links[(size_t)root].name + "'");
  m.name = d.name;
  m.source = d;
  m.serial = true;
  for (int i = 0; i < m.dof(); ++i) {
    m.max_depth = std::max(m.max_depth, m.bodies[(size_t)i].depth);
    if (m.bodies[(size_t)i].parent != i - 1) m.serial = false;
  }
  for (int i = 0; i < m.dof(); ++i) {
    bool kids = false;
    for (const Body& b : m.bodies) kids |= b.parent == i;
    if (kids && m.bodies[(size_t)i].inertia[35] <= 0.0)
      m.warnings.push_back("joint '" + m.bodies[(size_t)i].name + "' drives a zero-mass link but has moving children");
  }
  if (m.dof() > kMaxDof)
    throw Failure(kUnsupportedStructure, "model has " + std::to_string(m.dof()) + " dof; the device path supports at most " +
                                             std::to_string(kMaxDof));
  return m;
}

Model with_floating_base(const Model& model) {
  const Description& o = model.source;
  std::set<std::string> kids;
  for (const JointDesc& j : o.joints) kids.insert(j.child);
  std::string root;
  for (const LinkDesc& l : o.links)
    if (!kids.count(l.name)) {
      root = l.name;
      break;
    }
  Description d;
  d.name = o.name.empty() ? "floating" : o.name + "_floating";
  d.links.push_back(LinkDesc{"__world"});
  for (const char* s : {"__fb_x", "__fb_y", "__fb_z", "__fb_rz", "__fb_ry"}) {
    LinkDesc l;
    l.name = s;
    l.has_inertial = true;  // explicit zero inertials: massless by design
    d.links.push_back(l);
  }
  struct Stage {
    const char *name, *parent, *child;
    Kind kind;
    Vec3 axis;
  };
  const Stage stages[6] = {{"base_tx", "__world", "__fb_x", Kind::Prismatic, {1, 0, 0}},
                           {"base_ty", "__fb_x", "__fb_y", Kind::Prismatic, {0, 1, 0}},
                           {"base_tz", "__fb_y", "__fb_z", Kind::Prismatic, {0, 0, 1}},
                           {"base_rz", "__fb_z", "__fb_rz", Kind::Revolute, {0, 0, 1}},
                           {"base_ry", "__fb_rz", "__fb_ry", Kind::Revolute, {0, 1, 0}},
                           {"base_rx", "__fb_ry", root.c_str(), Kind::Revolute, {1, 0, 0}}};
  for (const Stage& s : stages) {
    JointDesc j;
    j.name = s.name;
    j.kind = s.kind;
    j.parent = s.parent;
    j.child = s.child;
    j.axis = s.axis;
    d.joints.push_back(j);
  }
  for (const LinkDesc& l : o.links) d.links.push_back(l);
  for (const JointDesc& j : o.joints) d.joints.push_back(j);
  return build(d);
}

Model load_urdf_text(std::string_view text) { return build(parse_urdf_text(text)); }

Model load_urdf_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Failure(kIo, "cannot open URDF file '" + path + "'");
  std::ostringstream ss;
  ss << f.rdbuf();
  return load_urdf_text(ss.str());
}

Model builtin(std::string_view name) {
  if (name == "chain7") return load_urdf_text(vd_asset_chain7);
  if (name == "humanoid23") return load_urdf_text(vd_asset_humanoid23);
  if (name == "tree29") return with_floating_base(load_urdf_text(vd_asset_humanoid23));
  throw Failure(kGeneric, "unknown builtin robot '" + std::string(name) + "'; available: chain7, humanoid23, tree29");
}

// ================================================================ packer
PackedModel pack(const Model& m) {
  PackedModel pm;
  std::memset(static_cast<void*>(&pm), 0, sizeof pm);
  pm.n = m.dof();
  if ((int)m.frames.size() > kMaxFrames) throw Failure(kUnsupportedStructure, "too many frames for the device model");
  pm.nframes = (int)m.frames.size();
  for (int i = 0; i < pm.n; ++i) {
    const Body& b = m.bodies[(size_t)i];
    pm.parent[i] = b.parent;
    pm.kind[i] = b.kind == Kind::Revolute ? 0 : 1;
    int code = 6;
    for (int a = 0; a < 3; ++a) {
      const bool unit = b.axis[a] == 1.0 || b.axis[a] == -1.0;
      bool others_zero = true;
      for (int o = 0; o < 3; ++o)
        if (o != a && b.axis[o] != 0.0) others_zero = false;
      if (unit && others_zero) code = b.axis[a] > 0 ? a : a + 3;
    }
    pm.axis_code[i] = code;
    for (int k = 0; k < 3; ++k) {
      pm.axis[i][k] = b.axis[k];
      pm.p[i][k] = b.offset.p[k];
    }
    for (int k = 0; k < 9; ++k) pm.R[i][k] = b.offset.R[k];
    // 10-parameter inertia; check the rigid-body structure of the folded 6x6.
    const Mat6& I = b.inertia;
    const double mass = I[21];
    const double h[3] = {I[2 * 6 + 4], I[0 * 6 + 5], I[1 * 6 + 3]};  // skew(h) in the top-right block
    double scale = 1.0, resid = 0.0;
    for (double x : I) scale = std::max(scale, std::abs(x));
    double rebuilt[36] = {0};
    const double Io[6] = {I[0], I[7], I[14], 0.5 * (I[1] + I[6]), 0.5 * (I[2] + I[12]), 0.5 * (I[8] + I[13])};
    const Mat3 hx = skew({h[0], h[1], h[2]});
    const int sym[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        rebuilt[r * 6 + c] = Io[sym[r][c]];
        rebuilt[r * 6 + c + 3] = hx[r * 3 + c];
        rebuilt[(r + 3) * 6 + c] = hx[c * 3 + r];
        rebuilt[(r + 3) * 6 + c + 3] = r == c ? mass : 0.0;
      }
    for (int k = 0; k < 36; ++k) resid = std::max(resid, std::abs(rebuilt[k] - I[k]));
    if (resid > 1e-12 * scale)
      throw Failure(kModel, "joint '" + b.name + "' inertia is not a rigid-body spatial inertia (residual " +
                                std::to_string(resid) + ")");
    pm.inertia[i][0] = mass;
    for (int k = 0; k < 3; ++k) pm.inertia[i][1 + k] = h[k];
    for (int k = 0; k < 6; ++k) pm.inertia[i][4 + k] = Io[k];
  }
  for (int f = 0; f < pm.nframes; ++f) {
    pm.frame_joint[f] = m.frames[(size_t)f].joint;
    for (int k = 0; k < 9; ++k) pm.frame_R[f][k] = m.frames[(size_t)f].offset.R[k];
    for (int k = 0; k < 3; ++k) pm.frame_p[f][k] = m.frames[(size_t)f].offset.p[k];
  }
  return pm;
}

uint64_t fingerprint(const PackedModel& pm) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* data, size_t len) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < len; ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  };
  mix(&pm.n, sizeof pm.n);
  for (int i = 0; i < pm.n; ++i) {
    mix(&pm.parent[i], sizeof(int));
    mix(&pm.kind[i], sizeof(int));
    mix(pm.axis[i], sizeof pm.axis[i]);
    mix(pm.R[i], sizeof pm.R[i]);
    mix(pm.p[i], sizeof pm.p[i]);
    mix(pm.inertia[i], sizeof pm.inertia[i]);
  }
  return h;
}

}  // namespace vdh
