// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_spatial.hpp header).
#include "orc_model.hpp"

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <set>
#include <sstream>

namespace orc {

// =====================================================================
// XML reader — behaviour of proj/core/src/xml.cpp:35-316: elements,
// attributes, comments, PIs, CDATA, 5 entities + numeric refs, DOCTYPE
// rejected, 1-based line/column in every ParseError.
// =====================================================================
namespace xml {

const std::string* Element::attr(std::string_view n) const {
  for (const Attr& a : attrs)
    if (a.name == n) return &a.value;
  return nullptr;
}
const Element* Element::child(std::string_view tag) const {
  for (const Element& c : children)
    if (c.name == tag) return &c;
  return nullptr;
}
std::vector<const Element*> Element::children_named(std::string_view tag) const {
  std::vector<const Element*> out;
  for (const Element& c : children)
    if (c.name == tag) out.push_back(&c);
  return out;
}

namespace {

struct Reader {
  std::string_view s;
  size_t i = 0;
  int line = 1, col = 1;

  bool done() const { return i >= s.size(); }
  char cur() const { return s[i]; }
  bool at(std::string_view t) const { return s.compare(i, t.size(), t) == 0; }
  char step() {
    char c = s[i++];
    if (c == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    return c;
  }
  void step(size_t k) {
    while (k-- > 0 && !done()) step();
  }
  void ws() {
    while (!done() && std::isspace((unsigned char)cur())) step();
  }
  [[noreturn]] void fail(const std::string& m) const { throw ParseError(m, line, col); }

  static bool name_start(char c) { return std::isalpha((unsigned char)c) || c == '_' || c == ':'; }
  static bool name_char(char c) {
    return name_start(c) || std::isdigit((unsigned char)c) || c == '-' || c == '.';
  }
  std::string name() {
    if (done() || !name_start(cur())) fail("expected a name");
    std::string n;
    while (!done() && name_char(cur())) n.push_back(step());
    return n;
  }
  void want(char c) {
    if (done() || cur() != c) fail(std::string("expected '") + c + "'");
    step();
  }
  void skip_past(std::string_view term, const char* what) {
    const int l0 = line, c0 = col;
    for (; !done(); step())
      if (at(term)) {
        step(term.size());
        return;
      }
    throw ParseError(std::string("unterminated ") + what, l0, c0);
  }

  static void utf8(std::string& out, unsigned long cp) {
    if (cp < 0x80) {
      out += char(cp);
    } else if (cp < 0x800) {
      out += char(0xC0 | (cp >> 6));
      out += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += char(0xE0 | (cp >> 12));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    } else {
      out += char(0xF0 | (cp >> 18));
      out += char(0x80 | ((cp >> 12) & 0x3F));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    }
  }

  // xml.cpp:129-181
  std::string entity() {
    const int l0 = line, c0 = col;
    step();  // '&'
    std::string e;
    while (!done() && cur() != ';') {
      e.push_back(step());
      if (e.size() > 10) throw ParseError("malformed entity reference", l0, c0);
    }
    if (done()) throw ParseError("unterminated entity reference", l0, c0);
    step();  // ';'
    static const std::map<std::string, std::string> named = {
        {"amp", "&"}, {"lt", "<"}, {"gt", ">"}, {"quot", "\""}, {"apos", "'"}};
    auto it = named.find(e);
    if (it != named.end()) return it->second;
    if (!e.empty() && e[0] == '#') {
      const bool hex = e.size() > 1 && (e[1] == 'x' || e[1] == 'X');
      const std::string digits = e.substr(hex ? 2 : 1);
      unsigned long cp = 0;
      try {
        cp = std::stoul(digits, nullptr, hex ? 16 : 10);
      } catch (const std::invalid_argument&) {
        throw ParseError("malformed character reference", l0, c0);
      } catch (const std::out_of_range&) {
        throw ParseError("character reference out of range", l0, c0);
      }
      if (cp == 0 || cp > 0x10FFFF) throw ParseError("character reference out of range", l0, c0);
      std::string out;
      utf8(out, cp);
      return out;
    }
    throw ParseError("unknown entity '&" + e + ";'", l0, c0);
  }

  std::string quoted() {
    if (done() || (cur() != '"' && cur() != '\'')) fail("expected a quoted attribute value");
    const char q = step();
    std::string v;
    for (;;) {
      if (done()) fail("unterminated attribute value");
      const char c = cur();
      if (c == q) {
        step();
        return v;
      }
      if (c == '<') fail("'<' is not allowed in attribute values");
      if (c == '&')
        v += entity();
      else
        v.push_back(step());
    }
  }

  void misc(bool prolog) {
    for (;;) {
      ws();
      if (at("<!--")) {
        step(4);
        skip_past("-->", "comment");
      } else if (at("<?")) {
        step(2);
        skip_past("?>", "processing instruction");
      } else if (prolog && at("<!DOCTYPE")) {
        fail("DOCTYPE declarations are not supported");
      } else {
        return;
      }
    }
  }

  Element element() {
    Element el;
    el.line = line;
    el.column = col;
    want('<');
    el.name = name();
    for (;;) {
      ws();
      if (done()) fail("unterminated start tag <" + el.name + ">");
      if (cur() == '>') {
        step();
        content(el);
        return el;
      }
      if (at("/>")) {
        step(2);
        return el;
      }
      Attr a;
      a.name = name();
      ws();
      want('=');
      ws();
      a.value = quoted();
      for (const Attr& b : el.attrs)
        if (b.name == a.name) fail("duplicate attribute '" + a.name + "'");
      el.attrs.push_back(std::move(a));
    }
  }

  void content(Element& el) {
    for (;;) {
      if (done()) fail("missing end tag </" + el.name + ">");
      if (at("</")) {
        const int l0 = line, c0 = col;
        step(2);
        const std::string close = name();
        if (close != el.name)
          throw ParseError("mismatched end tag </" + close + ">; expected </" + el.name + ">", l0, c0);
        ws();
        want('>');
        return;
      }
      if (at("<!--")) {
        step(4);
        skip_past("-->", "comment");
      } else if (at("<![CDATA[")) {
        step(9);
        skip_past("]]>", "CDATA section");
      } else if (at("<?")) {
        step(2);
        skip_past("?>", "processing instruction");
      } else if (cur() == '<') {
        el.children.push_back(element());
      } else if (cur() == '&') {
        (void)entity();
      } else {
        step();
      }
    }
  }
};

}  // namespace

Element parse(std::string_view text) {
  Reader r{text};
  r.misc(true);
  if (r.done()) r.fail("document has no root element");
  Element root = r.element();
  r.misc(false);
  if (!r.done()) r.fail("content after the root element");
  return root;
}

}  // namespace xml

// =====================================================================
// Model builder — proj/core/src/model.cpp
// =====================================================================
LinkSpec& Description::add_link(const std::string& n) {
  links.push_back(LinkSpec{});
  links.back().name = n;
  return links.back();
}
LinkSpec& Description::add_link(const std::string& n, double mass, const V3<double>& com,
                                const M3<double>& Ic) {
  LinkSpec& l = add_link(n);
  l.has_inertial = true;
  l.mass = mass;
  l.com = com;
  l.inertia = Ic;
  return l;
}
JointSpec& Description::add_joint(const std::string& n, JointType t, const std::string& parent,
                                  const std::string& child, const Xform<double>& origin,
                                  const V3<double>& axis) {
  JointSpec j;
  j.name = n;
  j.type = t;
  j.parent_link = parent;
  j.child_link = child;
  j.origin = origin;
  j.axis = axis;
  joints.push_back(j);
  return joints.back();
}

const Frame& Model::frame(std::string_view n) const {
  auto it = frame_index.find(std::string(n));
  if (it == frame_index.end()) throw UnknownFrameError("unknown frame '" + std::string(n) + "'");
  return frames[(size_t)it->second];
}
int Model::frame_id(std::string_view n) const {
  auto it = frame_index.find(std::string(n));
  if (it == frame_index.end()) throw UnknownFrameError("unknown frame '" + std::string(n) + "'");
  return it->second;
}
int Model::joint_index(std::string_view n) const {
  for (size_t i = 0; i < joints.size(); ++i)
    if (joints[i].name == n) return (int)i;
  return -1;
}

// model.cpp:44-65: row i = e_i + row(parent(i)).
std::vector<double> build_ancestor_mask(const std::vector<int>& parents) {
  const size_t n = parents.size();
  std::vector<double> u(n * n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    const int p = parents[i];
    if (p >= (int)i)
      throw ModelError("build_ancestor_mask: joint " + std::to_string(i) +
                       " has forward or self parent reference " + std::to_string(p) +
                       " (parents must be topologically sorted)");
    if (p < -1) throw ModelError("build_ancestor_mask: invalid parent index " + std::to_string(p));
    u[i * n + i] = 1.0;
    if (p >= 0)
      for (size_t j = 0; j < n; ++j) u[i * n + j] += u[(size_t)p * n + j];
  }
  return u;
}

namespace {

static bool valid_rotation(const M3<double>& r, double tol = 1e-9) {  // spatial.hpp:270-273
  return max_abs(transpose(r) * r - M3<double>::identity()) <= tol && std::abs(det3(r) - 1.0) <= tol;
}

struct Graph {
  std::map<std::string, int> link_of;
  std::vector<std::vector<int>> kids;   // joints hanging under each link, name-sorted
  std::vector<int> parent_joint;        // joint whose child is the link (-1 root)
  int root = -1;
};

// model.cpp:78-135
Graph analyze(const Description& d) {
  Graph g;
  for (size_t i = 0; i < d.links.size(); ++i)
    if (!g.link_of.emplace(d.links[i].name, (int)i).second)
      throw ModelError("duplicate link name '" + d.links[i].name + "'");
  std::set<std::string> seen;
  g.kids.assign(d.links.size(), {});
  g.parent_joint.assign(d.links.size(), -1);
  std::vector<char> is_child(d.links.size(), 0);
  for (size_t j = 0; j < d.joints.size(); ++j) {
    const JointSpec& s = d.joints[j];
    if (!seen.insert(s.name).second) throw ModelError("duplicate joint name '" + s.name + "'");
    auto pit = g.link_of.find(s.parent_link);
    auto cit = g.link_of.find(s.child_link);
    if (pit == g.link_of.end())
      throw ModelError("joint '" + s.name + "' references unknown parent link '" + s.parent_link + "'");
    if (cit == g.link_of.end())
      throw ModelError("joint '" + s.name + "' references unknown child link '" + s.child_link + "'");
    if (is_child[(size_t)cit->second])
      throw ModelError("link '" + s.child_link + "' is the child of more than one joint");
    is_child[(size_t)cit->second] = 1;
    g.parent_joint[(size_t)cit->second] = (int)j;
    g.kids[(size_t)pit->second].push_back((int)j);
  }
  for (auto& k : g.kids)
    std::sort(k.begin(), k.end(), [&](int a, int b) { return d.joints[(size_t)a].name < d.joints[(size_t)b].name; });
  for (size_t i = 0; i < d.links.size(); ++i) {
    if (is_child[i]) continue;
    if (g.root >= 0)
      throw ModelError("model has multiple root links ('" + d.links[(size_t)g.root].name + "' and '" +
                       d.links[i].name + "')");
    g.root = (int)i;
  }
  if (g.root < 0) throw ModelError("model has no root link (joint graph contains a cycle)");
  return g;
}

}  // namespace

// model.cpp:214-287
Model build_model(const Description& d) {
  const Graph g = analyze(d);
  for (size_t i = 0; i < d.links.size(); ++i) {
    const LinkSpec& l = d.links[i];
    if (l.has_inertial || (int)i == g.root) continue;
    const int pj = g.parent_joint[i];
    const bool moving_in = pj >= 0 && d.joints[(size_t)pj].type != JointType::Fixed;
    bool moving_out = false;
    for (int j : g.kids[i]) moving_out |= d.joints[(size_t)j].type != JointType::Fixed;
    if (moving_in && moving_out)
      throw ModelError("link '" + l.name + "' has no inertial but carries a moving child joint");
  }

  Model m;
  std::vector<char> visited(d.links.size(), 0);
  std::vector<int> depth;
  // DFS in name-sorted child order; fixed joints are fused into the nearest
  // moving ancestor (model.cpp:175-209).
  std::function<void(int, int, const Xform<double>&)> walk = [&](int link, int mover, const Xform<double>& rel) {
    visited[(size_t)link] = 1;
    const LinkSpec& ls = d.links[(size_t)link];
    if (m.frame_index.count(ls.name)) throw ModelError("duplicate frame name '" + ls.name + "'");
    m.frame_index.emplace(ls.name, (int)m.frames.size());
    m.frames.push_back(Frame{ls.name, mover, rel});
    if (mover >= 0) {
      const Mat6<double> li = ls.has_inertial ? inertia_from_params(ls.mass, ls.com, ls.inertia) : Mat6<double>();
      m.inertias[(size_t)mover] = m.inertias[(size_t)mover] + transform_inertia(rel, li);
      m.total_mass += ls.mass;
    }
    for (int j : g.kids[(size_t)link]) {
      const JointSpec& s = d.joints[(size_t)j];
      if (!valid_rotation(s.origin.R)) throw ModelError("joint '" + s.name + "' origin rotation is not orthonormal");
      const int child = g.link_of.at(s.child_link);
      if (s.type == JointType::Fixed) {
        walk(child, mover, rel * s.origin);
        continue;
      }
      const double nrm = norm3(s.axis);
      if (std::abs(nrm - 1.0) > 1e-9)
        throw ModelError("joint '" + s.name + "' axis has norm " + std::to_string(nrm) + "; expected a unit vector");
      Joint jt;
      jt.name = s.name;
      jt.type = s.type;
      jt.parent = mover;
      jt.offset = rel * s.origin;
      jt.axis = V3<double>(s.axis[0] / nrm, s.axis[1] / nrm, s.axis[2] / nrm);  // model.cpp:325 (spec.axis / norm)
      jt.limits = s.limits;
      const int idx = (int)m.joints.size();
      m.joints.push_back(jt);
      m.inertias.push_back(Mat6<double>());
      depth.push_back(mover >= 0 ? depth[(size_t)mover] + 1 : 1);
      walk(child, idx, Xform<double>::identity());
    }
  };
  walk(g.root, -1, Xform<double>::identity());
  for (size_t i = 0; i < d.links.size(); ++i)
    if (!visited[i])
      throw ModelError("link '" + d.links[i].name + "' is not connected to the root link '" +
                       d.links[(size_t)g.root].name + "'");

  m.name = d.name;
  m.description = d;
  const int n = m.dof();
  std::vector<int> parents((size_t)n);
  for (int i = 0; i < n; ++i) parents[(size_t)i] = m.joints[(size_t)i].parent;
  m.mask = build_ancestor_mask(parents);
  m.max_depth = depth.empty() ? 0 : *std::max_element(depth.begin(), depth.end());
  m.serial = true;
  for (int i = 0; i < n; ++i)
    if (parents[(size_t)i] != i - 1) m.serial = false;
  for (int i = 0; i < n; ++i) {
    bool has_kids = false;
    for (const Joint& j : m.joints) has_kids |= j.parent == i;
    if (has_kids && m.inertias[(size_t)i](5, 5) <= 0.0)
      m.warnings.push_back("joint '" + m.joints[(size_t)i].name + "' drives a zero-mass link but has moving children");
  }
  return m;
}

// model.cpp:289-331: prismatic x,y,z then revolute z,y,x, massless stages.
Model floating_base(const Model& model) {
  const Description& o = model.description;
  std::set<std::string> kids;
  for (const JointSpec& j : o.joints) kids.insert(j.child_link);
  std::string root;
  for (const LinkSpec& l : o.links)
    if (!kids.count(l.name)) {
      root = l.name;
      break;
    }
  Description d;
  d.name = o.name.empty() ? "floating" : o.name + "_floating";
  d.add_link("__world");
  const char* stages[5] = {"__fb_x", "__fb_y", "__fb_z", "__fb_rz", "__fb_ry"};
  for (const char* s : stages) d.add_link(s, 0.0, V3<double>(), M3<double>());
  const Xform<double> I = Xform<double>::identity();
  d.add_joint("base_tx", JointType::Prismatic, "__world", "__fb_x", I, {1, 0, 0});
  d.add_joint("base_ty", JointType::Prismatic, "__fb_x", "__fb_y", I, {0, 1, 0});
  d.add_joint("base_tz", JointType::Prismatic, "__fb_y", "__fb_z", I, {0, 0, 1});
  d.add_joint("base_rz", JointType::Revolute, "__fb_z", "__fb_rz", I, {0, 0, 1});
  d.add_joint("base_ry", JointType::Revolute, "__fb_rz", "__fb_ry", I, {0, 1, 0});
  d.add_joint("base_rx", JointType::Revolute, "__fb_ry", root, I, {1, 0, 0});
  for (const LinkSpec& l : o.links) d.links.push_back(l);
  for (const JointSpec& j : o.joints) d.joints.push_back(j);
  return build_model(d);
}

// =====================================================================
// URDF — proj/core/src/urdf.cpp
// =====================================================================
namespace urdf {

// urdf.cpp:14-31: R = Rz(yaw) Ry(pitch) Rx(roll).
M3<double> rpy_to_rotation(double roll, double pitch, double yaw) {
  const double cr = std::cos(roll), sr = std::sin(roll);
  const double cp = std::cos(pitch), sp = std::sin(pitch);
  const double cy = std::cos(yaw), sy = std::sin(yaw);
  M3<double> rx = M3<double>::identity(), ry = M3<double>::identity(), rz = M3<double>::identity();
  rx(1, 1) = cr; rx(1, 2) = -sr; rx(2, 1) = sr; rx(2, 2) = cr;
  ry(0, 0) = cp; ry(0, 2) = sp; ry(2, 0) = -sp; ry(2, 2) = cp;
  rz(0, 0) = cy; rz(0, 1) = -sy; rz(1, 0) = sy; rz(1, 1) = cy;
  return (rz * ry) * rx;
}

namespace {

[[noreturn]] void fail_at(const xml::Element& e, const std::string& m) { throw ParseError(m, e.line, e.column); }

// urdf.cpp:39-56: std::stod, trailing whitespace only.
double number(const xml::Element& e, const std::string& text, const char* what) {
  size_t used = 0;
  double v = 0;
  try {
    v = std::stod(text, &used);
  } catch (const std::exception&) {
    fail_at(e, std::string("invalid number '") + text + "' in " + what);
  }
  while (used < text.size() && std::isspace((unsigned char)text[used])) ++used;
  if (used != text.size()) fail_at(e, std::string("invalid number '") + text + "' in " + what);
  return v;
}

V3<double> triple(const xml::Element& e, const std::string& text, const char* what) {
  std::istringstream in(text);
  V3<double> v;
  std::string tok;
  for (int k = 0; k < 3; ++k) {
    if (!(in >> tok)) fail_at(e, std::string("expected 3 numbers in ") + what + ", got '" + text + "'");
    v[k] = number(e, tok, what);
  }
  if (in >> tok) fail_at(e, std::string("expected 3 numbers in ") + what + ", got '" + text + "'");
  return v;
}

double need(const xml::Element& e, const char* a) {
  const std::string* v = e.attr(a);
  if (!v) fail_at(e, "<" + e.name + "> is missing the '" + a + "' attribute");
  return number(e, *v, a);
}

void origin_of(const xml::Element& parent, V3<double>* xyz, V3<double>* rpy) {
  const xml::Element* o = parent.child("origin");
  if (!o) return;
  if (const std::string* v = o->attr("xyz")) *xyz = triple(*o, *v, "origin xyz");
  if (const std::string* v = o->attr("rpy")) *rpy = triple(*o, *v, "origin rpy");
}

Link read_link(const xml::Element& e, std::vector<std::string>* warn) {  // urdf.cpp:95-132
  Link l;
  const std::string* nm = e.attr("name");
  if (!nm) fail_at(e, "<link> is missing the 'name' attribute");
  l.name = *nm;
  for (const xml::Element& c : e.children) {
    if (c.name != "inertial") {
      warn->push_back("link '" + l.name + "': skipped <" + c.name + "> element");
      continue;
    }
    l.inertial.present = true;
    origin_of(c, &l.inertial.xyz, &l.inertial.rpy);
    const xml::Element* ms = c.child("mass");
    if (!ms) fail_at(c, "link '" + l.name + "' inertial is missing <mass>");
    l.inertial.mass = need(*ms, "value");
    const xml::Element* in = c.child("inertia");
    if (!in) fail_at(c, "link '" + l.name + "' inertial is missing <inertia>");
    const double ixx = need(*in, "ixx"), ixy = need(*in, "ixy"), ixz = need(*in, "ixz");
    const double iyy = need(*in, "iyy"), iyz = need(*in, "iyz"), izz = need(*in, "izz");
    M3<double>& I = l.inertial.inertia;
    I(0, 0) = ixx; I(0, 1) = ixy; I(0, 2) = ixz;
    I(1, 0) = ixy; I(1, 1) = iyy; I(1, 2) = iyz;
    I(2, 0) = ixz; I(2, 1) = iyz; I(2, 2) = izz;
  }
  return l;
}

UJoint read_joint(const xml::Element& e, std::vector<std::string>* warn) {  // urdf.cpp:134-200
  UJoint j;
  const std::string* nm = e.attr("name");
  if (!nm) fail_at(e, "<joint> is missing the 'name' attribute");
  j.name = *nm;
  const std::string* ty = e.attr("type");
  if (!ty) fail_at(e, "joint '" + j.name + "' is missing the 'type' attribute");
  if (*ty == "revolute") j.type = JType::Revolute;
  else if (*ty == "continuous") j.type = JType::Continuous;
  else if (*ty == "prismatic") j.type = JType::Prismatic;
  else if (*ty == "fixed") j.type = JType::Fixed;
  else if (*ty == "planar" || *ty == "floating")
    throw UnsupportedFeatureError("joint '" + j.name + "' has unsupported type '" + *ty + "'");
  else fail_at(e, "joint '" + j.name + "' has unknown type '" + *ty + "'");
  const xml::Element* p = e.child("parent");
  const xml::Element* c = e.child("child");
  if (!p || !p->attr("link")) fail_at(e, "joint '" + j.name + "' is missing <parent link=...>");
  if (!c || !c->attr("link")) fail_at(e, "joint '" + j.name + "' is missing <child link=...>");
  j.parent_link = *p->attr("link");
  j.child_link = *c->attr("link");
  origin_of(e, &j.xyz, &j.rpy);
  if (const xml::Element* ax = e.child("axis"))
    if (const std::string* v = ax->attr("xyz")) j.axis = triple(*ax, *v, "axis xyz");
  if (const xml::Element* lim = e.child("limit")) {
    Limits L;
    if (const std::string* v = lim->attr("lower")) L.lower = number(*lim, *v, "limit lower");
    if (const std::string* v = lim->attr("upper")) L.upper = number(*lim, *v, "limit upper");
    if (const std::string* v = lim->attr("effort")) L.effort = number(*lim, *v, "limit effort");
    if (const std::string* v = lim->attr("velocity")) L.velocity = number(*lim, *v, "limit velocity");
    j.limits = L;
  }
  for (const xml::Element& s : e.children)
    if (s.name != "parent" && s.name != "child" && s.name != "origin" && s.name != "axis" && s.name != "limit")
      warn->push_back("joint '" + j.name + "': skipped <" + s.name + "> element");
  return j;
}

void check_structure(const Document& d) {  // urdf.cpp:202-239
  std::set<std::string> links, joints, kids;
  for (const Link& l : d.links)
    if (!links.insert(l.name).second) throw ModelError("duplicate link name '" + l.name + "'");
  for (const UJoint& j : d.joints) {
    if (!joints.insert(j.name).second) throw ModelError("duplicate joint name '" + j.name + "'");
    if (!links.count(j.parent_link))
      throw ModelError("joint '" + j.name + "' references unknown parent link '" + j.parent_link + "'");
    if (!links.count(j.child_link))
      throw ModelError("joint '" + j.name + "' references unknown child link '" + j.child_link + "'");
    if (!kids.insert(j.child_link).second)
      throw ModelError("link '" + j.child_link + "' is the child of more than one joint");
  }
  int roots = 0;
  for (const Link& l : d.links) roots += kids.count(l.name) ? 0 : 1;
  if (roots != 1)
    throw ModelError("document must have exactly one root link, found " + std::to_string(roots) +
                     (roots == 0 ? " (joint graph contains a cycle)" : ""));
}

std::string num(double v) {
  char b[32];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
std::string num3(const V3<double>& v) { return num(v[0]) + " " + num(v[1]) + " " + num(v[2]); }

}  // namespace

Document parse_urdf(std::string_view text) {
  const xml::Element root = xml::parse(text);
  if (root.name != "robot")
    throw ParseError("root element must be <robot>, found <" + root.name + ">", root.line, root.column);
  Document d;
  if (const std::string* n = root.attr("name")) d.robot_name = *n;
  for (const xml::Element& c : root.children) {
    if (c.name == "link") d.links.push_back(read_link(c, &d.warnings));
    else if (c.name == "joint") d.joints.push_back(read_joint(c, &d.warnings));
    else d.warnings.push_back("skipped <" + c.name + "> element");
  }
  check_structure(d);
  return d;
}

Document parse_urdf_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error("cannot open URDF file '" + path + "'");
  std::ostringstream ss;
  ss << f.rdbuf();
  return parse_urdf(ss.str());
}

std::string serialize_urdf(const Document& d) {
  std::ostringstream o;
  o << "<?xml version=\"1.0\"?>\n<robot name=\"" << d.robot_name << "\">\n";
  for (const Link& l : d.links) {
    o << "  <link name=\"" << l.name << "\">";
    if (l.inertial.present) {
      const Inertial& in = l.inertial;
      o << "\n    <inertial>\n      <origin xyz=\"" << num3(in.xyz) << "\" rpy=\"" << num3(in.rpy) << "\"/>\n"
        << "      <mass value=\"" << num(in.mass) << "\"/>\n"
        << "      <inertia ixx=\"" << num(in.inertia(0, 0)) << "\" ixy=\"" << num(in.inertia(0, 1))
        << "\" ixz=\"" << num(in.inertia(0, 2)) << "\" iyy=\"" << num(in.inertia(1, 1)) << "\" iyz=\""
        << num(in.inertia(1, 2)) << "\" izz=\"" << num(in.inertia(2, 2)) << "\"/>\n    </inertial>\n  ";
    }
    o << "</link>\n";
  }
  for (const UJoint& j : d.joints) {
    static const char* names[] = {"revolute", "continuous", "prismatic", "fixed"};
    o << "  <joint name=\"" << j.name << "\" type=\"" << names[(int)j.type] << "\">\n"
      << "    <parent link=\"" << j.parent_link << "\"/>\n    <child link=\"" << j.child_link << "\"/>\n"
      << "    <origin xyz=\"" << num3(j.xyz) << "\" rpy=\"" << num3(j.rpy) << "\"/>\n";
    if (j.type != JType::Fixed) o << "    <axis xyz=\"" << num3(j.axis) << "\"/>\n";
    if (j.limits)
      o << "    <limit lower=\"" << num(j.limits->lower) << "\" upper=\"" << num(j.limits->upper)
        << "\" effort=\"" << num(j.limits->effort) << "\" velocity=\"" << num(j.limits->velocity) << "\"/>\n";
    o << "  </joint>\n";
  }
  o << "</robot>\n";
  return o.str();
}

// urdf.cpp:337-382: inertia symmetrized then rotated by the inertial rpy
// (the com is NOT rotated); continuous -> revolute.
Description to_description(const Document& doc) {
  Description d;
  d.name = doc.robot_name;
  for (const Link& l : doc.links) {
    LinkSpec& s = d.add_link(l.name);
    if (!l.inertial.present) continue;
    const Inertial& in = l.inertial;
    const double scale = std::max(1.0, max_abs(in.inertia));
    if (max_abs(in.inertia - transpose(in.inertia)) > 1e-6 * scale)
      throw ModelError("link '" + l.name + "': inertia tensor is not symmetric");
    const M3<double> sym = 0.5 * (in.inertia + transpose(in.inertia));
    const M3<double> r = rpy_to_rotation(in.rpy[0], in.rpy[1], in.rpy[2]);
    s.has_inertial = true;
    s.mass = in.mass;
    s.com = in.xyz;
    s.inertia = (r * sym) * transpose(r);
  }
  for (const UJoint& j : doc.joints) {
    JointType t = JointType::Fixed;
    if (j.type == JType::Revolute || j.type == JType::Continuous) t = JointType::Revolute;
    else if (j.type == JType::Prismatic) t = JointType::Prismatic;
    Xform<double> x;
    x.R = rpy_to_rotation(j.rpy[0], j.rpy[1], j.rpy[2]);
    x.p = j.xyz;
    JointSpec& s = d.add_joint(j.name, t, j.parent_link, j.child_link, x, j.axis);
    s.limits = j.limits;
  }
  return d;
}

Model load_model(const std::string& path) { return build_model(to_description(parse_urdf_file(path))); }
Model load_model_from_string(std::string_view text) { return build_model(to_description(parse_urdf(text))); }

}  // namespace urdf

// =====================================================================
// Builtin robots — proj/core/src/robots.cpp:12-32
// =====================================================================
namespace robots {

std::string asset_text(const std::string& file) {
  std::vector<std::string> dirs;
  if (const char* env = std::getenv("VECDYN_ASSET_DIR")) dirs.push_back(env);
#ifdef ORC_ASSET_DIR
  dirs.push_back(ORC_ASSET_DIR);
#endif
  dirs.push_back("assets");
  for (const std::string& d : dirs) {
    std::ifstream f(d + "/" + file, std::ios::binary);
    if (!f) continue;
    std::ostringstream ss;
    ss << f.rdbuf();
    return ss.str();
  }
  throw Error("cannot locate asset '" + file + "'");
}

Model chain7() { return urdf::load_model_from_string(asset_text("chain7.urdf")); }
Model humanoid23() { return urdf::load_model_from_string(asset_text("humanoid23.urdf")); }
Model tree29() { return floating_base(humanoid23()); }
Model by_name(std::string_view n) {
  if (n == "chain7") return chain7();
  if (n == "humanoid23") return humanoid23();
  if (n == "tree29") return tree29();
  throw Error("unknown builtin robot '" + std::string(n) + "'; available: chain7, humanoid23, tree29");
}

}  // namespace robots
}  // namespace orc
