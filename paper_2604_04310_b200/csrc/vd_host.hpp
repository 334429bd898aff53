// Host-side model layer of the B200 library: URDF/XML reader, model builder
// and the packer that turns a RobotModel into the device-resident tree.
//
// Semantics follow the reference exactly (it is the input side of the drop-in
// boundary): xml.cpp (reader), urdf.cpp:14-31/254-390 (URDF, Rz·Ry·Rx rpy,
// inertia rotated by the inertial rpy, continuous -> revolute), model.cpp
// (name-sorted DFS, fixed-joint fusion and inertia folding, ancestor mask,
// floating base).  The oracle/ restatement is NOT used here.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace vdh {

// ---------------------------------------------------------------- errors (errors.hpp:9-61)
struct Failure : std::runtime_error {
  int code;
  int line = 0, column = 0;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
  Failure(int c, const std::string& m, int l, int col)
      : std::runtime_error(m + " (line " + std::to_string(l) + ", column " + std::to_string(col) + ")"),
        code(c),
        line(l),
        column(col) {}
};
enum Code {
  kDimension = 1,
  kParse = 2,
  kModel = 3,
  kUnknownFrame = 4,
  kUnsupportedFeature = 5,
  kUnsupportedStructure = 6,
  kSingular = 7,
  kCuda = 8,
  kInvalid = 9,
  kIo = 10,
  kGeneric = 11,
};

// ---------------------------------------------------------------- small linear algebra
using Vec3 = std::array<double, 3>;
using Mat3 = std::array<double, 9>;   // row-major
using Mat6 = std::array<double, 36>;  // row-major
Mat3 mat3_identity();
Mat3 mat3_mul(const Mat3& a, const Mat3& b);
Vec3 mat3_vec(const Mat3& a, const Vec3& v);
Mat3 mat3_transpose(const Mat3& a);

struct Pose {  // x_parent = R x_child + p (spatial.hpp:129-131)
  Mat3 R = mat3_identity();
  Vec3 p{0, 0, 0};
};
Pose compose(const Pose& a, const Pose& b);

// ---------------------------------------------------------------- description / model
enum class Kind { Revolute, Prismatic, Fixed };

struct LinkDesc {
  std::string name;
  bool has_inertial = false;
  double mass = 0;
  Vec3 com{0, 0, 0};
  Mat3 inertia{};  // about the com, link axes
};
struct JointDesc {
  std::string name;
  Kind kind = Kind::Fixed;
  std::string parent, child;
  Pose origin;
  Vec3 axis{0, 0, 1};
  bool has_limits = false;
  double limits[4] = {0, 0, 0, 0};
};
struct Description {
  std::string name;
  std::vector<LinkDesc> links;
  std::vector<JointDesc> joints;
};

struct Body {  // one moving joint after fusion (model.hpp:64-71)
  std::string name;
  Kind kind = Kind::Revolute;
  int parent = -1;
  Pose offset;
  Vec3 axis{0, 0, 1};
  Mat6 inertia{};  // folded spatial inertia about the joint frame origin
  int depth = 1;
};
struct NamedFrame {
  std::string name;
  int joint = -1;
  Pose offset;
};
struct Model {
  std::string name;
  std::vector<Body> bodies;
  std::vector<NamedFrame> frames;
  std::map<std::string, int> frame_of;
  int max_depth = 0;
  bool serial = false;
  double total_mass = 0;
  std::vector<std::string> warnings;
  Description source;
  int dof() const { return (int)bodies.size(); }
  int frame_index(std::string_view name) const;  // throws kUnknownFrame
};

Model build(const Description& d);           // model.cpp:214-287
Model with_floating_base(const Model& m);    // model.cpp:289-331
Description parse_urdf_text(std::string_view text);  // urdf.cpp:254-275 + 337-382
Model load_urdf_text(std::string_view text);
Model load_urdf_file(const std::string& path);
Model builtin(std::string_view name);        // robots.cpp:12-32 (assets compiled in)

// ---------------------------------------------------------------- packed device tree
// Per-joint constants as the kernels consume them.  Inertia in 10-parameter
// form (m, h = m c, rotational inertia about the joint origin Ixx Iyy Izz Ixy
// Ixz Iyz) — exact for every folded inertia because each term keeps the
// [[I_o, h×], [h×ᵀ, m 1]] structure (spatial.hpp:291-297, model.cpp:180-181);
// the packer checks the residual.
constexpr int kMaxDof = 64;
constexpr int kMaxFrames = 128;

// axis code: 0..2 = +x,+y,+z; 3..5 = -x,-y,-z; 6 = general
struct PackedModel {
  int n = 0;
  int nframes = 0;
  int parent[kMaxDof];
  int kind[kMaxDof];       // 0 revolute, 1 prismatic
  int axis_code[kMaxDof];
  double axis[kMaxDof][3];
  double R[kMaxDof][9];    // offset rotation, row-major
  double p[kMaxDof][3];
  double inertia[kMaxDof][10];
  int frame_joint[kMaxFrames];
  double frame_R[kMaxFrames][9];
  double frame_p[kMaxFrames][3];
};
PackedModel pack(const Model& m);
// 64-bit FNV-1a over the packed numerical content (used to match compiled robots).
uint64_t fingerprint(const PackedModel& pm);

}  // namespace vdh
