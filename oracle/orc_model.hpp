// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_spatial.hpp header).
//
// Restatement of the reference model layer: XML reader (proj/core/src/xml.cpp),
// URDF front-end (proj/core/src/urdf.cpp), model builder with name-sorted DFS
// and fixed-joint fusion (proj/core/src/model.cpp), floating base
// (model.cpp:289-331) and the builtin robots (proj/core/src/robots.cpp).
#pragma once

#include <map>
#include <optional>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "orc_spatial.hpp"

namespace orc {

// ------------------------------------------------------------------ xml
namespace xml {
struct Attr {
  std::string name, value;
};
struct Element {
  std::string name;
  std::vector<Attr> attrs;
  std::vector<Element> children;
  int line = 0, column = 0;
  const std::string* attr(std::string_view n) const;
  const Element* child(std::string_view tag) const;
  std::vector<const Element*> children_named(std::string_view tag) const;
};
Element parse(std::string_view text);  // xml.cpp:316
}  // namespace xml

// ------------------------------------------------------------------ model
enum class JointType { Revolute, Prismatic, Fixed };

struct Limits {
  double lower = 0, upper = 0, effort = 0, velocity = 0;
};

struct LinkSpec {  // model.hpp:25-31
  std::string name;
  bool has_inertial = false;
  double mass = 0;
  V3<double> com;
  M3<double> inertia;
};

struct JointSpec {  // model.hpp:35-43
  std::string name;
  JointType type = JointType::Fixed;
  std::string parent_link, child_link;
  Xform<double> origin;
  V3<double> axis{0, 0, 1};
  std::optional<Limits> limits;
};

struct Description {  // model.hpp:47-59
  std::string name;
  std::vector<LinkSpec> links;
  std::vector<JointSpec> joints;
  LinkSpec& add_link(const std::string& n);
  LinkSpec& add_link(const std::string& n, double mass, const V3<double>& com, const M3<double>& Ic);
  JointSpec& add_joint(const std::string& n, JointType t, const std::string& parent,
                       const std::string& child, const Xform<double>& origin,
                       const V3<double>& axis = V3<double>(0, 0, 1));
};

struct Joint {  // model.hpp:64-71
  std::string name;
  JointType type = JointType::Revolute;
  int parent = -1;
  Xform<double> offset;
  V3<double> axis{0, 0, 1};
  std::optional<Limits> limits;
};

struct Frame {  // model.hpp:74-78
  std::string name;
  int joint = -1;
  Xform<double> offset;
};

// RobotModel, model.hpp:90-149.  Immutable after build.
struct Model {
  std::string name;
  std::vector<Joint> joints;
  std::vector<Mat6<double>> inertias;
  std::vector<double> mask;  // n*n row-major, mask[i*n+j] = U(i,j)
  std::vector<Frame> frames;
  std::unordered_map<std::string, int> frame_index;
  int max_depth = 0;
  bool serial = false;
  double total_mass = 0;
  std::vector<std::string> warnings;
  Description description;

  int dof() const { return (int)joints.size(); }
  double U(int i, int j) const { return mask[(size_t)i * joints.size() + j]; }
  bool has_frame(std::string_view n) const { return frame_index.count(std::string(n)) != 0; }
  const Frame& frame(std::string_view n) const;  // UnknownFrameError
  int frame_id(std::string_view n) const;
  int joint_index(std::string_view n) const;
};

std::vector<double> build_ancestor_mask(const std::vector<int>& parents);  // model.cpp:44-65
Model build_model(const Description& d);                                   // model.cpp:214-287
Model floating_base(const Model& m);                                      // model.cpp:289-331

// ------------------------------------------------------------------ urdf
namespace urdf {
enum class JType { Revolute, Continuous, Prismatic, Fixed };
struct Inertial {
  bool present = false;
  double mass = 0;
  V3<double> xyz, rpy;
  M3<double> inertia;
};
struct Link {
  std::string name;
  Inertial inertial;
};
struct UJoint {
  std::string name;
  JType type = JType::Fixed;
  std::string parent_link, child_link;
  V3<double> xyz, rpy;
  V3<double> axis{1, 0, 0};  // URDF default (urdf.hpp:30)
  std::optional<Limits> limits;
};
struct Document {
  std::string robot_name;
  std::vector<Link> links;
  std::vector<UJoint> joints;
  std::vector<std::string> warnings;
};
M3<double> rpy_to_rotation(double roll, double pitch, double yaw);  // urdf.cpp:14-31
Document parse_urdf(std::string_view text);                          // urdf.cpp:254-275
Document parse_urdf_file(const std::string& path);
std::string serialize_urdf(const Document& doc);                     // urdf.cpp:287-335
Description to_description(const Document& doc);                     // urdf.cpp:337-382
Model load_model(const std::string& path);
Model load_model_from_string(std::string_view text);
}  // namespace urdf

// ------------------------------------------------------------------ robots
namespace robots {
// robots.cpp:12-32.  Asset text is read from VECDYN_ASSET_DIR or the repo's
// assets/ directory (byte-identical copies of proj/assets).
std::string asset_text(const std::string& file);
Model chain7();
Model humanoid23();
Model tree29();
Model by_name(std::string_view name);
}  // namespace robots

}  // namespace orc
