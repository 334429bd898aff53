// Plain data shared by the host ABI layer (g++) and the kernels (nvcc).
#pragma once

#include <cstdint>

namespace vdk {

constexpr int kMaxDof = 64;

constexpr int kFlagLeaf = 1;
constexpr int kFlagBranch = 2;
constexpr int kOffRotIdentity = 1;  // offset rotation is exactly the identity
constexpr int kOffTransZero = 2;    // offset translation is exactly zero
constexpr int kMassless = 4;        // all 10 inertia parameters are zero

// Device-resident model for the generic (runtime-topology) kernels.
template <class T>
struct DevModel {
  int n;
  int parent[kMaxDof];
  int kind[kMaxDof];       // 0 revolute, 1 prismatic
  int axis_code[kMaxDof];  // 0..2 +x,+y,+z; 3..5 -x,-y,-z; 6 general
  int depth[kMaxDof];      // moving joints on the path root..i (1 for root joints)
  uint64_t anc[kMaxDof];   // bit j set iff j is i or an ancestor of i (ancestor mask row)
  int flags[kMaxDof];      // kFlagLeaf: no children; kFlagBranch: has a child other than i+1
  int oflags[kMaxDof];     // kOffRotIdentity | kOffTransZero | kMassless
  T axis[kMaxDof][3];
  T R[kMaxDof][9];         // offset rotation, row-major
  T p[kMaxDof][3];
  T I[kMaxDof][10];        // m, h(3), Ixx Iyy Izz Ixy Ixz Iyz (about the joint origin)
};

// Per-launch OSC constants (vd_osc_params, control.hpp:12-42).
struct OscShared {
  int frame_joint;
  double frame_R[9], frame_p[3];    // frame offset, row-major R
  double target_R[9], target_p[3];  // row-major
  double kp[6], kd[6], accel_ff[6];
  double posture[kMaxDof];
  double posture_kp, posture_kd;
  double gravity[3];
  double epsilon;
};

// Per-launch task constants for diff_ik_step / manipulability
// (vd_task_params, control.hpp:25-37, 79-97; kinematics.hpp:138-153).
struct TaskShared {
  int frame_joint;
  double frame_R[9], frame_p[3];    // frame offset, row-major R
  double target_R[9], target_p[3];  // row-major
  double kp[6], twist_ff[6];
  double damping;
};

}  // namespace vdk
