// vecdyn_b200/vecdyn.hpp — C++ host API mirroring the reference `vecdyn`
// names over the C-ABI (include/vecdyn_cuda.h).  Header-only; link with
// paper_2604_04310_b200/lib/libvecdyn_cuda.so.
//
// Reference interface                          this header
//   vecdyn::robots::chain7() ...  robots.hpp:11-20    vecdyn::robots::chain7() ...
//   vecdyn::urdf::load_model(path) urdf.hpp:70         vecdyn::urdf::load_model(path)
//   vecdyn::floating_base(model)   model.hpp:163       vecdyn::floating_base(model)
//   vecdyn::RobotModel             model.hpp:90-149    vecdyn::RobotModel (dof, joint_names, frame, ...)
//   vecdyn::GravitySpec            dynamics.hpp:39     vecdyn::GravitySpec
//   vecdyn::StateBatch / random_states   batch.hpp:15-75   same (column-major N x n, std::vector)
//   vecdyn::batch_rnea / batch_crba / batch_forward_dynamics  batch.hpp:128-165
//                                                   same, `workers` replaced by a device list
//   vecdyn::rnea / crba / forward_dynamics / ... on device buffers:
//                                                   vecdyn::device::* (DeviceModel + raw device pointers)
//
// Errors are re-thrown as the reference exception types (errors.hpp:9-61).
// Eigen callers: Eigen::MatrixXd is column-major, so batch.q.data() can be
// passed to the batch functions unchanged (StateBatch layout, batch.hpp:17-21).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../vecdyn_cuda.h"

namespace vecdyn {

// ------------------------------------------------------------------ errors (errors.hpp:9-61)
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionError : public Error {
 public:
  using Error::Error;
};
class ModelError : public Error {
 public:
  using Error::Error;
};
class UnknownFrameError : public ModelError {
 public:
  using ModelError::ModelError;
};
class ParseError : public Error {
 public:
  ParseError(const std::string& m, int l, int c) : Error(m), line(l), column(c) {}
  int line;
  int column;
};
class UnsupportedFeatureError : public Error {
 public:
  using Error::Error;
};
class UnsupportedStructureError : public Error {
 public:
  using Error::Error;
};
class SingularInertiaError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

namespace detail {
inline void check(int rc) {
  if (rc == VD_OK) return;
  const std::string msg = vd_last_error();
  switch (rc) {
    case VD_ERR_DIMENSION: throw DimensionError(msg);
    case VD_ERR_PARSE: throw ParseError(msg, vd_last_error_line(), vd_last_error_column());
    case VD_ERR_MODEL: throw ModelError(msg);
    case VD_ERR_UNKNOWN_FRAME: throw UnknownFrameError(msg);
    case VD_ERR_UNSUPPORTED_FEATURE: throw UnsupportedFeatureError(msg);
    case VD_ERR_UNSUPPORTED_STRUCTURE: throw UnsupportedStructureError(msg);
    case VD_ERR_SINGULAR_INERTIA: throw SingularInertiaError(msg);
    case VD_ERR_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}
}  // namespace detail

// ------------------------------------------------------------------ model
class RobotModel {
 public:
  explicit RobotModel(vd_model h) : h_(h, &vd_model_destroy) {}
  vd_model handle() const { return h_.get(); }
  int dof() const { return vd_model_dof(handle()); }
  int max_depth() const { return vd_model_max_depth(handle()); }
  bool is_serial_chain() const { return vd_model_is_serial_chain(handle()) == 1; }
  double total_mass() const { return vd_model_total_mass(handle()); }
  std::string name() const {
    char b[256];
    detail::check(vd_model_name(handle(), b, sizeof b));
    return b;
  }
  std::vector<int> parents() const {
    std::vector<int> p((size_t)dof());
    if (!p.empty()) detail::check(vd_model_parents(handle(), p.data()));
    return p;
  }
  // (rows, cols) of crba_packed's planes (vd_model_crba_pattern)
  std::pair<std::vector<int32_t>, std::vector<int32_t>> crba_pattern() const {
    int nnz = 0;
    detail::check(vd_model_crba_pattern(handle(), nullptr, nullptr, &nnz));
    std::vector<int32_t> r((size_t)nnz), c((size_t)nnz);
    if (nnz) detail::check(vd_model_crba_pattern(handle(), r.data(), c.data(), &nnz));
    return {r, c};
  }
  std::string joint_name(int i) const {
    char b[256];
    detail::check(vd_model_joint_name(handle(), i, b, sizeof b));
    return b;
  }
  int joint_index(std::string_view name) const { return vd_model_joint_index(handle(), std::string(name).c_str()); }
  // Attach this model's JIT module of generated routines (vd_model_attach_jit;
  // built by `python -m paper_2604_04310_b200.jit model.urdf`).
  void attach_jit(const std::string& module_path) { detail::check(vd_model_attach_jit(handle(), module_path.c_str())); }
  int frame_index(std::string_view name) const {  // RobotModel::frame, model.cpp:337-343
    int k = -1;
    detail::check(vd_model_frame_index(handle(), std::string(name).c_str(), &k));
    return k;
  }
  bool has_frame(std::string_view name) const {
    int k = -1;
    return vd_model_frame_index(handle(), std::string(name).c_str(), &k) == VD_OK;
  }
  std::vector<std::string> warnings() const {
    std::vector<std::string> w;
    for (int k = 0; k < vd_model_warning_count(handle()); ++k) {
      char b[512];
      detail::check(vd_model_warning(handle(), k, b, sizeof b));
      w.emplace_back(b);
    }
    return w;
  }

 private:
  std::shared_ptr<vd_model_s> h_;
};

namespace robots {
inline RobotModel by_name(std::string_view name) {
  vd_model h = nullptr;
  detail::check(vd_model_builtin(std::string(name).c_str(), &h));
  return RobotModel(h);
}
inline RobotModel chain7() { return by_name("chain7"); }
inline RobotModel humanoid23() { return by_name("humanoid23"); }
inline RobotModel tree29() { return by_name("tree29"); }
}  // namespace robots

namespace urdf {
inline RobotModel load_model(const std::string& path) {
  vd_model h = nullptr;
  detail::check(vd_model_load_urdf(path.c_str(), &h));
  return RobotModel(h);
}
inline RobotModel load_model_from_string(std::string_view text) {
  vd_model h = nullptr;
  detail::check(vd_model_load_urdf_string(text.data(), text.size(), &h));
  return RobotModel(h);
}
}  // namespace urdf

inline RobotModel floating_base(const RobotModel& m) {
  vd_model h = nullptr;
  detail::check(vd_model_floating_base(m.handle(), &h));
  return RobotModel(h);
}

struct GravitySpec {  // dynamics.hpp:35-50
  double accel[3] = {0.0, 0.0, 9.81};
  static GravitySpec standard() { return GravitySpec(); }
  static GravitySpec zero() { return GravitySpec{{0.0, 0.0, 0.0}}; }
  static GravitySpec from_field(double fx, double fy, double fz) { return GravitySpec{{-fx, -fy, -fz}}; }
};

// ------------------------------------------------------------------ batch layer (batch.hpp)
struct StateBatch {  // column-major N x n (element (i, j) at j*N + i)
  int64_t N = 0;
  int n = 0;
  std::vector<double> q, qd, qdd, tau;
  int64_t size() const { return N; }
  void validate(const RobotModel& model) const {
    if (n != model.dof()) throw DimensionError("StateBatch: q has " + std::to_string(n) + " columns, model has " +
                                               std::to_string(model.dof()) + " dof");
    const size_t want = (size_t)N * (size_t)n;
    for (const auto* v : {&q, &qd, &qdd, &tau})
      if (!v->empty() && v->size() != want) throw DimensionError("StateBatch: inconsistent buffer size");
  }
};

inline StateBatch random_states(const RobotModel& model, int64_t count, uint64_t seed, bool with_qdd = true,
                                bool with_tau = false) {
  StateBatch b;
  b.N = count;
  b.n = model.dof();
  const size_t sz = (size_t)count * (size_t)b.n;
  b.q.resize(sz);
  b.qd.resize(sz);
  if (with_qdd) b.qdd.resize(sz);
  if (with_tau) b.tau.resize(sz);
  detail::check(vd_random_states(model.handle(), count, seed, b.q.data(), b.qd.data(),
                                 with_qdd ? b.qdd.data() : nullptr, with_tau ? b.tau.data() : nullptr));
  return b;
}

// batch_rnea(model, batch, gravity, workers) -> rows are torque vectors (column-major N x n)
inline std::vector<double> batch_rnea(const RobotModel& model, const StateBatch& b,
                                      const GravitySpec& g = GravitySpec::standard(),
                                      const std::vector<int>& devices = {0}) {
  b.validate(model);
  std::vector<double> out((size_t)b.N * b.n);
  detail::check(vd_batch_rnea_host(model.handle(), b.N, b.q.data(), b.qd.data(), b.qdd.data(), g.accel, out.data(),
                                   devices.data(), (int)devices.size()));
  return out;
}
// batch_crba: rows are column-major flattened n x n matrices (batch.hpp:147-148)
inline std::vector<double> batch_crba(const RobotModel& model, const StateBatch& b,
                                      const std::vector<int>& devices = {0}) {
  b.validate(model);
  std::vector<double> out((size_t)b.N * b.n * b.n);
  detail::check(vd_batch_crba_host(model.handle(), b.N, b.q.data(), out.data(), devices.data(), (int)devices.size()));
  return out;
}
// batch_forward_dynamics (ABA on the device); SingularInertiaError like the reference
inline std::vector<double> batch_forward_dynamics(const RobotModel& model, const StateBatch& b,
                                                  const GravitySpec& g = GravitySpec::standard(),
                                                  const std::vector<int>& devices = {0}) {
  b.validate(model);
  std::vector<double> out((size_t)b.N * b.n);
  detail::check(vd_batch_forward_dynamics_host(model.handle(), b.N, b.q.data(), b.qd.data(), b.tau.data(), g.accel,
                                               out.data(), nullptr, devices.data(), (int)devices.size()));
  return out;
}

// ------------------------------------------------------------------ device-resident API
namespace device {

class DeviceModel {
 public:
  DeviceModel(const RobotModel& m, int device = 0) : model_(m) {
    vd_device_model h = nullptr;
    detail::check(vd_device_model_create(m.handle(), device, &h));
    h_.reset(h, &vd_device_model_destroy);
  }
  vd_device_model handle() const { return h_.get(); }
  const RobotModel& model() const { return model_; }
  int dof() const { return vd_device_model_dof(handle()); }
  int specialization() const { return vd_device_model_specialization(handle()); }

 private:
  RobotModel model_;
  std::shared_ptr<vd_device_model_s> h_;
};

enum class DType { F64 = VD_F64, F32 = VD_F32 };

// All pointers are device buffers in the SoA column-major layout of the C-ABI.
inline void rnea(const DeviceModel& dm, DType t, int64_t N, const void* q, const void* qd, const void* qdd,
                 void* tau, const GravitySpec& g = GravitySpec::standard(), const void* fext = nullptr,
                 void* stream = nullptr) {
  detail::check(vd_rnea(dm.handle(), (int)t, N, q, qd, qdd, N, g.accel, fext, tau, N, stream));
}
inline void crba(const DeviceModel& dm, DType t, int64_t N, const void* q, void* M, void* stream = nullptr) {
  detail::check(vd_crba(dm.handle(), (int)t, N, q, N, M, N, stream));
}
// M's branch-sparse lower triangle; plane k = M(rows[k], cols[k]) of crba_pattern
inline void crba_packed(const DeviceModel& dm, DType t, int64_t N, const void* q, void* M_packed,
                        void* stream = nullptr) {
  detail::check(vd_crba_packed(dm.handle(), (int)t, N, q, N, M_packed, N, stream));
}
inline void forward_dynamics(const DeviceModel& dm, DType t, int64_t N, const void* q, const void* qd,
                             const void* tau, void* qdd, int32_t* status = nullptr,
                             const GravitySpec& g = GravitySpec::standard(), const void* fext = nullptr,
                             void* stream = nullptr) {
  detail::check(vd_aba(dm.handle(), (int)t, N, q, qd, tau, N, g.accel, fext, qdd, N, status, stream));
}
// Per-state gravity (no reference analogue): gravity_planes = 3 device planes
// of a_g (= −field), state i's vector at (gravity_planes[i], [N + i], [2N + i]).
struct GravityPlanes {
  const void* planes;
};
inline void rnea(const DeviceModel& dm, DType t, int64_t N, const void* q, const void* qd, const void* qdd,
                 void* tau, GravityPlanes g, const void* fext = nullptr, void* stream = nullptr) {
  detail::check(vd_rnea_pg(dm.handle(), (int)t, N, q, qd, qdd, N, g.planes, fext, tau, N, stream));
}
inline void forward_dynamics(const DeviceModel& dm, DType t, int64_t N, const void* q, const void* qd,
                             const void* tau, void* qdd, int32_t* status, GravityPlanes g,
                             const void* fext = nullptr, void* stream = nullptr) {
  detail::check(vd_aba_pg(dm.handle(), (int)t, N, q, qd, tau, N, g.planes, fext, qdd, N, status, stream));
}
inline void forward_kinematics(const DeviceModel& dm, DType t, int64_t N, const void* q, void* frames,
                               void* stream = nullptr) {
  detail::check(vd_fk(dm.handle(), (int)t, N, q, N, frames, N, stream));
}
inline void geometric_jacobian(const DeviceModel& dm, DType t, int64_t N, const void* q, std::string_view frame,
                               void* pose, void* J, void* stream = nullptr) {
  detail::check(vd_jacobian(dm.handle(), (int)t, N, q, N, dm.model().frame_index(frame), pose, J, N, stream));
}

}  // namespace device
}  // namespace vecdyn
