// C-ABI implementation (include/vecdyn_cuda.h).  Host-side argument checking,
// model handles, device-model upload, kernel dispatch and the multi-device
// host batch path.  No CPU fallback exists: every numeric entry point runs
// the sm_100a kernels or fails with VD_ERR_CUDA.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/vecdyn_cuda.h"
#include "vd_shared.hpp"
#include "vd_host.hpp"
#include "vd_launch.hpp"

// A per-model JIT module (vd_jit_entry.cuh) loaded with dlopen.  Never
// unloaded: launches may still be in flight on some stream when the last
// model referencing it goes away.
struct JitModule {
  void* dl = nullptr;
  uint64_t fp = 0;
  vdk::JitLaunchFn launch = nullptr;
  vdk::JitTaskFn task_launch = nullptr;  // modules generated with task frames
  uint64_t task_mask = 0;
};

struct vd_model_s {
  vdh::Model m;
  std::shared_ptr<JitModule> jit;  // vd_model_attach_jit; read/written under jit_mutex()
};

// A model is otherwise immutable and shared across threads (model.hpp:86-89);
// attaching a JIT module is its one mutation.
static std::mutex& jit_mutex() {
  static std::mutex mu;
  return mu;
}

struct vd_device_model_s {
  int device = 0;
  int n = 0;
  int spec = 0;
  bool force_generic = false;
  std::shared_ptr<JitModule> jit;  // the model's JIT module (models without compile-time kernels)
  vdh::PackedModel pm;
  // Host copies of the packed model; the generic kernels receive them by
  // value in their parameter space (__grid_constant__), so no device
  // allocation is needed and a device model is valid on its device only.
  std::unique_ptr<vdk::DevModel<double>> h64;
  std::unique_ptr<vdk::DevModel<float>> h32;
};

namespace {

thread_local std::string g_msg;
thread_local int g_line = 0, g_col = 0;

int set_error(int code, const std::string& msg, int line = 0, int col = 0) {
  g_msg = msg;
  g_line = line;
  g_col = col;
  return code;
}
int from_failure(const vdh::Failure& f) { return set_error(f.code, f.what(), f.line, f.column); }
int cuda_fail(cudaError_t e, const char* where) {
  // Consume the thread's last-error state: a failed API call (not a sticky
  // context error) must not resurface as the result of the next launch check.
  cudaGetLastError();
  return set_error(VD_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
void copy_str(const std::string& s, char* buf, size_t len) {
  if (buf && len) std::snprintf(buf, len, "%s", s.c_str());
}
void pose_to_colmajor(const vdh::Pose& x, double* out12) {
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) out12[c * 3 + r] = x.R[r * 3 + c];
  for (int r = 0; r < 3; ++r) out12[9 + r] = x.p[r];
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const vdh::Failure& e) {
    return from_failure(e);
  } catch (const std::bad_alloc&) {
    return set_error(VD_ERR_GENERIC, "out of host memory");
  } catch (const std::exception& e) {
    return set_error(VD_ERR_GENERIC, e.what());
  }
}

template <class T>
void fill_dev_model(const vdh::PackedModel& pm, vdk::DevModel<T>& d) {
  std::memset(&d, 0, sizeof d);
  d.n = pm.n;
  for (int i = 0; i < pm.n; ++i) {
    d.parent[i] = pm.parent[i];
    d.kind[i] = pm.kind[i];
    d.axis_code[i] = pm.axis_code[i];
    d.depth[i] = pm.parent[i] < 0 ? 1 : d.depth[pm.parent[i]] + 1;
    d.anc[i] = (1ull << i) | (pm.parent[i] < 0 ? 0ull : d.anc[pm.parent[i]]);
    d.flags[i] = vdk::kFlagLeaf;
    {
      bool rid = true, tz = true, ml = true;
      for (int k = 0; k < 9; ++k) rid = rid && pm.R[i][k] == ((k % 4 == 0) ? 1.0 : 0.0);
      for (int k = 0; k < 3; ++k) tz = tz && pm.p[i][k] == 0.0;
      for (int k = 0; k < 10; ++k) ml = ml && pm.inertia[i][k] == 0.0;
      d.oflags[i] = (rid ? vdk::kOffRotIdentity : 0) | (tz ? vdk::kOffTransZero : 0) | (ml ? vdk::kMassless : 0);
    }
    for (int k = 0; k < 3; ++k) {
      d.axis[i][k] = T(pm.axis[i][k]);
      d.p[i][k] = T(pm.p[i][k]);
    }
    for (int k = 0; k < 9; ++k) d.R[i][k] = T(pm.R[i][k]);
    for (int k = 0; k < 10; ++k) d.I[i][k] = T(pm.inertia[i][k]);
  }
  for (int i = 0; i < pm.n; ++i) {
    const int p = pm.parent[i];
    if (p < 0) continue;
    d.flags[p] &= ~vdk::kFlagLeaf;
    if (p != i - 1) d.flags[p] |= vdk::kFlagBranch;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int check_common(vd_device_model dm, int dtype, int64_t N, int64_t ld_in, int64_t ld_out) {
  if (!dm) return set_error(VD_ERR_INVALID_ARGUMENT, "null device model");
  if (dtype != VD_F64 && dtype != VD_F32) return set_error(VD_ERR_INVALID_ARGUMENT, "dtype must be VD_F64 or VD_F32");
  if (N < 0) return set_error(VD_ERR_DIMENSION, "negative batch size");
  if (N > 0 && (ld_in < N || ld_out < N))
    return set_error(VD_ERR_DIMENSION, "leading dimension smaller than the batch size");
  return VD_OK;
}
#define VD_NEED(ptr, what)                                                  \
  do {                                                                      \
    if (N > 0 && dm->n > 0 && !(ptr)) return set_error(VD_ERR_INVALID_ARGUMENT, "null " what " buffer"); \
  } while (0)

vdk::Launch make_launch(vd_device_model dm, int dtype, int64_t N, int64_t ldi, int64_t ldo, void* stream) {
  vdk::Launch L;
  L.spec = dm->force_generic ? vdk::kGeneric : dm->spec;
  L.dtype = dtype;
  L.n = dm->n;
  L.model = dtype == VD_F64 ? static_cast<const void*>(dm->h64.get()) : static_cast<const void*>(dm->h32.get());
  L.N = N;
  L.ld_in = ldi;
  L.ld_out = ldo;
  L.stream = stream;
  L.serial = true;
  for (int i = 0; i < dm->n; ++i) L.serial = L.serial && dm->pm.parent[i] == i - 1;
  if (!dm->force_generic && dm->jit) {
    L.jit = dm->jit->launch;
    L.jit_task = dm->jit->task_launch;
    L.jit_task_mask = dm->jit->task_mask;
  }
  return L;
}
int finish(int rc, const char* where) {
  if (rc != 0) return cuda_fail((cudaError_t)rc, where);
  return VD_OK;
}

}  // namespace

extern "C" {

const char* vd_last_error(void) { return g_msg.c_str(); }
int vd_last_error_line(void) { return g_line; }
int vd_last_error_column(void) { return g_col; }
const char* vd_version(void) { return "vecdyn-b200 0.1 (sm_100a)"; }

// ------------------------------------------------------------------ host model
int vd_model_builtin(const char* name, vd_model* out) {
  if (!name || !out) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = new vd_model_s{vdh::builtin(name)};
    return VD_OK;
  });
}
int vd_model_load_urdf(const char* path, vd_model* out) {
  if (!path || !out) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = new vd_model_s{vdh::load_urdf_file(path)};
    return VD_OK;
  });
}
int vd_model_load_urdf_string(const char* text, size_t len, vd_model* out) {
  if (!text || !out) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = new vd_model_s{vdh::load_urdf_text(std::string_view(text, len))};
    return VD_OK;
  });
}
int vd_model_floating_base(vd_model m, vd_model* out) {
  if (!m || !out) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = new vd_model_s{vdh::with_floating_base(m->m)};
    return VD_OK;
  });
}
void vd_model_destroy(vd_model m) { delete m; }
int vd_model_dof(vd_model m) { return m ? m->m.dof() : -1; }
int vd_model_max_depth(vd_model m) { return m ? m->m.max_depth : -1; }
int vd_model_is_serial_chain(vd_model m) { return m ? (m->m.serial ? 1 : 0) : -1; }
double vd_model_total_mass(vd_model m) { return m ? m->m.total_mass : NAN; }
int vd_model_warning_count(vd_model m) { return m ? (int)m->m.warnings.size() : -1; }
int vd_model_warning(vd_model m, int k, char* buf, size_t len) {
  if (!m || k < 0 || k >= (int)m->m.warnings.size()) return set_error(VD_ERR_INVALID_ARGUMENT, "bad warning index");
  copy_str(m->m.warnings[(size_t)k], buf, len);
  return VD_OK;
}
int vd_model_name(vd_model m, char* buf, size_t len) {
  if (!m) return set_error(VD_ERR_INVALID_ARGUMENT, "null model");
  copy_str(m->m.name, buf, len);
  return VD_OK;
}
int vd_model_parents(vd_model m, int* parents) {
  if (!m || !parents) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  for (int i = 0; i < m->m.dof(); ++i) parents[i] = m->m.bodies[(size_t)i].parent;
  return VD_OK;
}
int vd_model_joint_name(vd_model m, int i, char* buf, size_t len) {
  if (!m || i < 0 || i >= m->m.dof()) return set_error(VD_ERR_INVALID_ARGUMENT, "bad joint index");
  copy_str(m->m.bodies[(size_t)i].name, buf, len);
  return VD_OK;
}
int vd_model_joint_index(vd_model m, const char* name) {
  if (!m || !name) return -1;
  for (int i = 0; i < m->m.dof(); ++i)
    if (m->m.bodies[(size_t)i].name == name) return i;
  return -1;
}
int vd_model_joint(vd_model m, int i, int* type, double axis[3], double offset[12], double inertia[36]) {
  if (!m || i < 0 || i >= m->m.dof()) return set_error(VD_ERR_INVALID_ARGUMENT, "bad joint index");
  const vdh::Body& b = m->m.bodies[(size_t)i];
  if (type) *type = b.kind == vdh::Kind::Revolute ? 0 : 1;
  if (axis)
    for (int k = 0; k < 3; ++k) axis[k] = b.axis[k];
  if (offset) pose_to_colmajor(b.offset, offset);
  if (inertia)
    for (int k = 0; k < 36; ++k) inertia[k] = b.inertia[k];
  return VD_OK;
}
int vd_model_ancestor_mask(vd_model m, double* mask) {
  if (!m || !mask) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  const int n = m->m.dof();
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) {
      bool anc = false;
      for (int j = r; j >= 0; j = m->m.bodies[(size_t)j].parent)
        if (j == c) anc = true;
      mask[c * n + r] = anc ? 1.0 : 0.0;
    }
  return VD_OK;
}
int vd_model_crba_pattern(vd_model m, int32_t* rows, int32_t* cols, int* nnz) {
  if (!m || !nnz) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  const int n = m->m.dof();
  int k = 0;
  for (int c = 0; c < n; ++c)
    for (int r = c; r < n; ++r) {
      int j = r;
      while (j >= 0 && j != c) j = m->m.bodies[(size_t)j].parent;
      if (j != c) continue;
      if (rows) rows[k] = r;
      if (cols) cols[k] = c;
      ++k;
    }
  *nnz = k;
  return VD_OK;
}
int vd_model_frame_count(vd_model m) { return m ? (int)m->m.frames.size() : -1; }
int vd_model_frame(vd_model m, int k, char* name, size_t len, int* joint, double offset[12]) {
  if (!m || k < 0 || k >= (int)m->m.frames.size()) return set_error(VD_ERR_INVALID_ARGUMENT, "bad frame index");
  const vdh::NamedFrame& f = m->m.frames[(size_t)k];
  copy_str(f.name, name, len);
  if (joint) *joint = f.joint;
  if (offset) pose_to_colmajor(f.offset, offset);
  return VD_OK;
}
int vd_model_frame_index(vd_model m, const char* name, int* out) {
  if (!m || !name || !out) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = m->m.frame_index(name);
    return VD_OK;
  });
}

int vd_random_states(vd_model m, int64_t N, uint64_t seed, double* q, double* qd, double* qdd, double* tau) {
  if (!m || N < 0 || (N > 0 && (!q || !qd))) return set_error(VD_ERR_INVALID_ARGUMENT, "bad argument");
  // batch.hpp:48-75: one mt19937_64 stream, per state per joint q, qd, [qdd], [tau].
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-M_PI, M_PI);
  const int n = m->m.dof();
  for (int64_t i = 0; i < N; ++i)
    for (int j = 0; j < n; ++j) {
      const int64_t k = (int64_t)j * N + i;
      q[k] = dist(rng);
      qd[k] = dist(rng);
      if (qdd) qdd[k] = dist(rng);
      if (tau) tau[k] = dist(rng);
    }
  return VD_OK;
}

// ------------------------------------------------------------------ device model
int vd_device_model_create(vd_model m, int device, vd_device_model* out) {
  if (!m || !out) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&]() -> int {
    auto dm = std::make_unique<vd_device_model_s>();
    dm->device = device;
    dm->pm = vdh::pack(m->m);
    dm->n = dm->pm.n;
    dm->spec = vdk::match_spec(vdh::fingerprint(dm->pm), dm->pm.n);
    if (dm->spec == vdk::kGeneric) {  // builtin robots keep their compiled-in kernels
      std::lock_guard<std::mutex> lk(jit_mutex());
      dm->jit = m->jit;
    }
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= count) return set_error(VD_ERR_CUDA, "device index out of range");
    DeviceGuard g(device);
    dm->h64 = std::make_unique<vdk::DevModel<double>>();
    dm->h32 = std::make_unique<vdk::DevModel<float>>();
    fill_dev_model(dm->pm, *dm->h64);
    fill_dev_model(dm->pm, *dm->h32);
    // touch the device so a missing / broken GPU fails here, loudly
    if ((e = cudaFree(nullptr)) != cudaSuccess) return cuda_fail(e, "cudaFree(0)");
    *out = dm.release();
    return VD_OK;
  });
}
void vd_device_model_destroy(vd_device_model dm) {
  if (!dm) return;
  delete dm;
}
int vd_device_model_dof(vd_device_model dm) { return dm ? dm->n : -1; }
int vd_device_model_jit(vd_device_model dm) { return dm ? ((dm->jit && !dm->force_generic) ? 1 : 0) : -1; }

int vd_model_attach_jit(vd_model m, const char* path) {
  if (!m || !path) return set_error(VD_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&]() -> int {
    void* dl = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!dl) return set_error(VD_ERR_INVALID_ARGUMENT, std::string("vd_model_attach_jit: ") + dlerror());
    auto abi = reinterpret_cast<int (*)()>(dlsym(dl, "vdj_abi_version"));
    auto fpf = reinterpret_cast<uint64_t (*)()>(dlsym(dl, "vdj_fingerprint"));
    auto init = reinterpret_cast<void (*)(int (*)(void**, size_t, void*), void (*)(void*, void*))>(dlsym(dl, "vdj_init"));
    auto launch = reinterpret_cast<vdk::JitLaunchFn>(dlsym(dl, "vdj_launch"));
    auto refuse = [&](const char* why) {
      dlclose(dl);  // nothing from a refused module was ever called into
      return set_error(VD_ERR_INVALID_ARGUMENT, std::string("vd_model_attach_jit: ") + why);
    };
    if (!abi || !fpf || !init || !launch) return refuse("not a vecdyn JIT module");
    if (abi() != vdk::kJitAbi) return refuse("JIT ABI mismatch");
    const uint64_t fp = vdh::fingerprint(vdh::pack(m->m));
    if (fpf() != fp) return refuse("module was generated for another model");
    init(&vdk::scratch_alloc, &vdk::scratch_free);
    auto jm = std::make_shared<JitModule>();
    jm->dl = dl;
    jm->fp = fp;
    jm->launch = launch;
    auto tmask = reinterpret_cast<uint64_t (*)()>(dlsym(dl, "vdj_task_mask"));
    jm->task_launch = reinterpret_cast<vdk::JitTaskFn>(dlsym(dl, "vdj_task_launch"));
    jm->task_mask = (tmask && jm->task_launch) ? tmask() : 0;
    std::lock_guard<std::mutex> lk(jit_mutex());
    m->jit = std::move(jm);
    return VD_OK;
  });
}
int vd_device_model_specialization(vd_device_model dm) { return dm ? (dm->force_generic ? 0 : dm->spec) : -1; }
int vd_device_model_set_generic(vd_device_model dm, int generic) {
  if (!dm) return set_error(VD_ERR_INVALID_ARGUMENT, "null device model");
  dm->force_generic = generic != 0;
  return VD_OK;
}

// ------------------------------------------------------------------ kernels
int vd_fk(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* out, int64_t ld_out,
          void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  VD_NEED(out, "output");
  if (dm->n == 0) return VD_OK;
  DeviceGuard g(dm->device);
  return finish(vdk::launch_fk(make_launch(dm, dtype, N, ld_in, ld_out, stream), q, out), "vd_fk");
}

int vd_fk_scan(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* out, int64_t ld_out,
               void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  // kinematics.hpp:63-67: serial chains only
  bool serial = true;
  for (int i = 0; i < dm->n; ++i) serial = serial && dm->pm.parent[i] == i - 1;
  if (!serial)
    return set_error(VD_ERR_UNSUPPORTED_STRUCTURE,
                     "forward_kinematics_scan requires a serial chain (every joint's parent must be its predecessor)");
  if (dm->n > 32) return set_error(VD_ERR_UNSUPPORTED_STRUCTURE, "forward_kinematics_scan supports at most 32 joints");
  VD_NEED(q, "q");
  VD_NEED(out, "output");
  if (dm->n == 0) return VD_OK;
  DeviceGuard g(dm->device);
  vdk::Launch L = make_launch(dm, dtype, N, ld_in, ld_out, stream);
  L.spec = vdk::kGeneric;
  return finish(vdk::launch_fk_scan(L, q, out), "vd_fk_scan");
}

int vd_jacobian(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, int frame, void* pose,
                void* J, int64_t ld_out, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  if (frame < 0 || frame >= dm->pm.nframes) return set_error(VD_ERR_UNKNOWN_FRAME, "frame index out of range");
  VD_NEED(q, "q");
  if (N == 0 || (!pose && !J)) return VD_OK;
  DeviceGuard g(dm->device);
  return finish(vdk::launch_jacobian(make_launch(dm, dtype, N, ld_in, ld_out, stream), q, dm->pm.frame_joint[frame],
                                     dm->pm.frame_R[frame], dm->pm.frame_p[frame], pose, dm->n ? J : nullptr),
                "vd_jacobian");
}

static int rnea_mode(vd_device_model dm, int dtype, int mode, int64_t N, const void* q, const void* qd,
                     const void* qdd, int64_t ld_in, const double* g3, const void* fext, void* out, int64_t ld_out,
                     void* stream, const void* gravity_planes = nullptr, bool pg = false) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  if (pg) VD_NEED(gravity_planes, "gravity_planes");
  VD_NEED(q, "q");
  if (mode != 2) VD_NEED(qd, "qd");
  if (mode == 0) VD_NEED(qdd, "qdd");
  VD_NEED(out, "output");
  if (dm->n == 0) return VD_OK;
  DeviceGuard g(dm->device);
  vdk::Launch L = make_launch(dm, dtype, N, ld_in, ld_out, stream);
  L.gravity_planes = gravity_planes;
  return finish(vdk::launch_rnea(L, mode, q, qd, qdd, g3, fext, out), "vd_rnea");
}
int vd_rnea(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* qdd, int64_t ld_in,
            const double* g3, const void* fext, void* tau, int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 0, N, q, qd, qdd, ld_in, g3, fext, tau, ld_out, stream);
}
int vd_bias(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in, const double* g3,
            const void* fext, void* out, int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 1, N, q, qd, nullptr, ld_in, g3, fext, out, ld_out, stream);
}
int vd_gravity(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, const double* g3, void* out,
               int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 2, N, q, nullptr, nullptr, ld_in, g3, nullptr, out, ld_out, stream);
}
// per-state gravity: the same calls with a_g read from 3 planes
int vd_rnea_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* qdd,
               int64_t ld_in, const void* gravity_planes, const void* fext, void* tau, int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 0, N, q, qd, qdd, ld_in, nullptr, fext, tau, ld_out, stream, gravity_planes, true);
}
int vd_bias_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in,
               const void* gravity_planes, const void* fext, void* out, int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 1, N, q, qd, nullptr, ld_in, nullptr, fext, out, ld_out, stream, gravity_planes, true);
}
int vd_gravity_pg(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, const void* gravity_planes,
                  void* out, int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 2, N, q, nullptr, nullptr, ld_in, nullptr, nullptr, out, ld_out, stream, gravity_planes,
                   true);
}
int vd_coriolis(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in, void* out,
                int64_t ld_out, void* stream) {
  return rnea_mode(dm, dtype, 3, N, q, qd, nullptr, ld_in, nullptr, nullptr, out, ld_out, stream);
}

int vd_crba(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* M, int64_t ld_out,
            void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  VD_NEED(M, "M");
  if (dm->n == 0) return VD_OK;
  DeviceGuard g(dm->device);
  return finish(vdk::launch_crba(make_launch(dm, dtype, N, ld_in, ld_out, stream), q, M), "vd_crba");
}

int vd_crba_packed(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* Mp, int64_t ld_out,
                   void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  VD_NEED(Mp, "M_packed");
  if (dm->n == 0) return VD_OK;
  // vd_model_crba_pattern's order, from the packed parents (same topology)
  vdk::PackTable tab{};
  const int n = dm->n;
  for (int c = 0; c < n; ++c)
    for (int r = c; r < n; ++r) {
      int j = r;
      while (j >= 0 && j != c) j = dm->pm.parent[j];
      if (j == c) tab.src[tab.nnz++] = (uint16_t)(c * n + r);
    }
  DeviceGuard g(dm->device);
  return finish(vdk::launch_crba_packed(make_launch(dm, dtype, N, ld_in, ld_out, stream), q, Mp, tab),
                "vd_crba_packed");
}

static int aba_call(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
                    int64_t ld_in, const double* g3, const void* gravity_planes, const void* fext, void* qdd,
                    int64_t ld_out, int32_t* status, void* stream, bool pg = false) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  if (pg) VD_NEED(gravity_planes, "gravity_planes");
  VD_NEED(q, "q");
  VD_NEED(qd, "qd");
  VD_NEED(tau, "tau");
  VD_NEED(qdd, "qdd");
  if (dm->n == 0) {
    if (status && N > 0 && cudaMemsetAsync(status, 0, sizeof(int32_t) * N, (cudaStream_t)stream) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "vd_aba");
    return VD_OK;
  }
  DeviceGuard g(dm->device);
  vdk::Launch L = make_launch(dm, dtype, N, ld_in, ld_out, stream);
  L.gravity_planes = gravity_planes;
  return finish(vdk::launch_aba(L, q, qd, tau, g3, fext, qdd, status), "vd_aba");
}
int vd_aba(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau, int64_t ld_in,
           const double* g3, const void* fext, void* qdd, int64_t ld_out, int32_t* status, void* stream) {
  return aba_call(dm, dtype, N, q, qd, tau, ld_in, g3, nullptr, fext, qdd, ld_out, status, stream);
}
int vd_aba_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau, int64_t ld_in,
              const void* gravity_planes, const void* fext, void* qdd, int64_t ld_out, int32_t* status, void* stream) {
  return aba_call(dm, dtype, N, q, qd, tau, ld_in, nullptr, gravity_planes, fext, qdd, ld_out, status, stream, true);
}

static int dynamics_call(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
                         int64_t ld_in, const double* g3, const void* gravity_planes, void* M, void* bias, void* qdd,
                         int64_t ld_out, int32_t* status, void* stream, bool pg = false) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  if (pg) VD_NEED(gravity_planes, "gravity_planes");
  VD_NEED(q, "q");
  VD_NEED(qd, "qd");
  if (qdd) VD_NEED(tau, "tau");
  if (dm->n == 0) return VD_OK;
  DeviceGuard g(dm->device);
  vdk::Launch L = make_launch(dm, dtype, N, ld_in, ld_out, stream);
  L.gravity_planes = gravity_planes;
  return finish(vdk::launch_dynamics(L, q, qd, tau, g3, M, bias, qdd, status), "vd_dynamics");
}
int vd_dynamics(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
                int64_t ld_in, const double* g3, void* M, void* bias, void* qdd, int64_t ld_out, int32_t* status,
                void* stream) {
  return dynamics_call(dm, dtype, N, q, qd, tau, ld_in, g3, nullptr, M, bias, qdd, ld_out, status, stream);
}
int vd_dynamics_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
                   int64_t ld_in, const void* gravity_planes, void* M, void* bias, void* qdd, int64_t ld_out,
                   int32_t* status, void* stream) {
  return dynamics_call(dm, dtype, N, q, qd, tau, ld_in, nullptr, gravity_planes, M, bias, qdd, ld_out, status, stream,
                       true);
}

int vd_osc(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in,
           const vd_osc_params* P, void* tau, void* lambda, int64_t ld_out, int32_t* status, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  if (!P) return set_error(VD_ERR_INVALID_ARGUMENT, "null osc parameters");
  if (P->frame < 0 || P->frame >= dm->pm.nframes) return set_error(VD_ERR_UNKNOWN_FRAME, "frame index out of range");
  for (int k = 0; k < 6; ++k)
    if (P->kp[k] < 0.0 || P->kd[k] < 0.0) return set_error(VD_ERR_GENERIC, "task gains must be nonnegative");
  if (dm->n > 0 && !P->posture) return set_error(VD_ERR_INVALID_ARGUMENT, "null posture");
  VD_NEED(q, "q");
  VD_NEED(qd, "qd");
  VD_NEED(tau, "tau");
  if (dm->n == 0) return VD_OK;
  vdk::OscShared S;
  std::memset(&S, 0, sizeof S);
  const int f = P->frame;
  S.frame_joint = dm->pm.frame_joint[f];
  for (int k = 0; k < 9; ++k) S.frame_R[k] = dm->pm.frame_R[f][k];
  for (int k = 0; k < 3; ++k) S.frame_p[k] = dm->pm.frame_p[f][k];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) S.target_R[r * 3 + c] = P->target[c * 3 + r];
  for (int k = 0; k < 3; ++k) S.target_p[k] = P->target[9 + k];
  for (int k = 0; k < 6; ++k) {
    S.kp[k] = P->kp[k];
    S.kd[k] = P->kd[k];
    S.accel_ff[k] = P->accel_ff[k];
  }
  for (int k = 0; k < dm->n; ++k) S.posture[k] = P->posture[k];
  S.posture_kp = P->posture_kp;
  S.posture_kd = P->posture_kd;
  for (int k = 0; k < 3; ++k) S.gravity[k] = P->gravity[k];
  S.epsilon = P->epsilon;
  DeviceGuard g(dm->device);
  return finish(vdk::launch_osc(make_launch(dm, dtype, N, ld_in, ld_out, stream), q, qd, S, tau, lambda, status),
                "vd_osc");
}

namespace {
void task_frame(const vd_device_model dm, int f, vdk::TaskShared& S) {
  std::memset(&S, 0, sizeof S);
  S.frame_joint = dm->pm.frame_joint[f];
  for (int k = 0; k < 9; ++k) S.frame_R[k] = dm->pm.frame_R[f][k];
  for (int k = 0; k < 3; ++k) S.frame_p[k] = dm->pm.frame_p[f][k];
}
}  // namespace

int vd_diff_ik(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, const vd_task_params* P,
               void* qdot, void* err, int64_t ld_out, int32_t* status, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  if (!P) return set_error(VD_ERR_INVALID_ARGUMENT, "null task parameters");
  if (!(P->damping > 0.0)) return set_error(VD_ERR_GENERIC, "diff_ik_step: damping must be positive");
  for (int k = 0; k < 6; ++k)
    if (P->kp[k] < 0.0) return set_error(VD_ERR_GENERIC, "task gains must be nonnegative");
  if (P->frame < 0 || P->frame >= dm->pm.nframes) return set_error(VD_ERR_UNKNOWN_FRAME, "frame index out of range");
  VD_NEED(q, "q");
  VD_NEED(qdot, "qdot");
  vdk::TaskShared S;
  task_frame(dm, P->frame, S);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) S.target_R[r * 3 + c] = P->target[c * 3 + r];
  for (int k = 0; k < 3; ++k) S.target_p[k] = P->target[9 + k];
  for (int k = 0; k < 6; ++k) {
    S.kp[k] = P->kp[k];
    S.twist_ff[k] = P->twist_ff[k];
  }
  S.damping = P->damping;
  DeviceGuard g(dm->device);
  return finish(vdk::launch_task(make_launch(dm, dtype, N, ld_in, ld_out, stream), q, S, 0, qdot, err, status),
                "vd_diff_ik");
}

int vd_manipulability(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, int frame, void* w,
                      void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_in)) return rc;
  if (frame < 0 || frame >= dm->pm.nframes) return set_error(VD_ERR_UNKNOWN_FRAME, "frame index out of range");
  VD_NEED(q, "q");
  VD_NEED(w, "w");
  vdk::TaskShared S;
  task_frame(dm, frame, S);
  DeviceGuard g(dm->device);
  return finish(vdk::launch_task(make_launch(dm, dtype, N, ld_in, ld_in, stream), q, S, 1, w, nullptr, nullptr),
                "vd_manipulability");
}

int vd_manipulability_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* dq, int64_t ld_in,
                          int frame, void* w, void* dw, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_in)) return rc;
  if (frame < 0 || frame >= dm->pm.nframes) return set_error(VD_ERR_UNKNOWN_FRAME, "frame index out of range");
  VD_NEED(q, "q");
  if (N > 0 && dm->n > 0 && !w && !dw) return set_error(VD_ERR_INVALID_ARGUMENT, "null output buffers");
  vdk::TaskShared S;
  task_frame(dm, frame, S);
  DeviceGuard g(dm->device);
  return finish(vdk::launch_manip_jvp(make_launch(dm, dtype, N, ld_in, ld_in, stream), q, dq, S, w, dw),
                "vd_manipulability_jvp");
}

// ---- forward-mode JVPs (autodiff.hpp:41-56 applied to the library's own functions)
// gravity3 is a host array (NULL = GravitySpec::standard()); it travels by value.
static double gcomp(const double* g3, int k) { return g3 ? g3[k] : (k == 2 ? 9.81 : 0.0); }
static int jvp_launch(vd_device_model dm, int dtype, int64_t N, int64_t ld_in, int64_t ld_out, void* stream,
                      const vdk::JvpArgs& a, const char* what) {
  if (N > 0 && dm->n > 0 && !a.out && !a.dout) return set_error(VD_ERR_INVALID_ARGUMENT, "null output buffers");
  if (dm->n == 0) {
    if (a.status && N > 0 && cudaMemsetAsync(a.status, 0, sizeof(int32_t) * N, (cudaStream_t)stream) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), what);
    return VD_OK;
  }
  DeviceGuard g(dm->device);
  return finish(vdk::launch_jvp(make_launch(dm, dtype, N, ld_in, ld_out, stream), a), what);
}

int vd_fk_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* dq, int64_t ld_in, void* frames,
              void* dframes, int64_t ld_out, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  vdk::JvpArgs a{vdk::kJvpFK, {q, nullptr, nullptr}, {dq, nullptr, nullptr}, {0.0, 0.0, 0.0}, nullptr, frames, dframes, nullptr};
  return jvp_launch(dm, dtype, N, ld_in, ld_out, stream, a, "vd_fk_jvp");
}

int vd_rnea_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* qdd,
                const void* dq, const void* dqd, const void* dqdd, int64_t ld_in, const double* g3, const void* fext,
                void* tau, void* dtau, int64_t ld_out, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  VD_NEED(qd, "qd");
  VD_NEED(qdd, "qdd");
  vdk::JvpArgs a{vdk::kJvpRNEA, {q, qd, qdd}, {dq, dqd, dqdd}, {gcomp(g3, 0), gcomp(g3, 1), gcomp(g3, 2)}, fext, tau, dtau, nullptr};
  return jvp_launch(dm, dtype, N, ld_in, ld_out, stream, a, "vd_rnea_jvp");
}

int vd_crba_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* dq, int64_t ld_in, void* M,
                void* dM, int64_t ld_out, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  vdk::JvpArgs a{vdk::kJvpCRBA, {q, nullptr, nullptr}, {dq, nullptr, nullptr}, {0.0, 0.0, 0.0}, nullptr, M, dM, nullptr};
  return jvp_launch(dm, dtype, N, ld_in, ld_out, stream, a, "vd_crba_jvp");
}

int vd_aba_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
               const void* dq, const void* dqd, const void* dtau, int64_t ld_in, const double* g3, const void* fext,
               void* qdd, void* dqdd, int64_t ld_out, int32_t* status, void* stream) {
  if (int rc = check_common(dm, dtype, N, ld_in, ld_out)) return rc;
  VD_NEED(q, "q");
  VD_NEED(qd, "qd");
  VD_NEED(tau, "tau");
  vdk::JvpArgs a{vdk::kJvpABA, {q, qd, tau}, {dq, dqd, dtau}, {gcomp(g3, 0), gcomp(g3, 1), gcomp(g3, 2)}, fext, qdd, dqdd, status};
  return jvp_launch(dm, dtype, N, ld_in, ld_out, stream, a, "vd_aba_jvp");
}

// ---- internal (not in the public header): packed tables for the robot-table generator
uint64_t vdi_model_fingerprint(vd_model m) { return m ? vdh::fingerprint(vdh::pack(m->m)) : 0; }
int vdi_model_packed(vd_model m, int* n, int* parent, int* kind, int* axis_code, double* axis, double* R, double* p,
                     double* inertia) {
  if (!m) return set_error(VD_ERR_INVALID_ARGUMENT, "null model");
  return guarded([&] {
    const vdh::PackedModel pm = vdh::pack(m->m);
    *n = pm.n;
    for (int i = 0; i < pm.n; ++i) {
      parent[i] = pm.parent[i];
      kind[i] = pm.kind[i];
      axis_code[i] = pm.axis_code[i];
      for (int k = 0; k < 3; ++k) axis[i * 3 + k] = pm.axis[i][k];
      for (int k = 0; k < 9; ++k) R[i * 9 + k] = pm.R[i][k];
      for (int k = 0; k < 3; ++k) p[i * 3 + k] = pm.p[i][k];
      for (int k = 0; k < 10; ++k) inertia[i * 10 + k] = pm.inertia[i][k];
    }
    return VD_OK;
  });
}

static int layout_call(int dtype, bool to_planes, int64_t N, int K, const void* src, int64_t ld_src, void* dst,
                       int64_t ld_dst, void* stream, const char* where) {
  if (dtype != VD_F64 && dtype != VD_F32) return set_error(VD_ERR_INVALID_ARGUMENT, "dtype must be VD_F64 or VD_F32");
  if (N < 0 || K < 0) return set_error(VD_ERR_DIMENSION, "negative size");
  if (N == 0 || K == 0) return VD_OK;
  if (!src || !dst) return set_error(VD_ERR_INVALID_ARGUMENT, "null buffer");
  const int64_t ld_rows = to_planes ? ld_src : ld_dst, ld_planes = to_planes ? ld_dst : ld_src;
  if (ld_rows < K || ld_planes < N) return set_error(VD_ERR_DIMENSION, "leading dimension too small");
  return finish(vdk::launch_layout(dtype == VD_F64 ? 0 : 1, to_planes, N, K, src, ld_src, dst, ld_dst, stream), where);
}
int vd_rows_to_planes(int dtype, int64_t N, int K, const void* rows, int64_t ld_rows, void* planes, int64_t ld_planes,
                      void* stream) {
  return layout_call(dtype, true, N, K, rows, ld_rows, planes, ld_planes, stream, "vd_rows_to_planes");
}
int vd_planes_to_rows(int dtype, int64_t N, int K, const void* planes, int64_t ld_planes, void* rows, int64_t ld_rows,
                      void* stream) {
  return layout_call(dtype, false, N, K, planes, ld_planes, rows, ld_rows, stream, "vd_planes_to_rows");
}

int vd_shard_range(int64_t N, int world, int rank, int64_t* begin, int64_t* end) {
  if (world <= 0 || rank < 0 || rank >= world || N < 0 || !begin || !end)
    return set_error(VD_ERR_INVALID_ARGUMENT, "bad shard arguments");
  // batch.hpp:111-119: chunk = ceil(count / workers), contiguous.
  const int64_t chunk = (N + world - 1) / world;
  *begin = std::min<int64_t>(N, (int64_t)rank * chunk);
  *end = std::min<int64_t>(N, *begin + chunk);
  return VD_OK;
}

// ------------------------------------------------------------------ host batch (multi-device)
// Drop-in for batch.hpp's batch_* helpers on HOST buffers.  Each device owns a
// persistent context (device model, two streams, double-buffered device
// chunks) so repeated calls do not re-allocate; the shard of each device is
// streamed in chunks with H2D(k+1) / kernel(k) / D2H(k-1) overlapping across
// the two streams.  Pinned host buffers are DMA'd directly; pageable ones go
// through pinned staging buffers.
namespace {
struct HostOp {
  int kind;  // 0 rnea, 1 crba, 2 fd
  int n_in;  // number of n-wide inputs
  int out_width;
};

// Chunks in flight per device: each slot owns a stream, device buffers and an
// event, and a slot is reused only once its previous chunk's D2H has landed.
// (3 or 4 slots measured the same as 2: tools/e2e_chunk.py.)
constexpr int kPipeSlots = 2;

struct DevCtx {
  std::mutex mu;
  int device = -1;
  vd_device_model dm = nullptr;
  uint64_t fp = 0;
  int n = -1;
  const void* jit_id = nullptr;  // the model's JIT module the cached device model was created with
  cudaStream_t st[kPipeSlots] = {};
  cudaEvent_t done[kPipeSlots] = {};
  double* din[kPipeSlots][3] = {};
  double* dout[kPipeSlots] = {};
  int32_t* dst[kPipeSlots] = {};
  double* pin_in[kPipeSlots][3] = {};  // staging (pageable inputs)
  double* pin_out[kPipeSlots] = {};
  int32_t* pin_st[kPipeSlots] = {};
  int64_t cap = 0;      // states per chunk buffer
  int64_t cap_in = 0;   // doubles per input chunk buffer
  int64_t cap_out = 0;  // doubles per output chunk buffer
  int64_t cap_pin = 0;     // doubles per pinned staging buffer
  int64_t cap_pin_st = 0;  // states per pinned status buffer
};

DevCtx& ctx_for(int device) {
  static std::mutex g;
  static std::map<int, std::unique_ptr<DevCtx>> all;
  std::lock_guard<std::mutex> lk(g);
  auto& p = all[device];
  if (!p) {
    p = std::make_unique<DevCtx>();
    p->device = device;
  }
  return *p;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int prepare_ctx(DevCtx& c, vd_model m, int n, int64_t chunk, int width, bool staging) {
  cudaError_t e;
  const uint64_t fp = vdh::fingerprint(vdh::pack(m->m));
  const void* jit_id;
  {
    std::lock_guard<std::mutex> lk(jit_mutex());
    jit_id = m->jit.get();
  }
  if (!c.dm || c.fp != fp || c.n != n || c.jit_id != jit_id) {
    if (c.dm) vd_device_model_destroy(c.dm);
    c.dm = nullptr;
    if (int rc = vd_device_model_create(m, c.device, &c.dm)) return rc;
    c.fp = fp;
    c.n = n;
    c.jit_id = jit_id;
  }
  if (!c.st[0]) {
    for (int k = 0; k < kPipeSlots; ++k) {
      if ((e = cudaStreamCreateWithFlags(&c.st[k], cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
      if ((e = cudaEventCreateWithFlags(&c.done[k], cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
    }
  }
  const int64_t need_out = chunk * width;
  if (chunk * n > c.cap_in || need_out > c.cap_out || c.cap < chunk) {
    // Release everything and zero the capacities first: a failed cudaMalloc
    // below must leave the context empty, never holding freed pointers.
    for (int b = 0; b < kPipeSlots; ++b) {
      for (int k = 0; k < 3; ++k) cudaFree(std::exchange(c.din[b][k], nullptr));
      cudaFree(std::exchange(c.dout[b], nullptr));
      cudaFree(std::exchange(c.dst[b], nullptr));
    }
    c.cap = c.cap_in = c.cap_out = 0;
    for (int b = 0; b < kPipeSlots; ++b) {
      for (int k = 0; k < 3; ++k)
        if ((e = cudaMalloc(&c.din[b][k], sizeof(double) * n * chunk)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
      if ((e = cudaMalloc(&c.dout[b], sizeof(double) * need_out)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
      if ((e = cudaMalloc(&c.dst[b], sizeof(int32_t) * chunk)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    }
    c.cap = chunk;
    c.cap_in = chunk * n;
    c.cap_out = need_out;
  }
  // (the status buffers are sized by states, the value buffers by planes: a
  // wide-output call with small chunks must not leave a short status buffer)
  if (staging && (c.cap_pin < chunk * std::max(n, width) || c.cap_pin_st < chunk)) {
    for (int b = 0; b < kPipeSlots; ++b) {
      for (int k = 0; k < 3; ++k) cudaFreeHost(std::exchange(c.pin_in[b][k], nullptr));
      cudaFreeHost(std::exchange(c.pin_out[b], nullptr));
      cudaFreeHost(std::exchange(c.pin_st[b], nullptr));
    }
    c.cap_pin = c.cap_pin_st = 0;
    for (int b = 0; b < kPipeSlots; ++b) {
      const int64_t cnt = chunk * std::max(n, width);
      for (int k = 0; k < 3; ++k)
        if ((e = cudaMallocHost(&c.pin_in[b][k], sizeof(double) * cnt)) != cudaSuccess) return cuda_fail(e, "pinned");
      if ((e = cudaMallocHost(&c.pin_out[b], sizeof(double) * cnt)) != cudaSuccess) return cuda_fail(e, "pinned");
      if ((e = cudaMallocHost(&c.pin_st[b], sizeof(int32_t) * chunk)) != cudaSuccess) return cuda_fail(e, "pinned");
    }
    c.cap_pin = chunk * std::max(n, width);
    c.cap_pin_st = chunk;
  }
  return VD_OK;
}

// Bytes of input + output per pipeline chunk (internal knob for
// tools/e2e_chunk.py; vdi_set_host_chunk_bytes).
// 96 MB: Panda 4M states 14.7 ms at 48 MB, 14.4 ms at 96 MB, 14.6 at 192 MB
// (pinned buffers; the same box copies the bytes in 13.2 ms).
constexpr int64_t kChunkBytesDefault = 96ll << 20;
std::atomic<int64_t> g_chunk_bytes{kChunkBytesDefault};

// Stream one device's shard [b, e) through the double-buffered pipeline.
int run_shard(DevCtx& c, vd_model m, const HostOp& op, int64_t N, int64_t b, int64_t e, const double* const* inputs,
              const double* g3, double* out, int32_t* status, bool* any_bad) {
  const int n = m->m.dof();
  const int width = op.out_width;
  const int64_t len = e - b;
  int64_t chunk = std::min<int64_t>(len, std::max<int64_t>(65536, g_chunk_bytes.load() / (8ll * (n * op.n_in + width))));
  chunk = (chunk + 127) / 128 * 128;  // device leading dimension: a multiple of the kernels' tile
  bool pinned = is_pinned(out);
  for (int k = 0; k < op.n_in; ++k) pinned = pinned && is_pinned(inputs[k]);
  const bool st_direct = pinned && status && is_pinned(status);
  if (int rc = prepare_ctx(c, m, n, chunk, width, !pinned || (op.kind == 2 && !st_direct))) return rc;
  // Chunk plan: full chunks, then a geometric taper (halving down to 16 K
  // states) over the last two chunks' worth, so the kernel + D2H that drain
  // after the last H2D move a small chunk, not a full one.
  std::vector<std::pair<int64_t, int64_t>> plan;
  for (int64_t lo = b; lo < e;) {
    const int64_t rem = e - lo;
    int64_t cl = chunk;
    if (rem <= 2 * chunk) cl = std::max<int64_t>(16384, ((rem + 1) / 2 + 127) / 128 * 128);
    cl = std::min(cl, rem);
    plan.emplace_back(lo, cl);
    lo += cl;
  }
  const int64_t nchunks = (int64_t)plan.size();
  std::vector<int32_t> st_host;
  int32_t* st_dst = status;
  if (op.kind == 2 && !status) {
    st_host.resize((size_t)len);
    st_dst = st_host.data() - b;  // indexed with the global row below
  }
  const int nslots = kPipeSlots;
  std::vector<int64_t> pending_lo(kPipeSlots, -1), pending_len(kPipeSlots, 0);
  auto finish_slot = [&](int slot) -> int {
    if (pending_lo[(size_t)slot] < 0) return VD_OK;
    cudaError_t ce = cudaEventSynchronize(c.done[slot]);
    if (ce != cudaSuccess) return cuda_fail(ce, "host batch");
    const int64_t lo = pending_lo[(size_t)slot], cl = pending_len[(size_t)slot];
    if (!pinned) {  // unstage
      for (int r = 0; r < width; ++r)
        std::memcpy(out + (int64_t)r * N + lo, c.pin_out[slot] + (int64_t)r * cl, sizeof(double) * cl);
    }
    if (op.kind == 2 && !st_direct) std::memcpy(st_dst + lo, c.pin_st[slot], sizeof(int32_t) * cl);
    if (op.kind == 2)
      for (int64_t k = 0; k < cl; ++k)
        if (st_dst[lo + k]) *any_bad = true;
    pending_lo[(size_t)slot] = -1;
    return VD_OK;
  };
  for (int64_t k = 0; k < nchunks; ++k) {
    const int slot = (int)(k % nslots);
    if (int rc = finish_slot(slot)) return rc;
    const int64_t lo = plan[(size_t)k].first, cl = plan[(size_t)k].second;
    cudaStream_t s = c.st[slot];
    cudaError_t ce = cudaSuccess;
    for (int i = 0; i < op.n_in && ce == cudaSuccess; ++i) {
      const double* src = inputs[i] + lo;
      size_t spitch = sizeof(double) * N;
      if (!pinned) {
        for (int r = 0; r < n; ++r)
          std::memcpy(c.pin_in[slot][i] + (int64_t)r * cl, inputs[i] + (int64_t)r * N + lo, sizeof(double) * cl);
        src = c.pin_in[slot][i];
        spitch = sizeof(double) * cl;
      }
      ce = cudaMemcpy2DAsync(c.din[slot][i], sizeof(double) * chunk, src, spitch, sizeof(double) * cl, n,
                             cudaMemcpyHostToDevice, s);
    }
    if (ce != cudaSuccess) return cuda_fail(ce, "host batch H2D");
    int rc;
    if (op.kind == 0)
      rc = vd_rnea(c.dm, VD_F64, cl, c.din[slot][0], c.din[slot][1], c.din[slot][2], chunk, g3, nullptr, c.dout[slot],
                   chunk, s);
    else if (op.kind == 1)
      rc = vd_crba(c.dm, VD_F64, cl, c.din[slot][0], chunk, c.dout[slot], chunk, s);
    else
      rc = vd_aba(c.dm, VD_F64, cl, c.din[slot][0], c.din[slot][1], c.din[slot][2], chunk, g3, nullptr, c.dout[slot],
                  chunk, c.dst[slot], s);
    if (rc) return rc;
    double* dst = pinned ? out + lo : c.pin_out[slot];
    const size_t dpitch = pinned ? sizeof(double) * N : sizeof(double) * cl;
    ce = cudaMemcpy2DAsync(dst, dpitch, c.dout[slot], sizeof(double) * chunk, sizeof(double) * cl, width,
                           cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess && op.kind == 2)
      ce = cudaMemcpyAsync(st_direct ? st_dst + lo : c.pin_st[slot], c.dst[slot], sizeof(int32_t) * cl,
                           cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaEventRecord(c.done[slot], s);
    if (ce != cudaSuccess) return cuda_fail(ce, "host batch D2H");
    pending_lo[(size_t)slot] = lo;
    pending_len[(size_t)slot] = cl;
  }
  // drain in issue order
  for (int64_t k = std::max<int64_t>(0, nchunks - nslots); k < nchunks; ++k)
    if (int rc = finish_slot((int)(k % nslots))) return rc;
  return VD_OK;
}

int host_batch(vd_model m, const HostOp& op, int64_t N, const double* const* inputs, const double* g3, double* out,
               int32_t* status, const int* devices, int ndev) {
  if (!m) return set_error(VD_ERR_INVALID_ARGUMENT, "null model");
  if (N < 0) return set_error(VD_ERR_DIMENSION, "negative batch size");
  const int n = m->m.dof();
  if (N == 0 || n == 0) return VD_OK;
  for (int k = 0; k < op.n_in; ++k)
    if (!inputs[k]) return set_error(VD_ERR_INVALID_ARGUMENT, "null input buffer");
  if (!out) return set_error(VD_ERR_INVALID_ARGUMENT, "null output buffer");
  std::vector<int> devs;
  if (devices && ndev > 0) devs.assign(devices, devices + ndev);
  else devs.push_back(0);
  const int W = (int)devs.size();
  std::vector<int> rcs((size_t)W, VD_OK);
  std::vector<std::string> msgs((size_t)W);
  std::vector<char> bad((size_t)W, 0);
  auto work = [&](int w) {
    int64_t b = 0, e = 0;
    vd_shard_range(N, W, w, &b, &e);
    if (e <= b) return;
    DevCtx& c = ctx_for(devs[(size_t)w]);
    std::lock_guard<std::mutex> lk(c.mu);
    DeviceGuard g(devs[(size_t)w]);
    bool any_bad = false;
    int rc = VD_OK;
    try {
      rc = run_shard(c, m, op, N, b, e, inputs, g3, out, status, &any_bad);
    } catch (const std::exception& ex) {
      rc = set_error(VD_ERR_GENERIC, ex.what());
    }
    if (rc) {
      rcs[(size_t)w] = rc;
      msgs[(size_t)w] = g_msg;
    }
    bad[(size_t)w] = any_bad ? 1 : 0;
  };
  if (W == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int w = 0; w < W; ++w) pool.emplace_back(work, w);
    for (auto& t : pool) t.join();
  }
  for (int w = 0; w < W; ++w)
    if (rcs[(size_t)w]) return set_error(rcs[(size_t)w], msgs[(size_t)w]);
  for (int w = 0; w < W; ++w)
    if (bad[(size_t)w])
      return set_error(VD_ERR_SINGULAR_INERTIA,
                       "forward_dynamics: mass matrix is not positive definite (zero-inertia degree of freedom?)");
  return VD_OK;
}
}  // namespace

int vd_batch_rnea_host(vd_model m, int64_t N, const double* q, const double* qd, const double* qdd, const double* g3,
                       double* tau, const int* devices, int n_devices) {
  const double* in[3] = {q, qd, qdd};
  return host_batch(m, HostOp{0, 3, m ? m->m.dof() : 0}, N, in, g3, tau, nullptr, devices, n_devices);
}
int vd_batch_crba_host(vd_model m, int64_t N, const double* q, double* M, const int* devices, int n_devices) {
  const double* in[1] = {q};
  const int n = m ? m->m.dof() : 0;
  return host_batch(m, HostOp{1, 1, n * n}, N, in, nullptr, M, nullptr, devices, n_devices);
}
int vd_batch_forward_dynamics_host(vd_model m, int64_t N, const double* q, const double* qd, const double* tau,
                                   const double* g3, double* qdd, int32_t* status, const int* devices, int n_devices) {
  const double* in[3] = {q, qd, tau};
  return host_batch(m, HostOp{2, 3, m ? m->m.dof() : 0}, N, in, g3, qdd, status, devices, n_devices);
}

// ---- internal (not in the public header): host-pipeline chunk size (bytes
// of inputs + outputs per chunk; <= 0 restores the default)
void vdi_set_host_chunk_bytes(int64_t bytes) { g_chunk_bytes.store(bytes > 0 ? bytes : kChunkBytesDefault); }

}  // extern "C"
