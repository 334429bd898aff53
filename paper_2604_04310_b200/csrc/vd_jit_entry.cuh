// C entry points of a per-model JIT module.  Included last by the translation
// unit paper_2604_04310_b200/jit.py generates for one robot model (after its
// generated routines, struct VD_JIT_ROBOT); the library dlopen()s the module
// (vd_model_attach_jit) and calls vdj_launch from the dispatch of the ops the
// module carries (vd_dispatch.cu).  Built with -fvisibility=hidden: only the
// vdj_* symbols are exported, so the module's copies of the launch machinery
// never interpose on the library's.
#pragma once

#include "vd_gen_launch.cuh"

#ifndef VD_JIT_ROBOT
#error "define VD_JIT_ROBOT (the generated robot struct) before including vd_jit_entry.cuh"
#endif

typedef int (*vdj_alloc_fn)(void** p, size_t bytes, void* stream);
typedef void (*vdj_free_fn)(void* p, void* stream);

namespace vdk {
namespace {
vdj_alloc_fn g_jit_alloc = nullptr;
vdj_free_fn g_jit_free = nullptr;
}  // namespace
// the library's private scratch pool, handed over by vdj_init
int scratch_alloc(void** p, size_t bytes, void* stream) { return g_jit_alloc(p, bytes, stream); }
void scratch_free(void* p, void* stream) {
  if (p) g_jit_free(p, stream);
}
}  // namespace vdk

#define VD_JIT_API extern "C" __attribute__((visibility("default")))

VD_JIT_API int vdj_abi_version(void) { return vdk::kJitAbi; }
VD_JIT_API uint64_t vdj_fingerprint(void) { return VD_JIT_ROBOT::kFingerprint; }
VD_JIT_API int vdj_dof(void) { return VD_JIT_ROBOT::kN; }
VD_JIT_API void vdj_init(vdj_alloc_fn a, vdj_free_fn f) {
  vdk::g_jit_alloc = a;
  vdk::g_jit_free = f;
}

// Same operand conventions as the library's generated dispatch
// (vd_inst_gen.cu): x0 = q, x1 = q̇, x2 = q̈ | τ; fext NULL or 6n planes;
// fp32 forward dynamics runs the mixed-precision routine.
VD_JIT_API int vdj_launch(int op, const vdk::Launch* L, const void* x0, const void* x1, const void* x2,
                          const double* g3, const void* fext, void* y, int32_t* status) {
  using R = VD_JIT_ROBOT;
  using namespace vdk;
  static const double zero3[3] = {0, 0, 0};
  const bool f64 = L->dtype == 0;
  switch (op) {
    case kJitAba:
      if (fext)
        return f64 ? launch_t<R::AbaFext, double>(*L, x0, x1, x2, g3, y, status, fext)
                   : launch_t<R::AbaMixedFext, float>(*L, x0, x1, x2, g3, y, status, fext);
      return f64 ? launch_t<R::Aba, double>(*L, x0, x1, x2, g3, y, status)
                 : launch_t<R::AbaMixed, float>(*L, x0, x1, x2, g3, y, status);
    case kJitRnea:
      if (!x1 || !x2) return -1;
      return fext ? launch_op<R::RneaFext>(*L, x0, x1, x2, g3, y, nullptr, fext)
                  : launch_op<R::Rnea>(*L, x0, x1, x2, g3, y, nullptr);
    case kJitBias:
      if (!x1) return -1;
      return fext ? launch_op<R::RneaBiasFext>(*L, x0, x1, nullptr, g3, y, nullptr, fext)
                  : launch_op<R::RneaBias>(*L, x0, x1, nullptr, g3, y, nullptr);
    case kJitGravity:
      return fext ? -1 : launch_op<R::RneaGrav>(*L, x0, nullptr, nullptr, g3, y, nullptr);
    case kJitCoriolis:
      if (!x1 || fext) return -1;
      return launch_op<R::RneaBias>(*L, x0, x1, nullptr, zero3, y, nullptr);
    case kJitCrba:
      return launch_op<R::Crba>(*L, x0, nullptr, nullptr, nullptr, y, nullptr);
    case kJitCrbaPacked:
      return launch_op<R::CrbaPacked>(*L, x0, nullptr, nullptr, nullptr, y, nullptr);
    case kJitFk:
      return launch_op<R::Fk>(*L, x0, nullptr, nullptr, nullptr, y, nullptr);
    default:
      return -1;
  }
}

#ifdef VD_JIT_TASKS
// Task-space routines on the frame joints the module was generated for:
// bit j of the mask = joint j has OSC, Jacobian, diff-IK and manipulability.
VD_JIT_API uint64_t vdj_task_mask(void) {
  uint64_t m = 0;
  for (int j : VD_JIT_ROBOT::kOscJoints) m |= 1ull << j;
  return m;
}
// which: 0 Jacobian (y0 pose, y1 J), 1 diff-IK (y0 q̇, y1 err), 2 manipulability
// (y0 w), 4 manipulability JVP along qd (y0 w, y1 dw); params =
// vdk::TaskShared.  3: OSC (y0 τ, y1 Λ), params =
// vdk::OscShared.  Same conventions as vd_inst_gen.cu's gen_task_t / gen_osc_t.
VD_JIT_API int vdj_task_launch(int which, const vdk::Launch* L, int frame_joint, const void* q, const void* qd,
                               const void* params, void* y0, void* y1, int32_t* status) {
  using R = VD_JIT_ROBOT;
  using namespace vdk;
  int rc = -1;
  const bool f64 = L->dtype == 0;
  if (which == 3) {
    const OscShared& P = *static_cast<const OscShared*>(params);
    R::with_osc(frame_joint, [&](auto op) {
      using Op = decltype(op);
      rc = f64 ? launch_osc_t<Op, double>(*L, q, qd, P, y0, y1, status)
               : launch_osc_t<Op, float>(*L, q, qd, P, y0, y1, status);
    });
    return rc;
  }
  const TaskShared& P = *static_cast<const TaskShared*>(params);
  const void* dq = which == 4 ? qd : nullptr;
  R::with_task(frame_joint, [&](auto jac, auto dik, auto man, auto man_jvp) {
    auto go = [&](auto op) {
      using Op = decltype(op);
      rc = f64 ? launch_task_t<Op, double>(*L, q, P, y0, y1, status, dq)
               : launch_task_t<Op, float>(*L, q, P, y0, y1, status, dq);
    };
    if (which == 0) go(jac);
    else if (which == 1) go(dik);
    else if (which == 2) go(man);
    else if (which == 4) go(man_jvp);
  });
  return rc;
}
#endif
