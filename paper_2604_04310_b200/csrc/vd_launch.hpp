// Internal launch interface between the C-ABI layer (vd_abi.cpp) and the
// kernels (vd_kernels.cu).  Not part of the public boundary.
#pragma once

#include <cstddef>
#include <cstdint>

namespace vdk {


// Stream-ordered scratch from a private per-device pool (vd_dispatch.cu).
// The pool keeps up to kScratchKeepBytes cached across synchronisations so a
// per-launch slab is not a real allocation every time; it never touches the
// device's default pool, whose release policy belongs to the application.
constexpr uint64_t kScratchKeepBytes = 512ull << 20;
int scratch_alloc(void** p, size_t bytes, void* stream);
void scratch_free(void* p, void* stream);

// Which compile-time robot a device model matched (0 = generic kernels).
enum Spec : int { kGeneric = 0, kChain7 = 1, kTree29 = 2, kHumanoid23 = 3 };

struct Launch;
// Per-model JIT modules (paper_2604_04310_b200/jit.py, vd_jit_entry.cuh):
// generated routines of a model without compile-time kernels, loaded at run
// time.  One entry point; returns -1 when the module has no routine for op.
enum JitOp : int {
  kJitAba = 0, kJitRnea = 1, kJitBias = 2, kJitGravity = 3, kJitCoriolis = 4, kJitCrba = 5, kJitCrbaPacked = 6,
  kJitFk = 7
};
constexpr int kJitAbi = 3;  // 2: Launch::gravity_planes; 3: task routine 4 (manipulability JVP)
using JitLaunchFn = int (*)(int op, const Launch* L, const void* x0, const void* x1, const void* x2,
                            const double* g3, const void* fext, void* y, int32_t* status);
// which: 0 Jacobian, 1 diff-IK, 2 manipulability (params TaskShared*), 3 OSC (params OscShared*),
// 4 manipulability JVP (qd = the tangent dq; y0 w, y1 dw)
using JitTaskFn = int (*)(int which, const Launch* L, int frame_joint, const void* q, const void* qd,
                          const void* params, void* y0, void* y1, int32_t* status);

struct Launch {
  int spec;                 // Spec
  int dtype;                // 0 f64, 1 f32
  int n;                    // dof
  const void* model;        // host DevModel<T>* (matching dtype), passed by value to the kernels
  int64_t N, ld_in, ld_out;
  void* stream;
  bool serial = false;      // every joint's parent is its predecessor
  JitLaunchFn jit = nullptr;  // the model's JIT module, if one is attached
  JitTaskFn jit_task = nullptr;  // its task-space routines, for the frame joints in jit_task_mask
  uint64_t jit_task_mask = 0;
  // Per-state gravity (vd_*_pg): 3 planes of a_g (= −field) with leading
  // dimension ld_in, in the call's dtype; NULL = the call's gravity3.  Read by
  // the RNEA (full / bias / gravity vector) and ABA kernels only.
  const void* gravity_planes = nullptr;
};

struct OscShared;
struct TaskShared;

// Compile-time robot whose packed-model fingerprint matches (0 = none).
int match_spec(uint64_t fingerprint, int n);

// All return cudaError_t as int.
int launch_fk(const Launch& L, const void* q, void* out);
// forward_kinematics_scan (serial chains, n <= 32)
int launch_fk_scan(const Launch& L, const void* q, void* out);
int launch_jacobian(const Launch& L, const void* q, int frame_joint, const double* frame_R, const double* frame_p,
                    void* pose, void* J);
// mode: 0 full rnea, 1 bias (qdd = 0), 2 gravity (qd = qdd = 0), 3 coriolis (qdd = 0, g = 0)
int launch_rnea(const Launch& L, int mode, const void* q, const void* qd, const void* qdd, const double* g3,
                const void* fext, void* tau);
int launch_crba(const Launch& L, const void* q, void* M);
// Branch-sparse lower triangle of M (vd_model_crba_pattern order): plane k of
// the output is dense plane src[k] (= c·n + r) of M.  At most 64·65/2 pairs.
struct PackTable {
  int nnz;
  uint16_t src[2080];
};
int launch_crba_packed(const Launch& L, const void* q, void* Mp, const PackTable& tab);
int launch_aba(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, const void* fext,
               void* qdd, int32_t* status);
// Generated straight-line kernel (vd_inst_gen.cu) when one exists for L.spec;
// -1 when not applicable.
int launch_gen_aba(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3,
                   const void* fext, void* qdd, int32_t* status);
int launch_gen_rnea(const Launch& L, int mode, const void* q, const void* qd, const void* qdd, const double* g3,
                    const void* fext, void* tau);
int launch_gen_crba(const Launch& L, const void* q, void* M);
int launch_gen_crba_packed(const Launch& L, const void* q, void* Mp);
int launch_gen_fk(const Launch& L, const void* q, void* frames);
// which: 0 Jacobian, 1 diff-IK, 2 manipulability, 4 manipulability JVP along dq (y0 w, y1 dw)
int launch_gen_task(const Launch& L, int which, int frame_joint, const TaskShared& P, const void* q, void* y0,
                    void* y1, int32_t* status, const void* dq = nullptr);
// generated fused M + bias + q̈ (chain7, fp64 and fp32); -1 when not applicable
int launch_gen_dyn(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* M,
                   void* bias, void* qdd, int32_t* status);
int launch_gen_osc(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lambda,
                   int32_t* status);
int launch_dynamics(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* M,
                    void* bias, void* qdd, int32_t* status);
int launch_osc(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lambda,
               int32_t* status);
// Forward-mode JVPs (vd_jvp.cuh): one launch of FK / RNEA / CRBA / ABA on dual numbers.
enum JvpOp : int { kJvpFK = 0, kJvpRNEA = 1, kJvpCRBA = 2, kJvpABA = 3 };
struct JvpArgs {
  int op;             // JvpOp
  const void* x[3];   // primal inputs (q, q̇, q̈ | τ)
  const void* dx[3];  // tangents (NULL = 0)
  double g[3];        // gravity a_g (rnea / aba), by value
  const void* fext;   // constant external wrenches (rnea / aba), NULL = none
  void* out;          // values (may be NULL)
  void* dout;         // tangents (may be NULL)
  int32_t* status;    // aba
};
int launch_jvp(const Launch& L, const JvpArgs& a);
// generated dual-number kernels (tree29 ABA / RNEA without f_ext); -1 otherwise
int launch_gen_jvp(const Launch& L, const JvpArgs& a);
// manipulability and its JVP along dq (vd_jvp.cuh k_manip_jvp); w / dw one plane each
int launch_manip_jvp(const Launch& L, const void* q, const void* dq, const TaskShared& P, void* w, void* dw);

// Row-major (N, K) batch <-> K planes (vd_layout.cu); to_planes: rows -> planes.
int launch_layout(int dtype, bool to_planes, int64_t N, int K, const void* src, int64_t ld_src, void* dst,
                  int64_t ld_dst, void* stream);

// mode 0: diff_ik_step (out = q̇, aux = pose error); mode 1: manipulability (out = w)
int launch_task(const Launch& L, const void* q, const TaskShared& P, int mode, void* out, void* aux,
                int32_t* status);

}  // namespace vdk
