/*
 * vecdyn_cuda.h — C-ABI of the B200-native batched rigid-body dynamics library.
 *
 * Drop-in boundary for the reference `vecdyn` hot path (a C++20/Eigen header
 * library, proj/core/include/vecdyn/).  The reference has no FFI; its
 * "operator API" is the C++ signatures cited on every entry point below.
 * These functions replace them one for one with plain pointers and sizes:
 *
 *   - models are opaque handles (the reference returns RobotModel by value,
 *     model.hpp:90-149);
 *   - batched buffers are DEVICE pointers in SoA column-major layout: element
 *     (instance i, component k) lives at  k * ld + i  (ld >= N).  This is the
 *     memory layout of Eigen's column-major N x K matrices used by StateBatch
 *     and batch_crba (batch.hpp:15-19, 147-148), so an Eigen caller can pass
 *     .data() unchanged;
 *   - dtype selects fp64 (the reference default, T = double) or fp32 (the
 *     reference's float instantiation, test_dynamics.cpp:398-413) for every
 *     floating buffer of the call;
 *   - errors are int status codes (VD_ERR_*) mirroring the reference exception
 *     hierarchy (errors.hpp:9-61) plus vd_last_error() (thread-local text);
 *     forward dynamics and OSC additionally report a per-instance status
 *     (the reference throws SingularInertiaError for the whole call,
 *     dynamics.hpp:437-442, control.hpp:131-134).
 *
 * Every kernel entry point is asynchronous on `stream` (a cudaStream_t passed
 * as void*, NULL = legacy default stream) and never allocates.
 */
#ifndef VECDYN_CUDA_H_
#define VECDYN_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VD_OK 0
#define VD_ERR_DIMENSION 1              /* DimensionError            errors.hpp:14-18 */
#define VD_ERR_PARSE 2                  /* ParseError(line, column)  errors.hpp:32-43 */
#define VD_ERR_MODEL 3                  /* ModelError                errors.hpp:20-24 */
#define VD_ERR_UNKNOWN_FRAME 4          /* UnknownFrameError         errors.hpp:26-30 */
#define VD_ERR_UNSUPPORTED_FEATURE 5    /* UnsupportedFeatureError   errors.hpp:45-49 */
#define VD_ERR_UNSUPPORTED_STRUCTURE 6  /* UnsupportedStructureError errors.hpp:51-55 */
#define VD_ERR_SINGULAR_INERTIA 7       /* SingularInertiaError      errors.hpp:57-61 */
#define VD_ERR_CUDA 8                   /* CUDA runtime failure (no reference analogue) */
#define VD_ERR_INVALID_ARGUMENT 9       /* null pointer, ld < N, bad dtype, ... */
#define VD_ERR_IO 10                    /* Error("cannot open URDF file ...") urdf.cpp:277-281 */
#define VD_ERR_GENERIC 11               /* vecdyn::Error */

#define VD_F64 0
#define VD_F32 1

/* per-instance status values written by vd_aba / vd_dynamics / vd_osc */
#define VD_STATUS_OK 0
#define VD_STATUS_SINGULAR 7 /* non-positive articulated pivot / mass-matrix pivot, or non-finite */

typedef struct vd_model_s* vd_model;
typedef struct vd_device_model_s* vd_device_model;

/* ------------------------------------------------------------------ errors */
const char* vd_last_error(void);
int vd_last_error_line(void);   /* ParseError::line (1-based), 0 otherwise */
int vd_last_error_column(void); /* ParseError::column */
const char* vd_version(void);

/* ------------------------------------------------------------------ host model */
/* robots::chain7 / humanoid23 / tree29 / by_name            robots.cpp:12-32 */
int vd_model_builtin(const char* name, vd_model* out);
/* urdf::load_model(path)                                     urdf.cpp:384-386 */
int vd_model_load_urdf(const char* path, vd_model* out);
/* urdf::load_model_from_string(text)                         urdf.cpp:388-390 */
int vd_model_load_urdf_string(const char* text, size_t len, vd_model* out);
/* floating_base(model)                                       model.cpp:289-331 */
int vd_model_floating_base(vd_model m, vd_model* out);
void vd_model_destroy(vd_model m);

/* RobotModel accessors                                       model.hpp:92-133 */
int vd_model_dof(vd_model m);
int vd_model_max_depth(vd_model m);
int vd_model_is_serial_chain(vd_model m);
double vd_model_total_mass(vd_model m);
int vd_model_warning_count(vd_model m);
int vd_model_warning(vd_model m, int k, char* buf, size_t len);
int vd_model_name(vd_model m, char* buf, size_t len);
int vd_model_parents(vd_model m, int* parents_out); /* n ints */
int vd_model_joint_name(vd_model m, int i, char* buf, size_t len);
int vd_model_joint_index(vd_model m, const char* name); /* -1 if absent (model.cpp:337-343) */
/* type: 0 revolute, 1 prismatic; offset: R column-major (9) then p (3);
 * inertia: 6x6 row-major about the joint frame origin, angular first. */
int vd_model_joint(vd_model m, int i, int* type, double axis[3], double offset[12], double inertia[36]);
int vd_model_ancestor_mask(vd_model m, double* mask_out); /* n*n, column-major (Eigen MatrixXd) */
/* Branch-sparse lower triangle of M (the reference's M_lower = U ⊙ (SᵀCS),
 * dynamics.hpp:337-350; every other entry is an exact zero,
 * test_dynamics.cpp:200-216): the pairs (r, c), r >= c, c an ancestor of r or
 * r itself, in compressed-column order (c ascending, then r).  *nnz_out
 * receives the count (chain7 28, tree29 242); rows / cols may be NULL. */
int vd_model_crba_pattern(vd_model m, int32_t* rows_out, int32_t* cols_out, int* nnz_out);
int vd_model_frame_count(vd_model m);
int vd_model_frame(vd_model m, int k, char* name, size_t len, int* joint, double offset[12]);
/* RobotModel::frame(name) index; VD_ERR_UNKNOWN_FRAME when absent (model.cpp:337-343) */
int vd_model_frame_index(vd_model m, const char* name, int* out);

/* StateBatch random_states(model, count, seed, with_qdd, with_tau), batch.hpp:48-75:
 * HOST column-major N x n arrays; qdd / tau may be NULL (with_qdd / with_tau
 * false).  Bit-identical to the reference's mt19937_64 + U[-π, π] stream. */
int vd_random_states(vd_model m, int64_t N, uint64_t seed, double* q, double* qd, double* qdd, double* tau);

/* ------------------------------------------------------------------ device model */
/* Packs the model for `device` (the reference has no device; the model is
 * uploaded once here and reused by every call).  When the model matches a
 * robot compiled into the library (chain7, tree29, humanoid23) the
 * compile-time specialised kernels are used, otherwise the generic
 * runtime-topology kernels (any tree with n <= 64). */
int vd_device_model_create(vd_model m, int device, vd_device_model* out);
void vd_device_model_destroy(vd_device_model dm);
int vd_device_model_dof(vd_device_model dm);
/* 0 = generic kernels, k > 0 = compile-time specialised robot k */
int vd_device_model_specialization(vd_device_model dm);
/* Force the generic kernels even for builtin robots (testing / comparison). */
int vd_device_model_set_generic(vd_device_model dm, int generic);
/* Per-model JIT module (no reference analogue: the reference has no device
 * code).  A model that is not one of the compile-time robots runs the loop
 * kernels unless a module of its generated straight-line routines (ABA, RNEA,
 * bias, gravity, Coriolis, CRBA, packed CRBA, FK; built by
 * paper_2604_04310_b200/jit.py, `python -m paper_2604_04310_b200.jit model.urdf`)
 * is attached: device models created from m afterwards use it.  Fails with
 * VD_ERR_INVALID_ARGUMENT if the module was generated for a different model. */
int vd_model_attach_jit(vd_model m, const char* module_path);
/* 1 if calls on dm run a JIT module, 0 if not, -1 for a null handle */
int vd_device_model_jit(vd_device_model dm);

/* ------------------------------------------------------------------ batched kernels
 * gravity3: the base acceleration a_g = −field (GravitySpec::accel.linear,
 * dynamics.hpp:35-50); NULL means GravitySpec::standard() = (0, 0, +9.81).
 * fext: NULL or 6n planes, plane j*6 + k = component k (angular first) of
 * the world-frame Plücker wrench on joint j (ExternalForcesT, dynamics.hpp:52-81). */

/* forward_kinematics, kinematics.hpp:43-56: plane j*12 + k (k < 9: R column-major, 9..11: p) */
int vd_fk(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* frames_out,
          int64_t ld_out, void* stream);
/* forward_kinematics_scan, kinematics.hpp:61-86: same output as vd_fk by a
 * Hillis–Steele scan (one lane segment per state); serial chains with n <= 32,
 * VD_ERR_UNSUPPORTED_STRUCTURE otherwise (kinematics.hpp:63-67). */
int vd_fk_scan(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* frames_out,
               int64_t ld_out, void* stream);
/* frame_transform + geometric_jacobian, kinematics.hpp:89-136: pose 12 planes,
 * J 6 x n column-major (plane c*6 + r).  Either output may be NULL. */
int vd_jacobian(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, int frame, void* pose_out,
                void* J_out, int64_t ld_out, void* stream);
/* rnea(model, q, qd, qdd, gravity, fext), dynamics.hpp:250-267 */
int vd_rnea(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* qdd, int64_t ld_in,
            const double* gravity3, const void* fext, void* tau_out, int64_t ld_out, void* stream);
/* c + g (− Σ Jᵀ f_ext): rnea(q, qd, 0, gravity, fext), dynamics.hpp:434-435 */
int vd_bias(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in,
            const double* gravity3, const void* fext, void* out, int64_t ld_out, void* stream);
/* gravity_vector, dynamics.hpp:402-408 */
int vd_gravity(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, const double* gravity3,
               void* out, int64_t ld_out, void* stream);
/* coriolis_vector, dynamics.hpp:410-416 */
int vd_coriolis(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in, void* out,
                int64_t ld_out, void* stream);
/* crba, dynamics.hpp:352-365: M n x n column-major, plane c*n + r */
int vd_crba(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* M_out, int64_t ld_out,
            void* stream);
/* crba in packed form (no reference analogue; the reference returns dense M,
 * dynamics.hpp:352-365): plane k = M(rows[k], cols[k]) of vd_model_crba_pattern.
 * Output planes 242 instead of 841 for tree29 (the dense output is HBM-bound). */
int vd_crba_packed(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, void* M_packed_out,
                   int64_t ld_out, void* stream);
/* forward_dynamics, dynamics.hpp:418-444, computed by the articulated-body
 * algorithm (absent from the reference).  status_out (int32 x N)
 * may be NULL. */
int vd_aba(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau, int64_t ld_in,
           const double* gravity3, const void* fext, void* qdd_out, int64_t ld_out, int32_t* status_out,
           void* stream);
/* Fused M + bias + q̈ (BASELINE config 3) sharing one FK; any output may be NULL. */
int vd_dynamics(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
                int64_t ld_in, const double* gravity3, void* M_out, void* bias_out, void* qdd_out, int64_t ld_out,
                int32_t* status_out, void* stream);

/* Per-state gravity (no reference analogue: GravitySpec is one
 * per call, dynamics.hpp:35-50).  The same calls as vd_rnea / vd_bias /
 * vd_gravity / vd_aba / vd_dynamics, with state i's base acceleration a_g read
 * from gravity_planes: 3 planes (x, y, z of a_g = −field) of dtype elements
 * with leading dimension ld_in.  Results equal the per-call entry point run on
 * state i alone with gravity3 = (its a_g). */
int vd_rnea_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* qdd,
               int64_t ld_in, const void* gravity_planes, const void* fext, void* tau_out, int64_t ld_out,
               void* stream);
int vd_bias_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in,
               const void* gravity_planes, const void* fext, void* out, int64_t ld_out, void* stream);
int vd_gravity_pg(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, const void* gravity_planes,
                  void* out, int64_t ld_out, void* stream);
int vd_aba_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau, int64_t ld_in,
              const void* gravity_planes, const void* fext, void* qdd_out, int64_t ld_out, int32_t* status_out,
              void* stream);
int vd_dynamics_pg(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
                   int64_t ld_in, const void* gravity_planes, void* M_out, void* bias_out, void* qdd_out,
                   int64_t ld_out, int32_t* status_out, void* stream);

/* osc_step, control.hpp:108-155.  Shared task / posture parameters. */
typedef struct vd_osc_params {
  int frame;              /* vd_model_frame_index */
  double target[12];      /* TaskTarget::pose, R column-major + p */
  double kp[6], kd[6];    /* TaskGains (angular first) */
  double accel_ff[6];     /* TaskTarget::accel_ff */
  const double* posture;  /* HOST pointer, n values */
  double posture_kp, posture_kd;
  double gravity[3];      /* a_g */
  double epsilon;         /* Λ regulariser (reference default 1e-6) */
} vd_osc_params;
/* tau n planes; Lambda_out (36 planes, column-major (J M⁻¹ Jᵀ + εI)⁻¹) may be NULL. */
int vd_osc(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, int64_t ld_in,
           const vd_osc_params* params, void* tau_out, void* Lambda_out, int64_t ld_out, int32_t* status_out,
           void* stream);

/* diff_ik_step, control.hpp:79-97: q̇ = Jᵀ (J Jᵀ + λ² I)⁻¹ (kp ⊙ err + twist_ff).
 * damping must be > 0 and gains nonnegative (control.hpp:82-86, 32-36). */
typedef struct vd_task_params {
  int frame;           /* vd_model_frame_index */
  double target[12];   /* TaskTarget::pose, R column-major + p */
  double kp[6];        /* TaskGains::kp (angular first) */
  double twist_ff[6];  /* TaskTarget::twist_ff */
  double damping;      /* λ */
} vd_task_params;
/* qdot_out n planes; err_out (6 planes, pose_error, control.hpp:73-77) may be NULL. */
int vd_diff_ik(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, const vd_task_params* params,
               void* qdot_out, void* err_out, int64_t ld_out, int32_t* status_out, void* stream);
/* manipulability(geometric_jacobian(frame)), kinematics.hpp:138-153: one plane,
 * sqrt(det(J Jᵀ)) as a Cholesky pivot product, 0 where the factorization fails. */
int vd_manipulability(vd_device_model dm, int dtype, int64_t N, const void* q, int64_t ld_in, int frame,
                      void* w_out, void* stream);
/* manipulability and its directional derivative D w(q)·dq (jvp_scalar of
 * kinematics.hpp:138-153 on dual.hpp scalars; autodiff.hpp:52-62): one plane
 * each, either may be NULL; dq NULL = zero tangent.  With dq = q̇ this is the
 * Lie derivative L_f w along the drift f = (q̇, q̈) (control.hpp:157-163). */
int vd_manipulability_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* dq, int64_t ld_in,
                          int frame, void* w_out, void* dw_out, void* stream);

/* ------------------------------------------------------------------ forward-mode JVPs
 * jvp(fn, x, v) of autodiff.hpp:41-52 applied to the library's own functions
 * (the reference runs them on the Dual scalar of dual.hpp:14-196): one pass on
 * dual numbers returns fn(x) and D fn(x)·v.  Tangent inputs (dq, dqd, ...) may
 * be NULL (zero tangent); value or tangent outputs may be NULL (not both).
 * Output layouts are those of the primal functions.  fext is a constant
 * (zero-tangent) input. */
int vd_fk_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* dq, int64_t ld_in,
              void* frames_out, void* dframes_out, int64_t ld_out, void* stream);
int vd_rnea_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* qdd,
                const void* dq, const void* dqd, const void* dqdd, int64_t ld_in, const double* gravity3,
                const void* fext, void* tau_out, void* dtau_out, int64_t ld_out, void* stream);
int vd_crba_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* dq, int64_t ld_in, void* M_out,
                void* dM_out, int64_t ld_out, void* stream);
/* forward dynamics by ABA on duals: q̈ and its directional derivative along (dq, dq̇, dτ). */
int vd_aba_jvp(vd_device_model dm, int dtype, int64_t N, const void* q, const void* qd, const void* tau,
               const void* dq, const void* dqd, const void* dtau, int64_t ld_in, const double* gravity3,
               const void* fext, void* qdd_out, void* dqdd_out, int64_t ld_out, int32_t* status_out, void* stream);

/* ------------------------------------------------------------------ host batch (drop-in for batch.hpp)
 * batch_rnea / batch_crba / batch_forward_dynamics (batch.hpp:128-165) with
 * HOST column-major N x n inputs and N x K outputs, fp64.  `workers` becomes a
 * device list: instances are split into contiguous shards (the partition rule
 * of batch_eval, batch.hpp:109-119), one host thread + stream per device, no
 * collective.  Pinned inputs are DMA'd directly; pageable ones are staged
 * through pinned chunks.  forward dynamics reports VD_ERR_SINGULAR_INERTIA if
 * any instance failed (status_out, if given, says which). */
int vd_batch_rnea_host(vd_model m, int64_t N, const double* q, const double* qd, const double* qdd,
                       const double* gravity3, double* tau_out, const int* devices, int n_devices);
int vd_batch_crba_host(vd_model m, int64_t N, const double* q, double* M_out, const int* devices, int n_devices);
int vd_batch_forward_dynamics_host(vd_model m, int64_t N, const double* q, const double* qd, const double* tau,
                                   const double* gravity3, double* qdd_out, int32_t* status_out,
                                   const int* devices, int n_devices);

/* Contiguous shard [begin, end) of N instances for rank r of w (batch.hpp:111-119 rule). */
int vd_shard_range(int64_t N, int world, int rank, int64_t* begin, int64_t* end);

/* ------------------------------------------------------------------ layout
 * Device buffers between a row-major batch (element (i, k) at i*ld_rows + k,
 * e.g. a C array of per-state records or a torch (N, K) tensor) and the
 * planes every kernel above reads and writes (element (i, k) at
 * k*ld_planes + i, the reference's column-major StateBatch layout,
 * batch.hpp:15-19).  Coalesced on both sides (shared-memory staged).  Runs
 * on the calling thread's current device; both buffers must live on it. */
int vd_rows_to_planes(int dtype, int64_t N, int K, const void* rows, int64_t ld_rows, void* planes,
                      int64_t ld_planes, void* stream);
int vd_planes_to_rows(int dtype, int64_t N, int K, const void* planes, int64_t ld_planes, void* rows,
                      int64_t ld_rows, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VECDYN_CUDA_H_ */
