// Host-side dispatch from a Launch descriptor to the per-view launchers.
#include <mutex>

#include "vd_kernels.cuh"

namespace vdk {

extern template struct Launcher<GenericD>;
extern template struct Launcher<GenericF>;
extern template struct Launcher<Chain7D>;
extern template struct Launcher<Chain7F>;

namespace {

// kTreeStatic: whether the compile-time tree29 kernels exist for this op.
// Fully unrolled 29-joint ABA/CRBA/OSC exceed the instruction cache, so those
// run the loop-based kernels with the model in parameter space instead.
template <bool kTreeStatic, class T, class Fn>
int with_view_t(const Launch& L, Fn&& fn) {
  if (L.spec == kChain7) return fn(StaticView<RobotChain7, T>{});
  if constexpr (kTreeStatic) {
    if (L.spec == kTree29) return fn(StaticView<RobotTree29, T>{});
  }
  return fn(RuntimeView<T>{*static_cast<const DevModel<T>*>(L.model)});
}
template <bool kTreeStatic = false, class Fn>
int with_view(const Launch& L, Fn&& fn) {
  return L.dtype == 0 ? with_view_t<kTreeStatic, double>(L, fn) : with_view_t<kTreeStatic, float>(L, fn);
}

}  // namespace

int match_spec(uint64_t fp, int n) { return match_spec_tables(fp, n); }

int scratch_alloc(void** p, size_t bytes, void* stream) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev & 63]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaError_t e = cudaMemPoolCreate(&pools[dev & 63], &props);
      if (e != cudaSuccess) return (int)e;
      uint64_t thr = kScratchKeepBytes;
      cudaMemPoolSetAttribute(pools[dev & 63], cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool = pools[dev & 63];
  }
  *p = nullptr;
  return (int)cudaMallocFromPoolAsync(p, bytes, pool, static_cast<cudaStream_t>(stream));
}

void scratch_free(void* p, void* stream) {
  if (p) cudaFreeAsync(p, static_cast<cudaStream_t>(stream));
}
int launch_jac_scan(const Launch& L, const void* q, const FrameArg& fr, void* pose, void* J);

static bool jit_has_task(const Launch& L, int frame_joint) {
  return L.jit_task && frame_joint >= 0 && frame_joint < 64 && ((L.jit_task_mask >> frame_joint) & 1);
}

// The model's JIT module (vd_jit_entry.cuh), when one is attached; -1 when
// there is none or it has no routine for the call.
static int jit_call(const Launch& L, JitOp op, const void* x0, const void* x1, const void* x2, const double* g3,
                    const void* fext, void* y, int32_t* status) {
  return L.jit ? L.jit(op, &L, x0, x1, x2, g3, fext, y, status) : -1;
}

int launch_fk(const Launch& L, const void* q, void* out) {
  if (L.N == 0) return 0;
  if (const int rc = jit_call(L, kJitFk, q, nullptr, nullptr, nullptr, nullptr, out, nullptr); rc >= 0) return rc;
  if (const int rc = launch_gen_fk(L, q, out); rc >= 0) return rc;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::fk(mv, L, q, out); });
}

int launch_jacobian(const Launch& L, const void* q, int frame_joint, const double* frame_R, const double* frame_p,
                    void* pose, void* J) {
  if (L.N == 0) return 0;
  FrameArg fr;
  fr.joint = frame_joint;
  for (int k = 0; k < 9; ++k) fr.R[k] = frame_R[k];
  for (int k = 0; k < 3; ++k) fr.p[k] = frame_p[k];
  // serial chains at batches below one wave of thread-per-state CTAs: 8 lanes
  // per state (config 2, Panda at N = 4096)
  if (L.serial && L.n <= 32 && L.N <= 32768) return launch_jac_scan(L, q, fr, pose, J);
  if (L.spec == kTree29 || L.spec == kChain7 || jit_has_task(L, frame_joint)) {
    TaskShared P{};
    for (int k = 0; k < 9; ++k) P.frame_R[k] = frame_R[k];
    for (int k = 0; k < 3; ++k) P.frame_p[k] = frame_p[k];
    if (jit_has_task(L, frame_joint)) {
      if (const int rc = L.jit_task(0, &L, frame_joint, q, nullptr, &P, pose, J, nullptr); rc >= 0) return rc;
    }
    if (const int rc = launch_gen_task(L, 0, frame_joint, P, q, pose, J, nullptr); rc >= 0) return rc;
  }
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::jac(mv, L, q, fr, pose, J); });
}

int launch_rnea(const Launch& L0, int mode, const void* q, const void* qd, const void* qdd, const double* g3,
                const void* fext, void* tau) {
  if (L0.N == 0) return 0;
  Launch L = L0;
  if (mode == 3) L.gravity_planes = nullptr;  // Coriolis: no gravity term at all
  static const double zero3[3] = {0, 0, 0};
  const double* g = (mode == 3) ? zero3 : g3;
  const void* qd_ = (mode == 2) ? nullptr : qd;
  const void* qdd_ = (mode == 0) ? qdd : nullptr;
  {
    static const JitOp ops[4] = {kJitRnea, kJitBias, kJitGravity, kJitCoriolis};
    if (const int rc = jit_call(L, ops[mode & 3], q, qd_, qdd_, g3, fext, tau, nullptr); rc >= 0) return rc;
  }
  if (const int rc = launch_gen_rnea(L, mode, q, qd, qdd, g3, fext, tau); rc >= 0) return rc;
  return with_view<true>(L, [&](auto mv) { return Launcher<decltype(mv)>::rnea(mv, L, q, qd_, qdd_, g, fext, tau); });
}

int launch_crba(const Launch& L, const void* q, void* M) {
  if (L.N == 0) return 0;
  if (const int rc = jit_call(L, kJitCrba, q, nullptr, nullptr, nullptr, nullptr, M, nullptr); rc >= 0) return rc;
  if (const int rc = launch_gen_crba(L, q, M); rc >= 0) return rc;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::crba(mv, L, q, M); });
}

namespace {
// Gather of the packed planes from a dense M (models without a generated
// kernel): blockIdx.y = packed plane, x strides over the batch (coalesced).
template <class T>
__global__ void k_pack_lower(int64_t N, const T* __restrict__ M, int64_t ld_m, const __grid_constant__ PackTable tab,
                             T* __restrict__ out, int64_t ld_out) {
  const int k = blockIdx.y;
  const T* src = M + (int64_t)tab.src[k] * ld_m;
  T* dst = out + (int64_t)k * ld_out;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

int launch_crba_packed(const Launch& L, const void* q, void* Mp, const PackTable& tab) {
  if (L.N == 0 || tab.nnz == 0) return 0;
  if (const int rc = jit_call(L, kJitCrbaPacked, q, nullptr, nullptr, nullptr, nullptr, Mp, nullptr); rc >= 0)
    return rc;
  if (const int rc = launch_gen_crba_packed(L, q, Mp); rc >= 0) return rc;
  // Dense M of a chunk of states into pool scratch, then gather.  Chunked so
  // the scratch stays bounded (a 64-dof model at 4M states would otherwise
  // need n²·N·8 B ≈ 137 GB): at most ~256 MB of dense planes per chunk.
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  const size_t es = L.dtype == 0 ? sizeof(double) : sizeof(float);
  const size_t plane_set = (size_t)L.n * L.n * es;
  const int64_t chunk = std::min<int64_t>(L.N, std::max<int64_t>(1024, (int64_t)((256ull << 20) / plane_set)) / 128 * 128);
  void* dense = nullptr;
  if (int rc = scratch_alloc(&dense, (size_t)chunk * plane_set, L.stream)) return rc;
  const size_t tsz = L.dtype == 0 ? sizeof(double) : sizeof(float);
  int rc = 0;
  for (int64_t b = 0; b < L.N && rc == 0; b += chunk) {
    Launch Ld = L;
    Ld.N = std::min<int64_t>(chunk, L.N - b);
    Ld.ld_out = chunk;
    rc = launch_crba(Ld, static_cast<const char*>(q) + b * tsz, dense);
    if (rc != 0) break;
    const dim3 grid((unsigned)std::min<int64_t>((Ld.N + 255) / 256, 1184), (unsigned)tab.nnz);
    if (L.dtype == 0)
      k_pack_lower<double><<<grid, 256, 0, s>>>(Ld.N, (const double*)dense, chunk, tab, (double*)Mp + b, L.ld_out);
    else
      k_pack_lower<float><<<grid, 256, 0, s>>>(Ld.N, (const float*)dense, chunk, tab, (float*)Mp + b, L.ld_out);
    rc = (int)cudaGetLastError();
  }
  scratch_free(dense, L.stream);
  return rc;
}

int launch_aba(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, const void* fext,
               void* qdd, int32_t* status) {
  if (L.N == 0) return 0;
  if (const int rc = jit_call(L, kJitAba, q, qd, tau, g3, fext, qdd, status); rc >= 0) return rc;
  if (const int rc = launch_gen_aba(L, q, qd, tau, g3, fext, qdd, status); rc >= 0) return rc;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::aba(mv, L, q, qd, tau, g3, fext, qdd, status); });
}

int launch_dynamics(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* M,
                    void* bias, void* qdd, int32_t* status) {
  if (L.N == 0) return 0;
  // the JIT module's routines, one launch per output (as tree29 below); per-state
  // gravity takes the same split (the fused loop kernel reads one a_g)
  if (L.jit || L.gravity_planes) {
    int rc = 0;
    if (M && (rc = launch_crba(L, q, M)) != 0) return rc;
    if (bias && (rc = launch_rnea(L, 1, q, qd, nullptr, g3, nullptr, bias)) != 0) return rc;
    if (qdd && (rc = launch_aba(L, q, qd, tau, g3, nullptr, qdd, status)) != 0) return rc;
    return 0;
  }
  if (const int rc = launch_gen_dyn(L, q, qd, tau, g3, M, bias, qdd, status); rc >= 0) return rc;
  if (L.spec == kTree29) {
    // generated kernels, one per output (each re-derives the joint
    // transforms; cheaper than the fused loop kernel's local-memory state)
    int rc = 0;
    if (M && (rc = launch_gen_crba(L, q, M)) != 0) return rc;
    if (bias && (rc = launch_gen_rnea(L, 1, q, qd, nullptr, g3, nullptr, bias)) != 0) return rc;
    if (qdd && (rc = launch_gen_aba(L, q, qd, tau, g3, nullptr, qdd, status)) != 0) return rc;
    return 0;
  }
  return with_view(L,
                   [&](auto mv) { return Launcher<decltype(mv)>::dyn(mv, L, q, qd, tau, g3, M, bias, qdd, status); });
}

int launch_osc(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lambda,
               int32_t* status) {
  if (L.N == 0) return 0;
  if (jit_has_task(L, P.frame_joint)) {
    if (const int rc = L.jit_task(3, &L, P.frame_joint, q, qd, &P, tau, lambda, status); rc >= 0) return rc;
  }
  if (const int rc = launch_gen_osc(L, q, qd, P, tau, lambda, status); rc >= 0) return rc;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::osc(mv, L, q, qd, P, tau, lambda, status); });
}

int launch_task(const Launch& L, const void* q, const TaskShared& P, int mode, void* out, void* aux,
                int32_t* status) {
  if (L.N == 0) return 0;
  if (jit_has_task(L, P.frame_joint)) {
    if (const int rc = L.jit_task(mode == 0 ? 1 : 2, &L, P.frame_joint, q, nullptr, &P, out, mode == 0 ? aux : nullptr,
                                  mode == 0 ? status : nullptr);
        rc >= 0)
      return rc;
  }
  if (const int rc = launch_gen_task(L, mode == 0 ? 1 : 2, P.frame_joint, P, q, out, mode == 0 ? aux : nullptr,
                                     mode == 0 ? status : nullptr);
      rc >= 0)
    return rc;
  return with_view(L, [&](auto mv) { return Launcher<decltype(mv)>::task(mv, L, q, P, mode, out, aux, status); });
}

}  // namespace vdk

// ---------------------------------------------------------------- forward_kinematics_scan
// kinematics.hpp:61-86: Hillis–Steele inclusive scan over transform
// composition, serial chains only.  One segment of `seg` lanes (seg = next
// power of two >= n, <= 32) per robot state: lane j builds the local
// transform of joint j, then log2(seg) shuffle rounds compose
// X_{j-d} ∘ X_j.  Wins over the sequential kernel when N is small (more
// threads in flight per state, log2 n dependent steps instead of n).
namespace vdk {
namespace {
template <class T>
__global__ void __launch_bounds__(128) k_fk_scan(const __grid_constant__ DevModel<T> m, int seg, int64_t N,
                                                 const T* __restrict__ q, int64_t ldi, T* __restrict__ out,
                                                 int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int sub = lane % seg;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t i = warp * (32 / seg) + lane / seg;
  const bool active = i < N && sub < m.n;
  T R[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)}, p[3] = {T(0), T(0), T(0)};
  if (active) {
    const T qi = q[(int64_t)sub * ldi + i];
    T QJ[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)}, tJ[3] = {T(0), T(0), T(0)};
    const T a[3] = {m.axis[sub][0], m.axis[sub][1], m.axis[sub][2]};
    if (m.kind[sub] == 0) {  // Rodrigues, spatial.hpp:302-308
      T s, c;
      sincos_t<T>(qi, &s, &c);
      const T omc = T(1) - c;
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) QJ[r * 3 + k] = a[r] * a[k] * omc + (r == k ? c : T(0));
      QJ[1] -= a[2] * s;
      QJ[2] += a[1] * s;
      QJ[3] += a[2] * s;
      QJ[5] -= a[0] * s;
      QJ[6] -= a[1] * s;
      QJ[7] += a[0] * s;
    } else {
      for (int k = 0; k < 3; ++k) tJ[k] = a[k] * qi;
    }
    for (int r = 0; r < 3; ++r) {  // X_off ∘ X_J
      for (int k = 0; k < 3; ++k)
        R[r * 3 + k] = m.R[sub][r * 3] * QJ[k] + m.R[sub][r * 3 + 1] * QJ[3 + k] + m.R[sub][r * 3 + 2] * QJ[6 + k];
      p[r] = m.R[sub][r * 3] * tJ[0] + m.R[sub][r * 3 + 1] * tJ[1] + m.R[sub][r * 3 + 2] * tJ[2] + m.p[sub][r];
    }
  }
  for (int d = 1; d < seg; d <<= 1) {
    T Rn[9], pn[3];
    for (int k = 0; k < 9; ++k) Rn[k] = __shfl_up_sync(0xffffffffu, R[k], d, seg);
    for (int k = 0; k < 3; ++k) pn[k] = __shfl_up_sync(0xffffffffu, p[k], d, seg);
    if (sub >= d) {
      T R2[9], p2[3];
      for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) R2[r * 3 + k] = Rn[r * 3] * R[k] + Rn[r * 3 + 1] * R[3 + k] + Rn[r * 3 + 2] * R[6 + k];
        p2[r] = Rn[r * 3] * p[0] + Rn[r * 3 + 1] * p[1] + Rn[r * 3 + 2] * p[2] + pn[r];
      }
      for (int k = 0; k < 9; ++k) R[k] = R2[k];
      for (int k = 0; k < 3; ++k) p[k] = p2[k];
    }
  }
  if (active) {
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) out[(int64_t)(sub * 12 + c * 3 + r) * ldo + i] = R[r * 3 + c];
    for (int r = 0; r < 3; ++r) out[(int64_t)(sub * 12 + 9 + r) * ldo + i] = p[r];
  }
}
}  // namespace

// frame pose + geometric Jacobian (kinematics.hpp:89-136) for serial chains
// at small batches: the scan above gives lane j its world transform W_j; the
// frame's lane composes the frame offset and broadcasts the frame point; lane
// j writes Jacobian column j (zero off the ancestor path).  8 lanes per state
// instead of one thread: a 4096-state batch fills 256 CTAs instead of 32.
// model accessors for the scan kernel: the packed model by value (any serial
// chain) or a robot's compile-time tables (no kernel-parameter payload)
template <class T>
struct ScanDev {
  DevModel<T> m;
  __device__ __forceinline__ int n() const { return m.n; }
  __device__ __forceinline__ int kind(int j) const { return m.kind[j]; }
  __device__ __forceinline__ T axis(int j, int k) const { return m.axis[j][k]; }
  __device__ __forceinline__ T R(int j, int k) const { return m.R[j][k]; }
  __device__ __forceinline__ T p(int j, int k) const { return m.p[j][k]; }
  __device__ __forceinline__ uint64_t anc(int j) const { return m.anc[j]; }
};
template <class Robot, class T>
struct ScanStatic {
  __device__ __forceinline__ int n() const { return Robot::kN; }
  __device__ __forceinline__ int kind(int j) const { return Robot::kind()[j]; }
  __device__ __forceinline__ T axis(int j, int k) const { return T(Robot::axis()[j * 3 + k]); }
  __device__ __forceinline__ T R(int j, int k) const { return T(Robot::rot()[j * 9 + k]); }
  __device__ __forceinline__ T p(int j, int k) const { return T(Robot::pos()[j * 3 + k]); }
  __device__ __forceinline__ uint64_t anc(int j) const { return Robot::anc()[j]; }
};

template <class T, class M>
__global__ void __launch_bounds__(128) k_jac_scan(const __grid_constant__ M m, int seg, int64_t N,
                                                  const T* __restrict__ q, int64_t ldi, int fj,
                                                  const __grid_constant__ FrameArg fr, T* __restrict__ pose,
                                                  T* __restrict__ J, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int sub = lane % seg;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t i = warp * (32 / seg) + lane / seg;
  const bool active = i < N && sub < m.n();
  const int64_t ii = i < N ? i : N - 1;
  T R[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)}, p[3] = {T(0), T(0), T(0)};
  if (sub < m.n()) {
    const T qi = q[(int64_t)sub * ldi + ii];
    T QJ[9] = {T(1), T(0), T(0), T(0), T(1), T(0), T(0), T(0), T(1)}, tJ[3] = {T(0), T(0), T(0)};
    const T a[3] = {m.axis(sub, 0), m.axis(sub, 1), m.axis(sub, 2)};
    if (m.kind(sub) == 0) {  // Rodrigues, spatial.hpp:302-308
      T s, c;
      sincos_t<T>(qi, &s, &c);
      const T omc = T(1) - c;
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) QJ[r * 3 + k] = a[r] * a[k] * omc + (r == k ? c : T(0));
      QJ[1] -= a[2] * s;
      QJ[2] += a[1] * s;
      QJ[3] += a[2] * s;
      QJ[5] -= a[0] * s;
      QJ[6] -= a[1] * s;
      QJ[7] += a[0] * s;
    } else {
      for (int k = 0; k < 3; ++k) tJ[k] = a[k] * qi;
    }
    for (int r = 0; r < 3; ++r) {  // X_off ∘ X_J
      for (int k = 0; k < 3; ++k)
        R[r * 3 + k] = m.R(sub, r * 3) * QJ[k] + m.R(sub, r * 3 + 1) * QJ[3 + k] + m.R(sub, r * 3 + 2) * QJ[6 + k];
      p[r] = m.R(sub, r * 3) * tJ[0] + m.R(sub, r * 3 + 1) * tJ[1] + m.R(sub, r * 3 + 2) * tJ[2] + m.p(sub, r);
    }
  }
  for (int d = 1; d < seg; d <<= 1) {
    T Rn[9], pn[3];
    for (int k = 0; k < 9; ++k) Rn[k] = __shfl_up_sync(0xffffffffu, R[k], d, seg);
    for (int k = 0; k < 3; ++k) pn[k] = __shfl_up_sync(0xffffffffu, p[k], d, seg);
    if (sub >= d) {
      T R2[9], p2[3];
      for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) R2[r * 3 + k] = Rn[r * 3] * R[k] + Rn[r * 3 + 1] * R[3 + k] + Rn[r * 3 + 2] * R[6 + k];
        p2[r] = Rn[r * 3] * p[0] + Rn[r * 3 + 1] * p[1] + Rn[r * 3 + 2] * p[2] + pn[r];
      }
      for (int k = 0; k < 9; ++k) R[k] = R2[k];
      for (int k = 0; k < 3; ++k) p[k] = p2[k];
    }
  }
  // frame pose on lane fj (frame_transform, kinematics.hpp:89-96), broadcast the frame point
  T PR[9], Pp[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c)
      PR[r * 3 + c] = R[r * 3] * T(fr.R[c]) + R[r * 3 + 1] * T(fr.R[3 + c]) + R[r * 3 + 2] * T(fr.R[6 + c]);
    Pp[r] = R[r * 3] * T(fr.p[0]) + R[r * 3 + 1] * T(fr.p[1]) + R[r * 3 + 2] * T(fr.p[2]) + p[r];
  }
  const int src = fj >= 0 ? fj : 0;
  T Pf[3];
  for (int k = 0; k < 3; ++k) Pf[k] = __shfl_sync(0xffffffffu, Pp[k], src, seg);
  if (!active) return;
  if (pose && sub == src) {
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) pose[(int64_t)(c * 3 + r) * ldo + i] = fj >= 0 ? PR[r * 3 + c] : T(r == c);
    for (int r = 0; r < 3; ++r) pose[(int64_t)(9 + r) * ldo + i] = fj >= 0 ? Pp[r] : T(fr.p[r]);
  }
  if (J) {  // geometric_jacobian (kinematics.hpp:108-129)
    T col[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
    if (fj >= 0 && ((m.anc(fj) >> sub) & 1ull)) {
      T ax[3];
      for (int r = 0; r < 3; ++r) ax[r] = R[r * 3] * m.axis(sub, 0) + R[r * 3 + 1] * m.axis(sub, 1) + R[r * 3 + 2] * m.axis(sub, 2);
      if (m.kind(sub) == 0) {
        const T d[3] = {Pf[0] - p[0], Pf[1] - p[1], Pf[2] - p[2]};
        col[0] = ax[0];
        col[1] = ax[1];
        col[2] = ax[2];
        col[3] = ax[1] * d[2] - ax[2] * d[1];
        col[4] = ax[2] * d[0] - ax[0] * d[2];
        col[5] = ax[0] * d[1] - ax[1] * d[0];
      } else {
        col[3] = ax[0];
        col[4] = ax[1];
        col[5] = ax[2];
      }
    }
    for (int r = 0; r < 6; ++r) J[(int64_t)(sub * 6 + r) * ldo + i] = col[r];
  }
}

int launch_jac_scan(const Launch& L, const void* q, const FrameArg& fr, void* pose, void* J) {
  int seg = 1;
  while (seg < L.n) seg <<= 1;
  const int64_t threads = ((L.N + (32 / seg) - 1) / (32 / seg)) * 32;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  auto go = [&](auto m, auto tag) {
    using T = decltype(tag);
    k_jac_scan<T><<<grid, 128, 0, s>>>(m, seg, L.N, (const T*)q, L.ld_in, fr.joint, fr, (T*)pose, (T*)J, L.ld_out);
  };
  if (L.spec == kChain7) {
    if (L.dtype == 0) go(ScanStatic<RobotChain7, double>{}, double());
    else go(ScanStatic<RobotChain7, float>{}, float());
  } else if (L.dtype == 0) {
    go(ScanDev<double>{*static_cast<const DevModel<double>*>(L.model)}, double());
  } else {
    go(ScanDev<float>{*static_cast<const DevModel<float>*>(L.model)}, float());
  }
  return (int)cudaGetLastError();
}

int launch_fk_scan(const Launch& L, const void* q, void* out) {
  if (L.N == 0) return 0;
  int seg = 1;
  while (seg < L.n) seg <<= 1;
  const int64_t threads = ((L.N + (32 / seg) - 1) / (32 / seg)) * 32;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  if (L.dtype == 0)
    k_fk_scan<double><<<grid, 128, 0, static_cast<cudaStream_t>(L.stream)>>>(
        *static_cast<const DevModel<double>*>(L.model), seg, L.N, (const double*)q, L.ld_in, (double*)out, L.ld_out);
  else
    k_fk_scan<float><<<grid, 128, 0, static_cast<cudaStream_t>(L.stream)>>>(
        *static_cast<const DevModel<float>*>(L.model), seg, L.N, (const float*)q, L.ld_in, (float*)out, L.ld_out);
  return (int)cudaGetLastError();
}

}  // namespace vdk
