// Launchers for the generated straight-line robot kernels (vd_gen_kernels.cuh,
// tools/gen_tree_kernels.py).  tree29 (G1) ABA, RNEA (+ bias / gravity /
// Coriolis), CRBA and FK run here: the fully unrolled template kernels are
// dominated by flag/select overhead and the loop kernels by local-memory
// state.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <utility>

#include "vd_gen_robots.cuh"
#include "vd_gen_launch.cuh"

namespace vdk {

// The headline kernel, N = 4M states (tools/async_sweep.cu, one B200):
// plain k_gen r44 s28 b4 0.599 ms; async r30 s35 b4 0.555, + evict-first
// 0.548, r24 s41 (3 CTAs/SM) 0.543 ms; the templated TMA kernel 0.61 ms.
// Double-buffered input (k_gen_db, every group of the next state in flight
// for a whole state; tools/pool_call_sweep.cu gdb4): r44 s21 b3 0.520 ms
// against the async kernel's 0.536-0.541 in the same run, same results.
template <>
struct Cfg<GenChain7::Aba, double> {
  static constexpr int kReg = 44, kSmem = 21, kMinB = 3;
  static constexpr int kFast = kTrigFast;
  static constexpr bool kStream = true, kDb = true;
};
// chain7 fp32 ABA: generated + async, 0.41 ms for the templated TMA kernel ->
// r40 s25 (6 CTAs/SM) 0.299 ms at 4M states with sincosf -> r30 s35 (5
// CTAs/SM) 0.287 ms with vd_sincos_f32 (async_sweep c7f) -> double-buffered
// input 0.278 ms (gdb4)
template <>
struct Cfg<GenChain7::Aba, float> {
  static constexpr int kReg = 30, kSmem = 35, kMinB = 5;
  static constexpr int kFast = kTrigFast;
  static constexpr bool kDb = true;
};
// chain7 RNEA family: all slots in registers, fast fp64 sincos (gen_sweep:
// fp64 0.252 vs 0.261 ms templated, fp32 0.142 vs 0.153 ms at 4M states);
// double-buffered input (gdb4): fp64 0.258 -> 0.240 ms, fp32 0.147 -> 0.139 ms
template <class T, int kSlotsAll>
struct Chain7RneaCfg {
  static constexpr int kReg = kSlotsAll, kSmem = 0, kMinB = sizeof(T) == 8 ? 4 : 6;
  static constexpr int kFast = sizeof(T) == 8 ? kTrigFast : kTrigLib;  // fp32: vd_sincos_f32 measured 4 % slower
  static constexpr bool kDb = true;
};
template <class T>
struct Cfg<GenChain7::Rnea, T> : Chain7RneaCfg<T, GenChain7::Rnea::kSlots> {};
template <class T>
struct Cfg<GenChain7::RneaBias, T> : Chain7RneaCfg<T, GenChain7::RneaBias::kSlots> {};
template <class T>
struct Cfg<GenChain7::RneaGrav, T> : Chain7RneaCfg<T, GenChain7::RneaGrav::kSlots> {};
// G1 ABA / dense CRBA with evict-first state I/O (gen_sweep, two runs each,
// N = 262144): ABA fp64 0.31-0.42 -> 0.29 ms, mixed fp32 0.19 -> 0.17 ms,
// CRBA fp64 0.39 (s40 b4) -> 0.30 ms (s55 b3), fp32 0.30 -> 0.16 ms
// f_ext routines: the placement of their plain counterparts
template <class T>
struct Cfg<GenChain7::RneaFext, T> : Chain7RneaCfg<T, GenChain7::RneaFext::kSlots> {};
template <class T>
struct Cfg<GenChain7::RneaBiasFext, T> : Chain7RneaCfg<T, GenChain7::RneaBiasFext::kSlots> {};
template <class T>
struct Cfg<GenChain7::AbaFext, T> : Cfg<GenChain7::Aba, T> {};
// G1 sin/cos: one out-of-line copy of the library routine (kTrigCall) in the
// ABA / RNEA families, whose straight-line code is instruction-cache bound
// (async_sweep "t29", sweep.py, 262144 states: ABA fp64 0.295 -> 0.264 ms,
// mixed fp32 0.170 -> 0.146 ms, RNEA fp64 0.100 -> 0.094 ms); the CRBA, FK
// and gravity routines stay inlined (the call makes them 1-15 % slower).
// The G1 ABA reads its constants from the __constant__ table (codegen
// POOL_OPS) and runs out of line per state (k_gen_call): 0.261 -> 0.242 ms.
template <>
struct Cfg<GenTree29::Aba, double> {
  static constexpr int kReg = 40, kSmem = 113, kMinB = 2;
  static constexpr int kFast = kTrigCall;
  static constexpr bool kStream = true, kCall = true;
};
template <>
struct Cfg<GenTree29::AbaMixed, float> {  // the trunk's fp64 slots (stored last) in registers
  static constexpr int kReg = 40, kSmem = 122, kMinB = 3;
  static constexpr int kFast = kTrigCall;
  static constexpr bool kStream = true;
};
template <>
struct Cfg<GenTree29::Crba, double> {
  static constexpr int kReg = 0, kSmem = 55, kMinB = 3;
  static constexpr int kFast = kTrigLib;
  static constexpr bool kStream = true;
};
template <>
struct Cfg<GenTree29::Crba, float> {
  static constexpr int kReg = 0, kSmem = 55, kMinB = 4;
  static constexpr int kFast = kTrigLib;
  static constexpr bool kStream = true;
};
// packed CRBA (gen_sweep, N = 262144 / 4M): tree29 fp64 all 55 slots in
// registers at 3 CTAs/SM 0.112 ms (vs 0.133 with the dense routine's
// placement); fp32 in shared memory at 6 CTAs/SM 0.061 ms; chain7 fp64 all in
// registers 0.21 ms at 4M states (85 % of HBM)
// fp64 with the out-of-line sin/cos and evict-first output
// (tools/pool_call_sweep.cu crbap): 0.114 -> 0.104 ms
template <>
struct Cfg<GenTree29::CrbaPacked, double> {
  static constexpr int kReg = GenTree29::CrbaPacked::kSlots, kSmem = 0, kMinB = 3;
  static constexpr int kFast = kTrigCall;
  static constexpr bool kStream = true;
};
template <>
struct Cfg<GenTree29::CrbaPacked, float> {
  static constexpr int kReg = 0, kSmem = GenTree29::CrbaPacked::kSlots, kMinB = 6;
  static constexpr int kFast = kTrigLib;
};
template <class T>
struct Cfg<GenChain7::CrbaPacked, T> {
  static constexpr int kReg = GenChain7::CrbaPacked::kSlots, kSmem = 0, kMinB = 4;
  static constexpr int kFast = kTrigLib;
};
template <>
struct Cfg<GenTree29::Rnea, double> {  // prologue: cos/sin, q̇, q̈ of every joint
  static constexpr int kReg = 58, kSmem = 55, kMinB = 2;
  static constexpr int kFast = kTrigCall;
};
template <>
struct Cfg<GenTree29::Rnea, float> {
  static constexpr int kReg = 55, kSmem = 0, kMinB = 3;
  static constexpr int kFast = kTrigCall;
};
template <>
struct Cfg<GenTree29::RneaBias, double> {
  static constexpr int kReg = 0, kSmem = 72, kMinB = 3;
  static constexpr int kFast = kTrigCall;
};
template <class T>
struct Cfg<GenTree29::RneaFext, T> : Cfg<GenTree29::Rnea, T> {};
template <>
struct Cfg<GenTree29::RneaBiasFext, double> : Cfg<GenTree29::RneaBias, double> {};
template <>
struct Cfg<GenTree29::AbaFext, double> : Cfg<GenTree29::Aba, double> {};
template <>
struct Cfg<GenTree29::AbaMixedFext, float> : Cfg<GenTree29::AbaMixed, float> {};

// chain7 (Panda `ee`), N = 4M, tools/async_sweep.cu "more": every slot on
// chip.  fp64 r80 s67 b2 1.45 ms, fp32 r60 s87 1.56 -> 0.70 ms, against the
// templated osc_one kernel 2.35 / 1.57 ms.
// fp32 with double-buffered asynchronous q, q̇ (k_gen_osc_db; pool_call_sweep
// oscdb, 2M states): 0.347 -> 0.332 ms; fp64 0.725 -> 0.716 ms, kept plain.
template <class T>
struct OscCfg<GenChain7::Osc6, T> {
  static constexpr int kReg = sizeof(T) == 8 ? 80 : 60, kSmem = sizeof(T) == 8 ? 67 : 87, kMinB = 2;
  static constexpr int kFast = kTrigLib;
  static constexpr bool kAsync = sizeof(T) == 4;
};

namespace {

// Placement caps, clamped to the routine's own slot count so a small routine
// (FK-JVP, CRBA-JVP) does not reserve shared memory it never touches and is
// not held at the occupancy of the largest one (ABA-JVP).
template <class Op, class T>
struct JvpCfg {
  static constexpr int kRegCap = sizeof(T) == 8 ? 40 : 0, kSmemCap = sizeof(T) == 8 ? 110 : 220;
  static constexpr int kReg = kRegCap < Op::kSlots ? kRegCap : Op::kSlots;
  static constexpr int kSmem = kSmemCap < Op::kSlots - kReg ? kSmemCap : Op::kSlots - kReg;
  // fp32 routines up to 110 slots at 3 CTAs/SM (async_sweep "jvp", G1 at
  // 262144: CRBA-JVP 0.50 -> 0.43 ms, FK-JVP 0.25 -> 0.20 ms); fp64 and the
  // larger routines measured best at 2 (255 registers)
  static constexpr int kMinB = sizeof(T) == 4 && Op::kSlots <= 110 ? 3 : 2;
  static constexpr int kFast = kTrigLib;
};

// G1 ABA-JVP (526 slots; measured as the dual routine, now replaced by
// aba_jvp_implicit below): one CTA/SM with 220 shared slots keeps the scratch
// slab in L2 (async_sweep "jvp", 262144 states: fp64 r40 s110 b2 1.50 ->
// r40 s220 b1 1.24 ms; fp32 s220 b2 0.72 -> r40 s220 b2 0.64 ms); G1 fp32
// RNEA-JVP s220 b2 0.27 -> s144 b3 0.25 ms.
// sin/cos by one out-of-line copy (kTrigCall; async_sweep "trig"): ABA-JVP
// fp64 1.244 -> 1.207 ms, fp32 0.590 -> 0.567 ms, RNEA-JVP fp32 0.201 -> 0.172
// ms (fp64 RNEA-JVP is slower with it: 0.50 -> 0.57 ms).
template <class T>
struct JvpCfg<GenTree29::AbaJvp, T> {
  static constexpr int kReg = 40, kSmem = 220, kMinB = sizeof(T) == 8 ? 1 : 2;
  static constexpr int kFast = kTrigCall;
};
template <>
struct JvpCfg<GenTree29::RneaJvp, float> {
  static constexpr int kReg = 0, kSmem = 144, kMinB = 3;
  static constexpr int kFast = kTrigCall;
  static constexpr bool kCall = true;
};
// Routine out of line once per state (k_gen_jvp_call; tools/pool_call_sweep.cu,
// G1, 262144 states, loop -> call): fp64 RNEA-JVP 0.511 -> 0.336 ms (with the
// sin/cos call), CRBA-JVP 0.727 -> 0.685 ms; fp32 RNEA-JVP 0.176 -> 0.171,
// FK-JVP 0.147 -> 0.137 ms.  The ABA-JVP and the fp64 FK-JVP are slower with it.
template <>
struct JvpCfg<GenTree29::RneaJvp, double> {
  static constexpr int kReg = 40, kSmem = 110, kMinB = 2;
  static constexpr int kFast = kTrigCall;
  static constexpr bool kCall = true;
};
template <>
struct JvpCfg<GenTree29::CrbaJvp, double> {
  static constexpr int kReg = 40, kSmem = GenTree29::CrbaJvp::kSlots - 40, kMinB = 2;
  static constexpr int kFast = kTrigCall;
  static constexpr bool kCall = true;
};
template <>
struct JvpCfg<GenTree29::FkJvp, float> {
  static constexpr int kReg = 0, kSmem = GenTree29::FkJvp::kSlots, kMinB = 3;
  static constexpr int kFast = kTrigLib;
  static constexpr bool kCall = true;
};

template <class Op, class T, bool kStream>
int launch_jvp_v(const Launch& L, const JvpArgs& a) {
  using C = JvpCfg<Op, T>;
  auto kern = [] {
    if constexpr (CallIo<C>::value) return k_gen_jvp_call<Op, T, C::kReg, C::kSmem, C::kMinB, kStream, C::kFast>;
    else return k_gen_jvp<Op, T, C::kReg, C::kSmem, C::kMinB, kStream, C::kFast>;
  }();
  constexpr size_t smem = (size_t)C::kSmem * kGenBlock * sizeof(T);
  const Occ o = occupancy<std::pair<Op, std::bool_constant<kStream>>, T>(kern, smem);
  const int64_t blocks = std::min<int64_t>((L.N + kGenBlock - 1) / kGenBlock, (int64_t)o.sms * o.blocks_per_sm);
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  const size_t scratch_bytes = (size_t)blocks * kGenBlock * gen_scratch_per_thread<Op, T, C::kReg, C::kSmem>() * sizeof(T);
  T* scratch = nullptr;
  if (scratch_bytes) {
    if (int rc = scratch_alloc(reinterpret_cast<void**>(&scratch), scratch_bytes, s)) return rc;
  }
  kern<<<(unsigned)blocks, kGenBlock, smem, s>>>(L.N, a, L.ld_in, L.ld_out, scratch);
  cudaError_t e = cudaGetLastError();
  scratch_free(scratch, s);
  return (int)e;
}

// The JVPs read and write every value/tangent plane once: evict-first I/O
// throughout (tools/jvp_time.py, G1, N = 262144, plain -> .cs): fp64 FK-JVP
// 0.46 -> 0.37 ms, RNEA-JVP 1.03 -> 0.82, CRBA-JVP 1.33 -> 0.80, ABA-JVP
// 1.81 -> 1.80; fp32 FK-JVP 0.40 -> 0.27, CRBA-JVP 1.12 -> 0.59, ABA-JVP
// 1.20 -> 0.93, RNEA-JVP 0.47 -> 0.47.
template <class Op, class T>
int launch_jvp_t(const Launch& L, const JvpArgs& a) {
  return launch_jvp_v<Op, T, true>(L, a);
}

}  // namespace

int launch_gen_aba(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3,
                   const void* fext, void* qdd, int32_t* status) {
  if (L.spec == kChain7) {
    if (fext)
      return L.dtype == 0 ? launch_t<GenChain7::AbaFext, double>(L, q, qd, tau, g3, qdd, status, fext)
                          : launch_t<GenChain7::AbaFext, float>(L, q, qd, tau, g3, qdd, status, fext);
    return L.dtype == 0 ? launch_t<GenChain7::Aba, double>(L, q, qd, tau, g3, qdd, status)
                        : launch_t<GenChain7::Aba, float>(L, q, qd, tau, g3, qdd, status);
  }
  if (L.spec != kTree29) return -1;
  // fp32: the mixed-precision routine (floating-base trunk in fp64)
  if (fext)
    return L.dtype == 0 ? launch_t<GenTree29::AbaFext, double>(L, q, qd, tau, g3, qdd, status, fext)
                        : launch_t<GenTree29::AbaMixedFext, float>(L, q, qd, tau, g3, qdd, status, fext);
  return L.dtype == 0 ? launch_t<GenTree29::Aba, double>(L, q, qd, tau, g3, qdd, status)
                      : launch_t<GenTree29::AbaMixed, float>(L, q, qd, tau, g3, qdd, status);
}

template <class R>
int gen_rnea_t(const Launch& L, int mode, const void* q, const void* qd, const void* qdd, const double* g3,
               const void* fext, void* tau) {
  // mode 0 full, 1 bias (q̈ = 0), 2 gravity (q̇ = q̈ = 0), 3 Coriolis (q̈ = 0, g = 0);
  // a NULL q̇ / q̈ means zeros, as in the template kernels
  static const double zero3[3] = {0, 0, 0};
  const bool has_qd = mode != 2 && qd, has_qdd = mode == 0 && qdd;
  const double* g = mode == 3 ? zero3 : g3;
  if (fext) {  // f_ext variants: full RNEA and the bias term
    if (has_qd && has_qdd) return launch_op<typename R::RneaFext>(L, q, qd, qdd, g, tau, nullptr, fext);
    if (has_qd && mode == 1) return launch_op<typename R::RneaBiasFext>(L, q, qd, nullptr, g, tau, nullptr, fext);
    return -1;
  }
  if (has_qd && has_qdd) return launch_op<typename R::Rnea>(L, q, qd, qdd, g, tau, nullptr);
  if (has_qd) return launch_op<typename R::RneaBias>(L, q, qd, nullptr, g, tau, nullptr);
  if (!has_qdd) return launch_op<typename R::RneaGrav>(L, q, nullptr, nullptr, g, tau, nullptr);
  return -1;  // q̇ = 0 with q̈: no generated variant, template kernel
}

int launch_gen_rnea(const Launch& L, int mode, const void* q, const void* qd, const void* qdd, const double* g3,
                    const void* fext, void* tau) {
  if (L.spec == kTree29) return gen_rnea_t<GenTree29>(L, mode, q, qd, qdd, g3, fext, tau);
  if (L.spec == kChain7) return gen_rnea_t<GenChain7>(L, mode, q, qd, qdd, g3, fext, tau);
  return -1;
}

template <class R>
int gen_osc_t(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lambda,
              int32_t* status) {
  int rc = -1;
  R::with_osc(P.frame_joint, [&](auto op) {
    using Op = decltype(op);
    rc = L.dtype == 0 ? launch_osc_t<Op, double>(L, q, qd, P, tau, lambda, status)
                      : launch_osc_t<Op, float>(L, q, qd, P, tau, lambda, status);
  });
  return rc;
}

// Panda M + bias + q̈ in one generated routine (GenChain7::Dyn: one prologue,
// CRBA, RNEA at q̈ = 0 and ABA straight-line; tools/dyn_sweep.cu, against
// the fused template kernel k_tiled<OpDyn> 20.5 us / 0.083 / 1.277 ms at
// 65536 / 262144 / 4M states): r40 s25 at 3 CTAs/SM with the Cody-Waite
// sin/cos 19.1 us / 0.070 / 1.040 ms.  fp32 (template 16.4 us / 0.648 ms at
// 65536 / 4M): every slot in registers at 4 CTAs/SM, 12.3 us / 0.561 ms.
// Per-state gravity takes the three-launch split.
template <class T>
int launch_gen_dyn_t(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* M,
                     void* bias, void* qdd, int32_t* status) {
  using Op = GenChain7::Dyn;
  constexpr bool f64 = sizeof(T) == 8;
  constexpr int kReg = f64 ? 40 : Op::kSlots, kSmem = Op::kSlots - kReg, kMinB = f64 ? 3 : 4;
  auto kern = k_gen_dyn<Op, T, kReg, kSmem, kMinB, kTrigFast, false>;
  constexpr size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  const Occ o = occupancy<Op, T>(kern, smem);
  const int64_t blocks = std::min<int64_t>((L.N + kGenBlock - 1) / kGenBlock, (int64_t)o.sms * o.blocks_per_sm);
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  static_assert(gen_scratch_per_thread<Op, T, kReg, kSmem>() == 0, "every Dyn slot on chip");
  const T g0 = g3 ? T(g3[0]) : T(0), g1 = g3 ? T(g3[1]) : T(0), g2 = g3 ? T(g3[2]) : T(9.81);
  kern<<<(unsigned)blocks, kGenBlock, smem, s>>>(L.N, (const T*)q, (const T*)qd, (const T*)tau, L.ld_in, g0, g1, g2,
                                                 (T*)M, (T*)bias, (T*)qdd, L.ld_out, status, nullptr);
  return (int)cudaGetLastError();
}
int launch_gen_dyn(const Launch& L, const void* q, const void* qd, const void* tau, const double* g3, void* M,
                   void* bias, void* qdd, int32_t* status) {
  if (L.spec != kChain7 || L.gravity_planes) return -1;
  return L.dtype == 0 ? launch_gen_dyn_t<double>(L, q, qd, tau, g3, M, bias, qdd, status)
                      : launch_gen_dyn_t<float>(L, q, qd, tau, g3, M, bias, qdd, status);
}

int launch_gen_osc(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lambda,
                   int32_t* status) {
  if (L.spec == kTree29) return gen_osc_t<GenTree29>(L, q, qd, P, tau, lambda, status);
  if (L.spec == kChain7) return gen_osc_t<GenChain7>(L, q, qd, P, tau, lambda, status);
  return -1;
}

template <class R>
int gen_jvp_t(const Launch& L, const JvpArgs& a) {
  // (the G1 ABA-JVP takes the implicit-function form below, never the dual routine)
  if constexpr (!std::is_same_v<R, GenTree29>) {
    if (a.op == kJvpABA)
      return L.dtype == 0 ? launch_jvp_t<typename R::AbaJvp, double>(L, a)
                          : launch_jvp_t<typename R::AbaJvp, float>(L, a);
  }
  if (a.op == kJvpRNEA)
    return L.dtype == 0 ? launch_jvp_t<typename R::RneaJvp, double>(L, a)
                        : launch_jvp_t<typename R::RneaJvp, float>(L, a);
  if (a.op == kJvpCRBA)
    return L.dtype == 0 ? launch_jvp_t<typename R::CrbaJvp, double>(L, a)
                        : launch_jvp_t<typename R::CrbaJvp, float>(L, a);
  return L.dtype == 0 ? launch_jvp_t<typename R::FkJvp, double>(L, a) : launch_jvp_t<typename R::FkJvp, float>(L, a);
}

// rhs planes of the ABA-JVP identity below: t <- dτ − t (dτ NULL = 0)
template <class T>
__global__ void k_jvp_rhs(int64_t N, int n, const T* __restrict__ dtau, int64_t ld, T* __restrict__ t) {
  const int64_t total = N * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / N, i = e - k * N;
    t[k * ld + i] = (dtau ? dtau[k * ld + i] : T(0)) - t[k * ld + i];
  }
}

// G1 ABA-JVP by the implicit-function identity instead of the dual-number
// ABA.  FD is the solution of ID(q, q̇, q̈) = τ, so its directional derivative
// along (dq, dq̇, dτ) is
//   dq̈ = M⁻¹ (dτ − ∂ID/∂q·dq − ∂ID/∂q̇·dq̇)
// where the bracketed term is the tangent of RNEA-JVP at (q, q̇, q̈) with
// tangent (dq, dq̇, 0), and M⁻¹ b is the ABA at zero velocity and zero gravity
// with b as the joint force.  Four launches — ABA (q̈, status), RNEA-JVP,
// t ← dτ − t, ABA(q, 0, t, g = 0) into dq̈ — replace the 526-slot dual ABA
// (one CTA/SM, its slot state in an L2 scratch slab): fp64 1.21 -> 0.875 ms,
// fp32 0.567 -> 0.531 ms at 262 144 states (tools/jvp_time.py, C-ABI on plane
// buffers), and the value output is the plain ABA's, bit for bit.  The same derivative up to
// rounding: parity against the oracle's dual-number LLT forward dynamics
// (tests/test_gpu_jvp.py, κ(M)-scaled bounds as for the dual kernel).
template <class T>
int aba_jvp_implicit(const Launch& L, const JvpArgs& a) {
  if (!a.dout) return launch_gen_aba(L, a.x[0], a.x[1], a.x[2], a.g, nullptr, a.out, a.status);
  const int n = L.n;
  const int64_t ld = L.ld_in;
  const size_t plane_set = sizeof(T) * (size_t)n * (size_t)ld;
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  // q̈ goes straight to the caller's output when its layout matches the inputs'
  const bool direct = a.out && L.ld_out == ld;
  unsigned char* buf = nullptr;
  if (int rc = scratch_alloc(reinterpret_cast<void**>(&buf), plane_set * (direct ? 2 : 3), s)) return rc;
  T* zero = reinterpret_cast<T*>(buf);
  T* t = reinterpret_cast<T*>(buf + plane_set);
  T* qdd = direct ? static_cast<T*>(a.out) : reinterpret_cast<T*>(buf + 2 * plane_set);
  Launch Li = L;  // intermediate launches: outputs laid out like the inputs
  Li.ld_out = ld;
  int rc = launch_gen_aba(Li, a.x[0], a.x[1], a.x[2], a.g, nullptr, qdd, a.status);
  if (!rc) {
    JvpArgs r{kJvpRNEA, {a.x[0], a.x[1], qdd}, {a.dx[0], a.dx[1], nullptr}, {a.g[0], a.g[1], a.g[2]}, nullptr,
              nullptr, t, nullptr};
    rc = launch_jvp_t<GenTree29::RneaJvp, T>(Li, r);
  }
  if (!rc) {
    const int64_t blocks = std::min<int64_t>((L.N * n + 255) / 256, 148 * 16);
    k_jvp_rhs<T><<<(unsigned)blocks, 256, 0, s>>>(L.N, n, static_cast<const T*>(a.dx[2]), ld, t);
    rc = (int)cudaGetLastError();
  }
  if (!rc) rc = (int)cudaMemsetAsync(zero, 0, plane_set, s);
  if (!rc) {
    const double g0[3] = {0.0, 0.0, 0.0};
    rc = launch_gen_aba(L, a.x[0], zero, t, g0, nullptr, a.dout, nullptr);
  }
  if (!rc && a.out && !direct)
    rc = (int)cudaMemcpy2DAsync(a.out, sizeof(T) * L.ld_out, qdd, sizeof(T) * ld, sizeof(T) * L.N, n,
                                cudaMemcpyDeviceToDevice, s);
  scratch_free(buf, s);
  return rc;
}

int launch_gen_jvp(const Launch& L, const JvpArgs& a) {
  if (a.fext && (a.op == kJvpABA || a.op == kJvpRNEA)) return -1;
  if (L.spec == kTree29 && a.op == kJvpABA)
    return L.dtype == 0 ? aba_jvp_implicit<double>(L, a) : aba_jvp_implicit<float>(L, a);
  if (L.spec == kTree29) return gen_jvp_t<GenTree29>(L, a);
  // chain7 (tools/jvp_time.py, 1M states, Python API, template -> generated):
  // fp64 FK-JVP 0.39 -> 0.37, RNEA-JVP 0.55 -> 0.36, CRBA-JVP 0.35 -> 0.25,
  // ABA-JVP 0.84 -> 0.66 ms; fp32 0.22/0.34/0.17/0.56 -> 0.21/0.23/0.16/0.43 ms
  if (L.spec == kChain7) return gen_jvp_t<GenChain7>(L, a);
  return -1;
}

// which: 0 Jacobian (y0 pose, y1 J), 1 diff-IK (y0 q̇, y1 err), 2 manipulability (y0 w)
template <class R>
int gen_task_t(const Launch& L, int which, int frame_joint, const TaskShared& P, const void* q, void* y0, void* y1,
               int32_t* status, const void* dq) {
  int rc = -1;
  R::with_task(frame_joint, [&](auto jac, auto dik, auto man, auto man_jvp) {
    auto go = [&](auto op) {
      using Op = decltype(op);
      rc = L.dtype == 0 ? launch_task_t<Op, double>(L, q, P, y0, y1, status, dq)
                        : launch_task_t<Op, float>(L, q, P, y0, y1, status, dq);
    };
    if (which == 0) go(jac);
    else if (which == 1) go(dik);
    else if (which == 2) go(man);
    else if (which == 4) go(man_jvp);
  });
  return rc;
}

// Jacobian / diff-IK / manipulability on a generated frame joint.  chain7
// `ee` (tools/async_sweep.cu "jac", 4M states): geometric Jacobian + pose
// fp64 1.55 -> 0.39 ms, fp32 1.13 -> 0.37 ms against the template kernel.
int launch_gen_task(const Launch& L, int which, int frame_joint, const TaskShared& P, const void* q, void* y0,
                    void* y1, int32_t* status, const void* dq) {
  if (L.spec == kTree29) return gen_task_t<GenTree29>(L, which, frame_joint, P, q, y0, y1, status, dq);
  if (L.spec == kChain7) return gen_task_t<GenChain7>(L, which, frame_joint, P, q, y0, y1, status, dq);
  return -1;
}

int launch_gen_crba(const Launch& L, const void* q, void* M) {
  if (L.spec != kTree29) return -1;
  return launch_op<GenTree29::Crba>(L, q, nullptr, nullptr, nullptr, M, nullptr);
}

int launch_gen_crba_packed(const Launch& L, const void* q, void* Mp) {
  if (L.spec == kTree29) return launch_op<GenTree29::CrbaPacked>(L, q, nullptr, nullptr, nullptr, Mp, nullptr);
  if (L.spec == kChain7) return launch_op<GenChain7::CrbaPacked>(L, q, nullptr, nullptr, nullptr, Mp, nullptr);
  return -1;
}

int launch_gen_fk(const Launch& L, const void* q, void* frames) {
  if (L.spec != kTree29) return -1;
  return launch_op<GenTree29::Fk>(L, q, nullptr, nullptr, nullptr, frames, nullptr);
}

}  // namespace vdk
