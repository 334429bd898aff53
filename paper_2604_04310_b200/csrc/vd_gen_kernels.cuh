// Kernels around the generated straight-line per-robot routines
// (vd_gen_robots.cuh, tools/gen_tree_kernels.py).
//
// One thread = one robot state, persistent grid (one wave of resident CTAs,
// each thread strides over the batch).  The generated ABA hands its
// pass-2 -> pass-3 state (per joint U/D, u/D and cos/sin or q) to the context
// by slot number; slot k lives
//   * in registers     when k >= kSlots - kReg  (stored last, read first: the
//                       root chain of the tree),
//   * in shared memory when k <  kSmem           ([k][thread] layout),
//   * otherwise in a global scratch slab [k - kSmem][thread slot] that a
//     persistent grid re-uses for every state it processes, so it stays
//     resident in L2 (footprint = resident threads x slots).
// Loads/stores are SoA-coalesced (element (i, k) at k*ld + i).
#pragma once

#include <cuda_runtime.h>

#include "vd_gen_prelude.cuh"
#include "vd_launch.hpp"
#include "vd_shared.hpp"

namespace vdk {

constexpr int kGenBlock = 128;

// Opaque state ops: a value written through st() must really go to its slot
// (plain C++ stores would be forwarded to the matching loads, keeping every
// value live in registers).  Inputs are read once each (prologue / pass 2), so
// they are plain read-only loads the scheduler may hoist.
template <class T>
struct GenMem;
template <>
struct GenMem<double> {
  static __device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
  static __device__ __forceinline__ void stg(double* p, double v) {
    asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v));
  }
  static __device__ __forceinline__ double ldgs(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
  static __device__ __forceinline__ void sts(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
  static __device__ __forceinline__ double lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
  }
};
template <>
struct GenMem<float> {
  static __device__ __forceinline__ float ldg(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ void stg(float* p, float v) { asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v)); }
  static __device__ __forceinline__ float ldgs(const float* p) {
    float v;
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
  }
  static __device__ __forceinline__ void sts(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }
  static __device__ __forceinline__ float lds(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
  }
};

// kStream: state inputs are read and outputs written with the evict-first
// (.cs) cache operator, so the streamed batch does not push the per-thread
// scratch slab out of L2 (gen_sweep: G1 ABA fp64 0.31-0.42 -> 0.29 ms, dense
// CRBA 1.1-1.8x; it slows the OSC routines, which keep the default).
// kSyncEvery > 0: a CTA barrier at every kSyncEvery-th phase point of the
// generated routine (one per joint step), so the CTA's warps walk the
// straight-line code together and share its instruction-cache lines.
template <class T, int kSlots, int kReg, int kSmem, int kFast = kTrigLib, bool kStream = false, int kSyncEvery = 0,
          int kBlk = kGenBlock>
struct GenCx {
  static constexpr int kFastTrig = kFast;  // kTrigLib / kTrigFast / kTrigCall (vd_gen_prelude.cuh)
  static constexpr int kGlobal = kSlots - kReg - kSmem > 0 ? kSlots - kReg - kSmem : 0;
  const T* in_[3];  // &x_g[i]; element (i, j) of input g at in_[g][j * ld]
  T* out_;          // &y[i]; element (i, k) at out_[k * ldo]
  const T* fx_;     // &fext[i] (NULL: no external wrenches); plane 6 j + k at fx_[(6 j + k) * ld]
  const T* gp_ = nullptr;  // &gravity_planes[i] (NULL: g3); a_g component k at gp_[k * ld]
  T* sb;            // this thread's scratch: slot k at sb[(k - kSmem) * 32] (warp-interleaved)
  uint32_t sm;      // shared address of slot 0 for this thread ([k][threadIdx.x])
  int64_t ld, ldo;
  bool active;      // false on the padding lanes of the last round (they compute, but write nothing)
  T g3[3];
  T reg[kReg > 0 ? kReg : 1];
  __device__ __forceinline__ T x(int g, int j) const {
    if constexpr (kStream) return __ldcs(in_[g] + j * ld);
    else return GenMem<T>::ldg(in_[g] + j * ld);
  }
  __device__ __forceinline__ T fx(int k) const {
    if constexpr (kStream) return __ldcs(fx_ + k * ld);
    else return GenMem<T>::ldg(fx_ + k * ld);
  }
  __device__ __forceinline__ void prefetch(int g, int j) const {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(in_[g] + j * ld));
  }
  // every read of input group g for this state is done (GenAsyncCx overrides)
  __device__ __forceinline__ void fetch_next(int) const {}
  template <int K>
  __device__ __forceinline__ void phase() const {
    if constexpr (kSyncEvery > 0) {
      if constexpr (K % kSyncEvery == 0) __syncthreads();
    }
  }
  __device__ __forceinline__ T g(int k) const {
    if (gp_) {
      if constexpr (kStream) return __ldcs(gp_ + k * ld);
      else return GenMem<T>::ldg(gp_ + k * ld);
    }
    return g3[k];
  }
  __device__ __forceinline__ void st(int k, T v) {
    if (k >= kSlots - kReg) reg[k - (kSlots - kReg)] = v;
    else if (k < kSmem) GenMem<T>::sts(sm + (uint32_t)(k * kBlk * sizeof(T)), v);
    else GenMem<T>::stg(sb + (k - kSmem) * 32, v);
  }
  __device__ __forceinline__ T get(int k) const {
    if (k >= kSlots - kReg) return reg[k - (kSlots - kReg)];
    if (k < kSmem) return GenMem<T>::lds(sm + (uint32_t)(k * kBlk * sizeof(T)));
    return GenMem<T>::ldgs(sb + (k - kSmem) * 32);
  }
  // a double in slots k, k + 1 (mixed-precision joints of the fp32 routines;
  // one slot when T is double)
  __device__ __forceinline__ void st2(int k, double v) {
    if constexpr (sizeof(T) == 8) {
      st(k, v);
    } else {
      st(k, __int_as_float(__double2loint(v)));
      st(k + 1, __int_as_float(__double2hiint(v)));
    }
  }
  __device__ __forceinline__ double get2(int k) const {
    if constexpr (sizeof(T) == 8) return get(k);
    else return __hiloint2double(__float_as_int(get(k + 1)), __float_as_int(get(k)));
  }
  __device__ __forceinline__ void y(int, int k, T v) const {
    if constexpr (kStream) {
      if (active) __stcs(out_ + k * ldo, v);
    } else {
      if (active) out_[k * ldo] = v;
    }
  }
};

// Scratch elements per resident thread (0 when every slot is on chip).
template <class Op, class T, int kReg, int kSmem>
constexpr int64_t gen_scratch_per_thread() {
  return GenCx<T, Op::kSlots, kReg, kSmem>::kGlobal;
}

// One generated routine (Op = GenRobot::Aba / Rnea / RneaBias / RneaGrav /
// Crba / Fk) over a persistent grid: every thread strides over the batch.
template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast = kTrigLib, bool kStream = false,
          int kSyncEvery = 0, int kBlk = kGenBlock>
__global__ void __launch_bounds__(kBlk, kMinB)
    k_gen(int64_t N, const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2, int64_t ldi,
          T g0, T g1, T g2, T* __restrict__ y, int64_t ldo, int32_t* __restrict__ status, T* __restrict__ scratch,
          const T* __restrict__ fext, const T* __restrict__ gpl) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenCx<T, Op::kSlots, kReg, kSmem, kFast, kStream, kSyncEvery, kBlk>;
  Cx cx;
  const int64_t slot = (int64_t)blockIdx.x * kBlk + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kBlk;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  cx.g3[0] = g0;
  cx.g3[1] = g1;
  cx.g3[2] = g2;
  for (int64_t base = (int64_t)blockIdx.x * kBlk; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    // launder the strides each round so the per-column addresses are not
    // hoisted out of the loop (n x 3 live 64-bit addresses otherwise spill)
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    cx.in_[0] = x0 + i;
    cx.in_[1] = (Op::kIn > 1 ? x1 : x0) + i;
    cx.in_[2] = (Op::kIn > 2 ? x2 : x0) + i;
    cx.out_ = y + i;
    cx.fx_ = fext ? fext + i : nullptr;
    cx.gp_ = gpl ? gpl + i : nullptr;
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) y[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
}

// k_gen with the routine called out of line once per state (Cfg::kCall).
// A routine that reads its constants from the robot's __constant__ table
// (codegen POOL_OPS) needs this: inside the persistent loop the compiler
// hoists every table read out of the loop into registers (and spills them);
// in the per-state function there is no loop, so the reads become
// constant-bank operands of the DFMAs (G1 ABA fp64 0.261 -> 0.242 ms,
// tools/call_sweep.cu).
template <class Op, class T, int kReg, int kSmem, int kFast, bool kStream>
__device__ __noinline__ bool gen_state(const T* x0, const T* x1, const T* x2, const T* fx, const T* gp, int64_t ld,
                                       T* y, int64_t ldo, bool active, T* sb, uint32_t sm, T g0, T g1, T g2) {
  GenCx<T, Op::kSlots, kReg, kSmem, kFast, kStream> cx;
  cx.in_[0] = x0;
  cx.in_[1] = x1;
  cx.in_[2] = x2;
  cx.fx_ = fx;
  cx.gp_ = gp;
  cx.out_ = y;
  cx.ld = ld;
  cx.ldo = ldo;
  cx.active = active;
  cx.sb = sb;
  cx.sm = sm;
  cx.g3[0] = g0;
  cx.g3[1] = g1;
  cx.g3[2] = g2;
  return Op::template run<T>(cx);
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast = kTrigLib, bool kStream = false>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_call(int64_t N, const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2, int64_t ldi,
               T g0, T g1, T g2, T* __restrict__ y, int64_t ldo, int32_t* __restrict__ status,
               T* __restrict__ scratch, const T* __restrict__ fext, const T* __restrict__ gpl) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenCx<T, Op::kSlots, kReg, kSmem, kFast, kStream>;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  T* sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  const uint32_t sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    const bool active = i0 < N;
    const int64_t i = active ? i0 : N - 1;
    const bool ok = gen_state<Op, T, kReg, kSmem, kFast, kStream>(
        x0 + i, (Op::kIn > 1 ? x1 : x0) + i, (Op::kIn > 2 ? x2 : x0) + i, fext ? fext + i : nullptr,
        gpl ? gpl + i : nullptr, ldi, y + i, ldo, active, sb, sm, g0, g1, g2);
    if (active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) y[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
}

// Asynchronous state input.  The inputs of the state a thread processes next
// are copied global -> shared memory with per-thread cp.async (no CTA barrier:
// each thread reads only the elements it copied) while it computes the current
// state.  A generated routine calls fetch_next(g) once its reads of group g are
// done, so the copy of the next state's group g overlaps the rest of the
// routine: the next state starts with q and q̇ on chip, and the ABA's τ (read
// in pass 2, released before pass 3) is never waited for.  ncu of the plain
// kernel (chain7 ABA fp64): 30 % of the warp-stall samples were long-scoreboard
// waits on exactly these loads (profiles/README.md).
// Shared memory per thread: kSmem slots, then kIn × kDof input elements
// ([k][thread] layout, conflict-free).
// kStream: the copies carry an L2 evict-first policy (as GenCx's .cs loads).
template <bool kStream, class T>
__device__ __forceinline__ void vd_cp_async(uint32_t dst, const T* src, uint64_t pol) {
  if constexpr (kStream)
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(sizeof(T)),
                 "l"(pol)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(src), "n"(sizeof(T)) : "memory");
}

template <class T, int kSlots, int kReg, int kSmem, int kFast, bool kStream, int kDof, int kSyncEvery = 0>
struct GenAsyncCx : GenCx<T, kSlots, kReg, kSmem, kFast, kStream, kSyncEvery> {
  uint32_t ib;     // shared address of this thread's input element (0, 0)
  const T* nx[3];  // &x_g[next state]
  uint64_t pol;    // L2 evict-first policy (kStream)
  static __device__ __forceinline__ uint32_t off(int g, int j) {
    return (uint32_t)((g * kDof + j) * kGenBlock * (int)sizeof(T));
  }
  __device__ __forceinline__ T x(int g, int j) const { return GenMem<T>::lds(ib + off(g, j)); }
  __device__ __forceinline__ void fetch_next(int g) const { fetch(ib, nx[g], this->ld, g, pol); }
  // the call's a_g only: per-state gravity runs k_gen (launch_t)
  __device__ __forceinline__ T g(int k) const { return this->g3[k]; }
  static __device__ __forceinline__ void fetch(uint32_t ib, const T* src, int64_t ld, int g, uint64_t pol) {
#pragma unroll
    for (int j = 0; j < kDof; ++j) vd_cp_async<kStream>(ib + off(g, j), src + j * ld, pol);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
};

template <class Op, class T, int kReg, int kSmem>
constexpr size_t gen_async_smem() {
  return (size_t)(kSmem + Op::kIn * Op::kDof) * kGenBlock * sizeof(T);
}

// k_gen with asynchronous state input (same arguments, same results; gpl must
// be NULL: launch_t sends per-state gravity to k_gen).
template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast = kTrigLib, bool kStream = false,
          int kSyncEvery = 0>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_async(int64_t N, const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2, int64_t ldi,
                T g0, T g1, T g2, T* __restrict__ y, int64_t ldo, int32_t* __restrict__ status,
                T* __restrict__ scratch, const T* __restrict__ fext, const T* __restrict__ gpl) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenAsyncCx<T, Op::kSlots, kReg, kSmem, kFast, kStream, Op::kDof, kSyncEvery>;
  Cx cx;
  cx.pol = 0;
  if constexpr (kStream) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(cx.pol));
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  cx.ib = cx.sm + (uint32_t)(kSmem * kGenBlock * sizeof(T));
  cx.g3[0] = g0;
  cx.g3[1] = g1;
  cx.g3[2] = g2;
  const T* xs[3] = {x0, Op::kIn > 1 ? x1 : x0, Op::kIn > 2 ? x2 : x0};
  // the first state's inputs (padding lanes of the last round read state N-1)
  {
    const int64_t i = slot < N ? slot : N - 1;
#pragma unroll
    for (int g = 0; g < Op::kIn; ++g) Cx::fetch(cx.ib, xs[g] + i, ldi, g, cx.pol);
  }
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    const int64_t inext = i0 + stride < N ? i0 + stride : N - 1;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      cx.in_[g] = xs[g] + i;
      cx.nx[g] = xs[g] + inext;
    }
    cx.out_ = y + i;
    cx.fx_ = fext ? fext + i : nullptr;
    asm volatile("cp.async.wait_all;" ::: "memory");
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) y[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // no copy outlives the CTA
}

// osc_step context: task parameters (OscShared, kernel parameter space) and
// a second output (Λ, 36 planes, optional).
template <class T, int kSlots, int kReg, int kSmem, int kTrig = kTrigLib>
struct GenOscCx : GenCx<T, kSlots, kReg, kSmem, kTrig> {
  const OscShared* P;
  T* out1_;  // &Λ[i] or nullptr
  __device__ __forceinline__ T g(int k) const { return T(P->gravity[k]); }
  __device__ __forceinline__ T fR(int k) const { return T(P->frame_R[k]); }
  __device__ __forceinline__ T fp(int k) const { return T(P->frame_p[k]); }
  __device__ __forceinline__ T tR(int k) const { return T(P->target_R[k]); }
  __device__ __forceinline__ T tp(int k) const { return T(P->target_p[k]); }
  __device__ __forceinline__ T kp(int k) const { return T(P->kp[k]); }
  __device__ __forceinline__ T kd(int k) const { return T(P->kd[k]); }
  __device__ __forceinline__ T aff(int k) const { return T(P->accel_ff[k]); }
  __device__ __forceinline__ T pkp() const { return T(P->posture_kp); }
  __device__ __forceinline__ T pkd() const { return T(P->posture_kd); }
  __device__ __forceinline__ T eps() const { return T(P->epsilon); }
  __device__ __forceinline__ T post(int k) const { return T(P->posture[k]); }
  __device__ __forceinline__ bool want_lambda() const { return out1_ != nullptr; }
  __device__ __forceinline__ void y(int o, int k, T v) const {
    if (this->active) (o == 0 ? this->out_ : out1_)[k * this->ldo] = v;
  }
};

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig = kTrigLib>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_osc(int64_t N, const T* __restrict__ q, const T* __restrict__ qd, int64_t ldi,
              const __grid_constant__ OscShared P, T* __restrict__ tau, T* __restrict__ lam, int64_t ldo,
              int32_t* __restrict__ status, T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenOscCx<T, Op::kSlots, kReg, kSmem, kTrig>;
  Cx cx;
  cx.P = &P;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    cx.in_[0] = q + i;
    cx.in_[1] = qd + i;
    cx.in_[2] = q + i;
    cx.out_ = tau + i;
    cx.out1_ = lam ? lam + i : nullptr;
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) tau[(int64_t)j * ldo + i] = T(0);
        if (lam)
          for (int j = 0; j < 36; ++j) lam[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
}

// k_gen with double-buffered asynchronous state input (Cfg::kDb):
// state s reads its inputs from shared buffer s & 1 while the cp.async copies
// of state s + 1 (every input group) land in the other, issued as state s
// starts; the routine's fetch_next release points are not used.  Shared
// memory per thread: kSmem slots, then 2 × kIn × kDof inputs.
template <class T, int kSlots, int kReg, int kSmem, int kFast, bool kStream, int kDof>
struct GenDbCx : GenCx<T, kSlots, kReg, kSmem, kFast, kStream> {
  uint32_t ib;
  static __device__ __forceinline__ uint32_t off(int g, int j) {
    return (uint32_t)((g * kDof + j) * kGenBlock * (int)sizeof(T));
  }
  __device__ __forceinline__ T x(int g, int j) const { return GenMem<T>::lds(ib + off(g, j)); }
  __device__ __forceinline__ T g(int k) const { return this->g3[k]; }
};

template <class Op, class T, int kSmem>
constexpr size_t gen_db_smem() {
  return (size_t)(kSmem + 2 * Op::kIn * Op::kDof) * kGenBlock * sizeof(T);
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kFast = kTrigLib, bool kStream = false>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_db(int64_t N, const T* __restrict__ x0, const T* __restrict__ x1, const T* __restrict__ x2, int64_t ldi,
             T g0, T g1, T g2, T* __restrict__ y, int64_t ldo, int32_t* __restrict__ status, T* __restrict__ scratch,
             const T* __restrict__ fext, const T* __restrict__) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenDbCx<T, Op::kSlots, kReg, kSmem, kFast, kStream, Op::kDof>;
  Cx cx;
  uint64_t pol = 0;
  if constexpr (kStream) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  cx.g3[0] = g0;
  cx.g3[1] = g1;
  cx.g3[2] = g2;
  cx.gp_ = nullptr;
  const uint32_t ib0 = cx.sm + (uint32_t)(kSmem * kGenBlock * sizeof(T));
  const uint32_t ib1 = ib0 + (uint32_t)(Op::kIn * Op::kDof * kGenBlock * sizeof(T));
  const T* xs[3] = {x0, Op::kIn > 1 ? x1 : x0, Op::kIn > 2 ? x2 : x0};
  auto fetch = [&](uint32_t buf, int64_t i) {
#pragma unroll
    for (int g = 0; g < Op::kIn; ++g)
#pragma unroll
      for (int j = 0; j < Op::kDof; ++j) vd_cp_async<kStream>(buf + Cx::off(g, j), xs[g] + i + j * ldi, pol);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  fetch(ib0, slot < N ? slot : N - 1);
  int buf = 0;
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride, buf ^= 1) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (base + stride < N) fetch(buf ? ib0 : ib1, i0 + stride < N ? i0 + stride : N - 1);
    cx.ib = buf ? ib1 : ib0;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    cx.in_[0] = xs[0] + i;
    cx.in_[1] = xs[1] + i;
    cx.in_[2] = xs[2] + i;
    cx.out_ = y + i;
    cx.fx_ = fext ? fext + i : nullptr;  // external wrenches stay global reads
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) y[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// k_gen_osc with double-buffered asynchronous state input (OscCfg::kAsync):
// the OSC routine reads q again at its end (posture torque), so the
// single-buffer release scheme of k_gen_async would start the next state's
// q copy only then.  Here state s reads its q, q̇ from shared buffer s & 1
// while the copies of state s + 1 land in the other buffer, issued as state
// s starts.  Shared memory per thread: kSmem slots, then 2 × 2 × kDof inputs.
template <class T, int kSlots, int kReg, int kSmem, int kTrig, int kDof>
struct GenOscDbCx : GenOscCx<T, kSlots, kReg, kSmem, kTrig> {
  uint32_t ib;  // shared address of this state's input element (0, 0)
  static __device__ __forceinline__ uint32_t off(int g, int j) {
    return (uint32_t)((g * kDof + j) * kGenBlock * (int)sizeof(T));
  }
  __device__ __forceinline__ T x(int g, int j) const { return GenMem<T>::lds(ib + off(g, j)); }
  static __device__ __forceinline__ void fetch(uint32_t buf, const T* q, const T* qd, int64_t ld) {
#pragma unroll
    for (int j = 0; j < kDof; ++j) vd_cp_async<false>(buf + off(0, j), q + j * ld, 0);
#pragma unroll
    for (int j = 0; j < kDof; ++j) vd_cp_async<false>(buf + off(1, j), qd + j * ld, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
};

template <class Op, class T, int kSmem>
constexpr size_t gen_osc_db_smem() {
  return (size_t)(kSmem + 4 * Op::kDof) * kGenBlock * sizeof(T);
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig = kTrigLib>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_osc_db(int64_t N, const T* __restrict__ q, const T* __restrict__ qd, int64_t ldi,
                 const __grid_constant__ OscShared P, T* __restrict__ tau, T* __restrict__ lam, int64_t ldo,
                 int32_t* __restrict__ status, T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenOscDbCx<T, Op::kSlots, kReg, kSmem, kTrig, Op::kDof>;
  Cx cx;
  cx.P = &P;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  const uint32_t ib0 = cx.sm + (uint32_t)(kSmem * kGenBlock * sizeof(T));
  const uint32_t ib1 = ib0 + (uint32_t)(2 * Op::kDof * kGenBlock * sizeof(T));
  {
    const int64_t i = slot < N ? slot : N - 1;
    Cx::fetch(ib0, q + i, qd + i, ldi);
  }
  int buf = 0;
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride, buf ^= 1) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    asm volatile("cp.async.wait_all;" ::: "memory");
    // the next state's inputs into the other buffer (its previous reader,
    // state s - 1, has finished)
    if (base + stride < N) {
      const int64_t inext = i0 + stride < N ? i0 + stride : N - 1;
      Cx::fetch(buf ? ib0 : ib1, q + inext, qd + inext, ldi);
    }
    cx.ib = buf ? ib1 : ib0;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    cx.in_[0] = q + i;
    cx.in_[1] = qd + i;
    cx.in_[2] = q + i;
    cx.out_ = tau + i;
    cx.out1_ = lam ? lam + i : nullptr;
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) tau[(int64_t)j * ldo + i] = T(0);
        if (lam)
          for (int j = 0; j < 36; ++j) lam[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// k_gen_osc with the routine called out of line once per state (OscCfg::kCall;
// see k_gen_call): a routine that reads its model constants from the robot's
// __constant__ table (codegen POOL_OPS) gets them as constant-bank operands.
template <class Op, class T, int kReg, int kSmem, int kTrig>
__device__ __noinline__ bool gen_osc_state(const OscShared* P, const T* q, const T* qd, int64_t ld, T* tau, T* lam,
                                           int64_t ldo, bool active, T* sb, uint32_t sm) {
  GenOscCx<T, Op::kSlots, kReg, kSmem, kTrig> cx;
  cx.P = P;
  cx.in_[0] = q;
  cx.in_[1] = qd;
  cx.in_[2] = q;
  cx.out_ = tau;
  cx.out1_ = lam;
  cx.ld = ld;
  cx.ldo = ldo;
  cx.active = active;
  cx.sb = sb;
  cx.sm = sm;
  return Op::template run<T>(cx);
}

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig = kTrigLib>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_osc_call(int64_t N, const T* __restrict__ q, const T* __restrict__ qd, int64_t ldi,
                   const __grid_constant__ OscShared P, T* __restrict__ tau, T* __restrict__ lam, int64_t ldo,
                   int32_t* __restrict__ status, T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenOscCx<T, Op::kSlots, kReg, kSmem, kTrig>;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  T* sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  const uint32_t sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    const bool active = i0 < N;
    const int64_t i = active ? i0 : N - 1;
    const bool ok = gen_osc_state<Op, T, kReg, kSmem, kTrig>(&P, q + i, qd + i, ldi, tau + i, lam ? lam + i : nullptr,
                                                             ldo, active, sb, sm);
    if (active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) tau[(int64_t)j * ldo + i] = T(0);
        if (lam)
          for (int j = 0; j < 36; ++j) lam[(int64_t)j * ldo + i] = T(0);
      }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
}

// Fused forward-dynamics context (GenRobot::Dyn): output group 0 = M (n²
// planes), 1 = bias (n), 2 = q̈ (n); a NULL group is not written.
template <class T, int kSlots, int kReg, int kSmem, int kTrig = kTrigLib, bool kStream = false>
struct GenDynCx : GenCx<T, kSlots, kReg, kSmem, kTrig, kStream> {
  T* outs_[3];
  __device__ __forceinline__ void y(int o, int k, T v) const {
    T* p = outs_[o];
    if (this->active && p) {
      if constexpr (kStream) __stcs(p + k * this->ldo, v);
      else p[k * this->ldo] = v;
    }
  }
};

template <class Op, class T, int kReg, int kSmem, int kMinB, int kTrig = kTrigLib, bool kStream = false>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_dyn(int64_t N, const T* __restrict__ q, const T* __restrict__ qd, const T* __restrict__ tau, int64_t ldi,
              T g0, T g1, T g2, T* __restrict__ M, T* __restrict__ bias, T* __restrict__ qdd, int64_t ldo,
              int32_t* __restrict__ status, T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenDynCx<T, Op::kSlots, kReg, kSmem, kTrig, kStream>;
  Cx cx;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  cx.g3[0] = g0;
  cx.g3[1] = g1;
  cx.g3[2] = g2;
  cx.fx_ = nullptr;
  cx.gp_ = nullptr;
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    cx.in_[0] = q + i;
    cx.in_[1] = qd + i;
    cx.in_[2] = tau + i;
    cx.out_ = nullptr;
    cx.outs_[0] = M ? M + i : nullptr;
    cx.outs_[1] = bias ? bias + i : nullptr;
    cx.outs_[2] = qdd ? qdd + i : nullptr;
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok && qdd)
        for (int j = 0; j < Op::kDof; ++j) qdd[(int64_t)j * ldo + i] = T(0);
      if (status) status[i] = ok ? 0 : 7;
    }
  }
}

// Forward-mode JVP context (JvpArgs): NULL primal inputs read as 0, NULL
// tangents as 0; output group 0 = values, 1 = tangents (either may be NULL).
template <class T, int kSlots, int kReg, int kSmem, bool kStream = false, int kTrig = kTrigLib>
struct GenJvpCx : GenCx<T, kSlots, kReg, kSmem, kTrig> {
  const T* din_[3];
  T* dout_;
  static __device__ __forceinline__ T ld_(const T* p) {
    if constexpr (kStream) return __ldcs(p);
    else return GenMem<T>::ldg(p);
  }
  __device__ __forceinline__ T x(int g, int j) const { return this->in_[g] ? ld_(this->in_[g] + j * this->ld) : T(0); }
  __device__ __forceinline__ T dx(int g, int j) const { return din_[g] ? ld_(din_[g] + j * this->ld) : T(0); }
  __device__ __forceinline__ T g(int k) const { return this->g3[k]; }
  __device__ __forceinline__ void y(int o, int k, T v) const {
    T* p = o == 0 ? this->out_ : dout_;
    if (this->active && p) {
      if constexpr (kStream) __stcs(p + k * this->ldo, v);
      else p[k * this->ldo] = v;
    }
  }
};

template <class Op, class T, int kReg, int kSmem, int kMinB, bool kStream = false, int kTrig = kTrigLib>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_jvp(int64_t N, const __grid_constant__ JvpArgs a, int64_t ldi, int64_t ldo, T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenJvpCx<T, Op::kSlots, kReg, kSmem, kStream, kTrig>;
  Cx cx;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  for (int k = 0; k < 3; ++k) cx.g3[k] = T(a.g[k]);
  T* out = (T*)a.out;
  T* dout = (T*)a.dout;
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    for (int k = 0; k < 3; ++k) {
      cx.in_[k] = a.x[k] ? (const T*)a.x[k] + i : nullptr;
      cx.din_[k] = a.dx[k] ? (const T*)a.dx[k] + i : nullptr;
    }
    cx.out_ = out ? out + i : nullptr;
    cx.dout_ = dout ? dout + i : nullptr;
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) {
          if (out) out[(int64_t)j * ldo + i] = T(0);
          if (dout) dout[(int64_t)j * ldo + i] = T(0);
        }
      }
      if (a.status) a.status[i] = ok ? 0 : 7;
    }
  }
}

// k_gen_jvp with the routine out of line once per state (JvpCfg::kCall; see
// k_gen_call).
template <class Op, class T, int kReg, int kSmem, bool kStream, int kTrig>
__device__ __noinline__ bool gen_jvp_state(const JvpArgs* a, int64_t i, int64_t ld, int64_t ldo, bool active, T* sb,
                                           uint32_t sm) {
  GenJvpCx<T, Op::kSlots, kReg, kSmem, kStream, kTrig> cx;
  cx.sb = sb;
  cx.sm = sm;
  for (int k = 0; k < 3; ++k) cx.g3[k] = T(a->g[k]);
  cx.active = active;
  cx.ld = ld;
  cx.ldo = ldo;
  for (int k = 0; k < 3; ++k) {
    cx.in_[k] = a->x[k] ? (const T*)a->x[k] + i : nullptr;
    cx.din_[k] = a->dx[k] ? (const T*)a->dx[k] + i : nullptr;
  }
  cx.out_ = a->out ? (T*)a->out + i : nullptr;
  cx.dout_ = a->dout ? (T*)a->dout + i : nullptr;
  return Op::template run<T>(cx);
}

template <class Op, class T, int kReg, int kSmem, int kMinB, bool kStream = false, int kTrig = kTrigLib>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_jvp_call(int64_t N, const __grid_constant__ JvpArgs a, int64_t ldi, int64_t ldo, T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenJvpCx<T, Op::kSlots, kReg, kSmem, kStream, kTrig>;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  T* sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  const uint32_t sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  T* out = (T*)a.out;
  T* dout = (T*)a.dout;
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    const bool active = i0 < N;
    const int64_t i = active ? i0 : N - 1;
    const bool ok = gen_jvp_state<Op, T, kReg, kSmem, kStream, kTrig>(&a, i, ldi, ldo, active, sb, sm);
    if (active) {
      if (!ok) {
        for (int j = 0; j < Op::kOut; ++j) {
          if (out) out[(int64_t)j * ldo + i] = T(0);
          if (dout) dout[(int64_t)j * ldo + i] = T(0);
        }
      }
      if (a.status) a.status[i] = ok ? 0 : 7;
    }
  }
}

// Task-space context (Jacobian / diff-IK / manipulability): TaskShared in
// kernel parameter space, two nullable output groups.
template <class T, int kSlots, int kReg, int kSmem>
struct GenTaskCx : GenCx<T, kSlots, kReg, kSmem> {
  const TaskShared* P;
  T* out1_;
  const T* din_;  // &dq[i] (the ManipJvp tangent; NULL = 0)
  __device__ __forceinline__ T dx(int, int j) const { return din_ ? GenMem<T>::ldg(din_ + j * this->ld) : T(0); }
  __device__ __forceinline__ T fR(int k) const { return T(P->frame_R[k]); }
  __device__ __forceinline__ T fp(int k) const { return T(P->frame_p[k]); }
  __device__ __forceinline__ T tR(int k) const { return T(P->target_R[k]); }
  __device__ __forceinline__ T tp(int k) const { return T(P->target_p[k]); }
  __device__ __forceinline__ T kp(int k) const { return T(P->kp[k]); }
  __device__ __forceinline__ T tw(int k) const { return T(P->twist_ff[k]); }
  __device__ __forceinline__ T damp() const { return T(P->damping); }
  __device__ __forceinline__ void y(int o, int k, T v) const {
    T* p = o == 0 ? this->out_ : out1_;
    if (this->active && p) p[k * this->ldo] = v;
  }
};

template <class Op, class T, int kReg, int kSmem, int kMinB>
__global__ void __launch_bounds__(kGenBlock, kMinB)
    k_gen_task(int64_t N, const T* __restrict__ q, int64_t ldi, const __grid_constant__ TaskShared P,
               T* __restrict__ y0, T* __restrict__ y1, int64_t ldo, int32_t* __restrict__ status,
               T* __restrict__ scratch, const T* __restrict__ dq) {
  extern __shared__ __align__(16) unsigned char vd_gen_smem[];
  using Cx = GenTaskCx<T, Op::kSlots, kReg, kSmem>;
  Cx cx;
  cx.P = &P;
  const int64_t slot = (int64_t)blockIdx.x * kGenBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kGenBlock;
  cx.sb = scratch + (slot >> 5) * (int64_t)(Cx::kGlobal * 32) + (slot & 31);
  cx.sm = (uint32_t)__cvta_generic_to_shared(vd_gen_smem) + threadIdx.x * (uint32_t)sizeof(T);
  for (int64_t base = (int64_t)blockIdx.x * kGenBlock; base < N; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    cx.active = i0 < N;
    const int64_t i = cx.active ? i0 : N - 1;
    int64_t ld, lo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ld) : "l"(ldi));
    asm volatile("mov.b64 %0, %1;" : "=l"(lo) : "l"(ldo));
    cx.ld = ld;
    cx.ldo = lo;
    cx.in_[0] = cx.in_[1] = cx.in_[2] = q + i;
    cx.din_ = dq ? dq + i : nullptr;
    cx.out_ = y0 ? y0 + i : nullptr;
    cx.out1_ = y1 ? y1 + i : nullptr;
    const bool ok = Op::template run<T>(cx);
    if (cx.active) {
      if (!ok)
        for (int j = 0; j < Op::kOut; ++j) {
          if (y0) y0[(int64_t)j * ldo + i] = T(0);
          if (dq && y1) y1[(int64_t)j * ldo + i] = T(0);  // ManipJvp: the tangent too
        }
      if (status) status[i] = ok ? 0 : 7;
    }
  }
}

}  // namespace vdk
