// Launch machinery of the generated straight-line routines, shared by the
// library's instantiation unit (vd_inst_gen.cu) and the per-model JIT
// translation units (vd_jit_entry.cuh): per-(op, dtype) placement config,
// occupancy cache, the persistent-grid launch with its L2 scratch slab.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <utility>

#include "vd_gen_kernels.cuh"
#include "vd_launch.hpp"

namespace vdk {

// Slot placement and CTAs/SM per (op, dtype), from ablib/gen_sweep*.cu on a
// B200 (kReg: last slots kept in registers; kSmem: first slots in shared
// memory; the rest in the L2-resident scratch slab).
template <class Op, class T>
struct Cfg {
  static constexpr int kReg = 0, kSmem = Op::kSlots < 55 ? Op::kSlots : 55, kMinB = sizeof(T) == 8 ? 3 : 4;
  // sin/cos evaluation (vd_gen_prelude.cuh): the large-state routines of
  // robots with >= 20 joints (ABA / RNEA families of JIT models) call one
  // out-of-line copy, the measured win for the G1 ABA / RNEA
  static constexpr int kFast = Op::kDof >= 20 && Op::kSlots >= 80 ? kTrigCall : kTrigLib;
};
// kStream (GenCx): evict-first state I/O; false unless a Cfg sets it
template <class C, class = void>
struct StreamIo : std::false_type {};
template <class C>
struct StreamIo<C, std::void_t<decltype(C::kStream)>> : std::bool_constant<C::kStream> {};
// kAsync (k_gen_async): the next state's inputs are prefetched into shared
// memory with cp.async while the current one is computed; false unless a Cfg
// sets it
template <class C, class = void>
struct AsyncIo : std::false_type {};
template <class C>
struct AsyncIo<C, std::void_t<decltype(C::kAsync)>> : std::bool_constant<C::kAsync> {};
// kDb (k_gen_db): double-buffered asynchronous input, every group of the next
// state copied while the current one computes; false unless a Cfg sets it
template <class C, class = void>
struct DbIo : std::false_type {};
template <class C>
struct DbIo<C, std::void_t<decltype(C::kDb)>> : std::bool_constant<C::kDb> {};
struct Occ {
  int blocks_per_sm = 0, sms = 0;
};

inline bool debug_launches() {
  static const bool on = std::getenv("VD_DEBUG_LAUNCH") != nullptr;
  return on;
}

// Occupancy (and the dynamic shared-memory opt-in) once per device for each
// kernel instantiation; keyed by <Op, T, kVariant>, not by the kernel's
// function type (all kernels of one dtype share that).
template <class Op, class T, int kVariant = 0, class Kern>
Occ occupancy(Kern kern, size_t smem) {
  static std::mutex mu;
  static Occ occ[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Occ& c = occ[dev & 63];
  if (!c.blocks_per_sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.blocks_per_sm, kern, kGenBlock, smem);
    if (c.blocks_per_sm < 1) c.blocks_per_sm = 1;
  }
  return c;
}

// kCall (k_gen_call): the routine out of line once per state; false unless a Cfg sets it
template <class C, class = void>
struct CallIo : std::false_type {};
template <class C>
struct CallIo<C, std::void_t<decltype(C::kCall)>> : std::bool_constant<C::kCall> {};

// The kernel of a Cfg (kMode 0 k_gen, 1 k_gen_async, 2 k_gen_call, 3 k_gen_db).
template <class Op, class T, class C, int kMode>
constexpr auto gen_kernel() {
  if constexpr (kMode == 3)
    return k_gen_db<Op, T, C::kReg, C::kSmem, C::kMinB, C::kFast, StreamIo<C>::value>;
  else if constexpr (kMode == 1)
    return k_gen_async<Op, T, C::kReg, C::kSmem, C::kMinB, C::kFast, StreamIo<C>::value>;
  else if constexpr (kMode == 2)
    return k_gen_call<Op, T, C::kReg, C::kSmem, C::kMinB, C::kFast, StreamIo<C>::value>;
  else
    return k_gen<Op, T, C::kReg, C::kSmem, C::kMinB, C::kFast, StreamIo<C>::value>;
}

template <class Op, class T, int kMode>
int launch_gen(const Launch& L, const void* x0, const void* x1, const void* x2, const double* g3, void* y,
               int32_t* status, const void* fext) {
  using C = Cfg<Op, T>;
  constexpr bool kAsync = kMode == 1;
  auto kern = gen_kernel<Op, T, C, kMode>();
  constexpr size_t smem = kMode == 3 ? gen_db_smem<Op, T, C::kSmem>()
                         : kAsync  ? gen_async_smem<Op, T, C::kReg, C::kSmem>()
                                   : (size_t)C::kSmem * kGenBlock * sizeof(T);
  const Occ o = occupancy<Op, T, kMode>(kern, smem);
  const int64_t blocks = std::min<int64_t>((L.N + kGenBlock - 1) / kGenBlock, (int64_t)o.sms * o.blocks_per_sm);
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  if (debug_launches())
    std::fprintf(stderr, "[vd] k_gen%s slots %d reg %d smem %d: %d CTAs/SM x %d SMs, grid %lld, smem %zu B\n",
                 kMode == 1 ? "_async" : (kMode == 2 ? "_call" : ""), Op::kSlots, C::kReg, C::kSmem, o.blocks_per_sm, o.sms, (long long)blocks, smem);
  // L2-resident scratch for the slots that are neither in registers nor in
  // shared memory: one slab per resident thread, stream-ordered from the
  // library's private pool (scratch_alloc: no synchronisation, safe for
  // concurrent streams, bounded caching).
  const size_t scratch_bytes = (size_t)blocks * kGenBlock * gen_scratch_per_thread<Op, T, C::kReg, C::kSmem>() * sizeof(T);
  T* scratch = nullptr;
  if (scratch_bytes) {
    if (int rc = scratch_alloc(reinterpret_cast<void**>(&scratch), scratch_bytes, s)) return rc;
  }
  // gravity3 == NULL: GravitySpec::standard() (dynamics.hpp:39-50), as g3_of
  const T g0 = g3 ? T(g3[0]) : T(0), g1 = g3 ? T(g3[1]) : T(0), g2 = g3 ? T(g3[2]) : T(9.81);
  kern<<<(unsigned)blocks, kGenBlock, smem, s>>>(L.N, (const T*)x0, (const T*)x1, (const T*)x2, L.ld_in, g0, g1, g2,
                                                 (T*)y, L.ld_out, status, scratch, (const T*)fext,
                                                 (const T*)L.gravity_planes);
  cudaError_t e = cudaGetLastError();
  scratch_free(scratch, s);
  return (int)e;
}

// One generated routine over the batch.  Per-state gravity (L.gravity_planes)
// runs the plain kernel even where the Cfg asks for asynchronous input: the
// asynchronous kernel (the headline Panda ABA) carries no per-state gravity
// load at all.
template <class Op, class T>
int launch_t(const Launch& L, const void* x0, const void* x1, const void* x2, const double* g3, void* y,
             int32_t* status, const void* fext = nullptr) {
  if constexpr (DbIo<Cfg<Op, T>>::value) {
    if (!L.gravity_planes) return launch_gen<Op, T, 3>(L, x0, x1, x2, g3, y, status, fext);
  }
  if constexpr (AsyncIo<Cfg<Op, T>>::value) {
    if (!L.gravity_planes) return launch_gen<Op, T, 1>(L, x0, x1, x2, g3, y, status, fext);
  }
  if constexpr (CallIo<Cfg<Op, T>>::value) return launch_gen<Op, T, 2>(L, x0, x1, x2, g3, y, status, fext);
  return launch_gen<Op, T, 0>(L, x0, x1, x2, g3, y, status, fext);
}

template <class Op>
int launch_op(const Launch& L, const void* x0, const void* x1, const void* x2, const double* g3, void* y,
              int32_t* status, const void* fext = nullptr) {
  return L.dtype == 0 ? launch_t<Op, double>(L, x0, x1, x2, g3, y, status, fext)
                      : launch_t<Op, float>(L, x0, x1, x2, g3, y, status, fext);
}


// OSC on branched trees: the articulated-body form (gen_osc_aba, ~255 slots
// for a G1 hand/foot frame instead of the 486 of the M-based form).
// tools/async_sweep.cu "more", G1 `l_palm`, N = 262144: fp64 r40 s110 (2
// CTAs/SM) 0.61 ms, s55 b3 0.69 ms (the M-based routine: 1.23 ms); fp32
// r40 s144 (3 CTAs/SM) 0.27 ms (M-based: 0.50 ms).
// sin/cos: one out-of-line copy (G1 `l_palm` fp32 0.238 -> 0.213 ms).  In
// fp64 an earlier A/B put the inlined library routine ahead (0.593 vs 0.603
// ms); tools/pool_call_sweep.cu over all five G1 frame joints, two builds
// each, has the call ahead on every one: 0.64 -> 0.56 (11), 0.63 -> 0.60
// (17), 0.46 -> 0.41 (18), 0.67 -> 0.57 (23), 0.71 -> 0.60 ms (28) — the
// inlined variant's time varies from box to box, the call's much less.
template <class Op, class T>
struct OscCfg {
  static constexpr int kReg = 40, kSmem = sizeof(T) == 8 ? 110 : 144, kMinB = sizeof(T) == 8 ? 2 : 3;
  static constexpr int kFast = Op::kDof >= 20 ? kTrigCall : kTrigLib;
};
template <class Op, class T>
int launch_osc_t(const Launch& L, const void* q, const void* qd, const OscShared& P, void* tau, void* lam,
                 int32_t* status) {
  using C = OscCfg<Op, T>;
  // OscCfg::kAsync: double-buffered asynchronous state input (k_gen_osc_db)
  constexpr bool kDb = AsyncIo<C>::value;
  auto kern = [] {
    if constexpr (kDb) return k_gen_osc_db<Op, T, C::kReg, C::kSmem, C::kMinB, C::kFast>;
    else return k_gen_osc<Op, T, C::kReg, C::kSmem, C::kMinB, C::kFast>;
  }();
  constexpr size_t smem = kDb ? gen_osc_db_smem<Op, T, C::kSmem>() : (size_t)C::kSmem * kGenBlock * sizeof(T);
  const Occ o = occupancy<Op, T>(kern, smem);
  const int64_t blocks = std::min<int64_t>((L.N + kGenBlock - 1) / kGenBlock, (int64_t)o.sms * o.blocks_per_sm);
  cudaStream_t s = static_cast<cudaStream_t>(L.stream);
  const size_t scratch_bytes = (size_t)blocks * kGenBlock * gen_scratch_per_thread<Op, T, C::kReg, C::kSmem>() * sizeof(T);
  T* scratch = nullptr;
  if (scratch_bytes) {
    if (int rc = scratch_alloc(reinterpret_cast<void**>(&scratch), scratch_bytes, s)) return rc;
  }
  kern<<<(unsigned)blocks, kGenBlock, smem, s>>>(L.N, (const T*)q, (const T*)qd, L.ld_in, P, (T*)tau, (T*)lam,
                                                 L.ld_out, status, scratch);
  cudaError_t e = cudaGetLastError();
  scratch_free(scratch, s);
  return (int)e;
}

template <class Op, class T>
int launch_task_t(const Launch& L, const void* q, const TaskShared& P, void* y0, void* y1, int32_t* status,
                  const void* dq = nullptr) {
  constexpr int kReg = 0, kSmem = Op::kSlots, kMinB = sizeof(T) == 8 ? 3 : 4;  // path-only state: all on chip
  auto kern = k_gen_task<Op, T, kReg, kSmem, kMinB>;
  constexpr size_t smem = (size_t)kSmem * kGenBlock * sizeof(T);
  const Occ o = occupancy<Op, T>(kern, smem);
  const int64_t blocks = std::min<int64_t>((L.N + kGenBlock - 1) / kGenBlock, (int64_t)o.sms * o.blocks_per_sm);
  kern<<<(unsigned)blocks, kGenBlock, smem, static_cast<cudaStream_t>(L.stream)>>>(
      L.N, (const T*)q, L.ld_in, P, (T*)y0, (T*)y1, L.ld_out, status, nullptr, (const T*)dq);
  return (int)cudaGetLastError();
}


}  // namespace vdk
