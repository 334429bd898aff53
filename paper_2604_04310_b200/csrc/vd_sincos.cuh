// fp64 sin/cos of a joint angle for the sm_100a kernels.
//
// CUDA's sincos(double) inlines ~70 instructions per call; the kernels
// evaluate it once per revolute joint (7 per Panda, 26 per G1 state).  This
// version:
//   * reduces x = k·π/2 + r (k by the 1.5·2^52 rounding trick, no XU
//     conversions) with a three-part Cody–Waite split of π/2 and
//     FMAs (exact products), valid far beyond any joint angle; |x| > 1e6 falls
//     back to the library routine (full Payne–Hanek reduction);
//   * evaluates sin/cos of r ∈ [−π/4, π/4] with the fdlibm minimax kernels
//     (__kernel_sin / __kernel_cos coefficients, < 1 ulp on that interval);
//   * has no XU-pipe conversions and only 16 coefficients.
// Accuracy: within ~2 ulp of the correctly rounded result on the joint range,
// far inside the 1e-10 parity bar (tests compare against the oracle's libm).
#pragma once

namespace vdk {

#if defined(__CUDACC__)
// coefficients in constant memory: c[bank][offset] operands of the DFMAs
static __constant__ double vd_sc_c[16] = {
    0x1.45f306dc9c883p-1,         // 2/π
    0x1.921fb54442d18p+0,         // π/2, three-part split (P1 + P2 + P3)
    0x1.1a62633145c07p-54,
    -0x1.f1976b7ed8fbcp-110,
    -1.66666666666666324348e-01,  // S1..S6 (fdlibm __kernel_sin)
    8.33333333332248946124e-03,
    -1.98412698298579493134e-04,
    2.75573137070700676789e-06,
    -2.50507602534068634195e-08,
    1.58969099521155010221e-10,
    4.16666666666666019037e-02,   // C1..C6 (fdlibm __kernel_cos)
    -1.38888888888741095749e-03,
    2.48015872894767294178e-05,
    -2.75573143513906633035e-07,
    2.08757232129817482790e-09,
    -1.13596475577881948265e-11,
};
// out of line: the library routine inlines ~70 instructions (and its own
// coefficient UMOVs) at every call site otherwise
static __device__ __noinline__ void vd_sincos_f64_slow(double x, double* sp, double* cp) { sincos(x, sp, cp); }

__device__ __forceinline__ void vd_sincos_f64(double x, double* sp, double* cp) {
#if defined(VD_LIB_SINCOS)  // A/B switch for measurements
  sincos(x, sp, cp);
  return;
#endif
  if (fabs(x) > 1.0e6) {
    vd_sincos_f64_slow(x, sp, cp);
    return;
  }
  const double* K = vd_sc_c;
  // k = nearest integer to x·2/π without the XU pipe: adding 1.5·2^52 rounds
  // to an integer in the low mantissa bits (exact for |x·2/π| < 2^51), and
  // the low word of that sum is k in two's complement
  const double t = fma(x, K[0], 0x1.8p52);
  const double kf = t - 0x1.8p52;
  const int q = __double2loint(t);
  double r = fma(-kf, K[1], x);
  r = fma(-kf, K[2], r);
  r = fma(-kf, K[3], r);
  const double z = r * r;
  double ps = fma(z, K[9], K[8]);
  ps = fma(z, ps, K[7]);
  ps = fma(z, ps, K[6]);
  ps = fma(z, ps, K[5]);
  ps = fma(z, ps, K[4]);
  const double s = fma(r * z, ps, r);
  double pc = fma(z, K[15], K[14]);
  pc = fma(z, pc, K[13]);
  pc = fma(z, pc, K[12]);
  pc = fma(z, pc, K[11]);
  pc = fma(z, pc, K[10]);
  const double c = fma(z * z, pc, fma(-0.5, z, 1.0));
  // x = k·π/2 + r: sin x = (sin r, cos r, −sin r, −cos r)[k mod 4],
  //                cos x = (cos r, −sin r, −cos r, sin r)[k mod 4]
  double sn = (q & 1) ? c : s;
  double cs = (q & 1) ? s : c;
  if (q & 2) sn = -sn;
  if ((q + 1) & 2) cs = -cs;
  *sp = sn;
  *cp = cs;
}

// fp32: the same structure with float constants.  k by the 1.5·2^23 trick
// (exact for |x·2/π| < 2^22), a three-part Cody–Waite π/2 (FMA products
// exact) valid for |x| ≤ 1e4, the Cephes sinf / cosf minimax kernels on
// [−π/4, π/4] (< 1 ulp there); |x| > 1e4 falls back to sincosf.  CUDA's
// sincosf carries its Payne–Hanek slow path inline at every call site.
static __device__ __noinline__ void vd_sincos_f32_slow(float x, float* sp, float* cp) { sincosf(x, sp, cp); }

__device__ __forceinline__ void vd_sincos_f32(float x, float* sp, float* cp) {
  if (fabsf(x) > 1.0e4f) {
    vd_sincos_f32_slow(x, sp, cp);
    return;
  }
  const float t = fmaf(x, 0x1.45f306p-1f, 0x1.8p23f);
  const float kf = t - 0x1.8p23f;
  const int q = __float_as_int(t);
  float r = fmaf(-kf, 0x1.921fb6p+0f, x);
  r = fmaf(-kf, -0x1.777a5cp-25f, r);
  r = fmaf(-kf, -0x1.ee59dap-50f, r);
  const float z = r * r;
  const float s = fmaf(r * z, fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f), r);
  const float c = fmaf(z * z, fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z, 4.166664568298827e-2f),
                       fmaf(-0.5f, z, 1.0f));
  float sn = (q & 1) ? c : s;
  float cs = (q & 1) ? s : c;
  if (q & 2) sn = -sn;
  if ((q + 1) & 2) cs = -cs;
  *sp = sn;
  *cp = cs;
}
#endif

}  // namespace vdk
