// salf_fastmath.h -- fp64 exp / expm1 for the render hot loops.
//
// libdevice's exp/expm1 load each 64-bit polynomial coefficient into uniform
// registers (two UMOVs per coefficient) on every call inside the composite
// and backward loops; the ncu source view put ~7% of the backward's
// instructions there.  These versions keep the coefficients in the constant
// bank (DFMA takes them as c[] operands) and share one reduction:
//   x = n ln2 + r, |r| <= ln2/2 (Cody-Waite; the rounding of r is recovered and folded in),
//   expm1(r) = r + r^2 P(r), P the degree-11 Taylor tail (1/2! .. 1/13!),
//   truncation r^14/14! < 4.4e-18, i.e. < 0.05 ulp of expm1(r) on the range,
//   exp(x)   = 2^n + 2^n expm1(r)           (one fma),
//   expm1(x) = 2^n expm1(r) + (2^n - 1)     (one fma; 2^n - 1 exact for n >= -53).
// Max error vs long-double expl/expm1l (tools/fastmath_check.cpp, which
// compiles this same header with g++ -ffp-contract=off; run by
// tests/test_native_cpu.py): exp <= 1 ulp; expm1 <= 1.03 ulp for x <= 0 (the
// render path's -sigma delta), <= 1.8 ulp for x > 0 (2^n scaling of the
// core's error at n = 1).
// Used wherever NumPy's exp/expm1 is restated (the reference's own libm
// results differ from any GPU libm by the same <= 1 ulp).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define SALF_FM_FN __host__ __device__ __forceinline__
#define SALF_FM_CONST __constant__
#else
#define SALF_FM_FN static inline
#define SALF_FM_CONST static const
#endif

namespace salf_fm {

// 1/k! for k = 13 .. 2 (Horner order): a constant-bank copy for the device,
// a plain one for host callers (the host-side checks of these functions)
#define SALF_FM_INV_FACT                                                                                      \
  {1.6059043836821613e-10, 2.08767569878681e-09,  2.505210838544172e-08, 2.755731922398589e-07,               \
   2.7557319223985893e-06, 2.48015873015873e-05,  0.0001984126984126984, 0.001388888888888889,                \
   0.008333333333333333,   0.041666666666666664, 0.16666666666666666,   0.5}
SALF_FM_CONST double kInvFact[12] = SALF_FM_INV_FACT;
#ifdef __CUDACC__
static const double kInvFactHost[12] = SALF_FM_INV_FACT;
#endif

constexpr double kLog2e = 1.4426950408889634;
constexpr double kLn2Hi = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000 (trailing zeros)
constexpr double kLn2Lo = 1.90821492927058770002e-10;  // ln2 - kLn2Hi
constexpr double kShift = 6755399441055744.0;          // 1.5 * 2^52: round-to-nearest integer
constexpr double kExpMax = 709.782712893384;           // above: exp overflows
constexpr double kExpMin = -745.1332191019412;         // below: exp underflows to 0

SALF_FM_FN double fm_fma(double a, double b, double c) { return fma(a, b, c); }
SALF_FM_FN double fm_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
SALF_FM_FN double fm_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}

SALF_FM_FN double fm_pow2(int n) {  // 2^n for -1022 <= n <= 1023
  const int64_t bits = (int64_t)(n + 1023) << 52;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(bits);
#else
  double d;
  memcpy(&d, &bits, 8);
  return d;
#endif
}

// expm1(r) for |r| <= ~0.35
SALF_FM_FN double fm_expm1_core(double r) {
#if defined(__CUDACC__) && !defined(__CUDA_ARCH__)
  const double *c = kInvFactHost;
#else
  const double *c = kInvFact;
#endif
  double p = c[0];
#pragma unroll
  for (int k = 1; k < 12; ++k) p = fm_fma(p, r, c[k]);
  return fm_fma(fm_mul(r, r), p, r);
}

// expm1(r) for r = x - n ln2 (Cody-Waite: fma(-n, ln2_hi, x) is exact since
// ln2_hi has 32 significant bits), with the rounding error r_lo of the second
// step recovered (Fast2Sum) and folded in to first order:
// expm1(r + r_lo) ~= expm1(r) + r_lo (1 + expm1(r)).
SALF_FM_FN double fm_expm1_reduced(double x, int &n) {
  const double t = fm_add(fm_mul(x, kLog2e), kShift);
  const double nd = fm_add(t, -kShift);
  n = (int)nd;
  const double r_hi = fm_fma(-nd, kLn2Hi, x);
  const double r = fm_fma(-nd, kLn2Lo, r_hi);
  const double r_lo = fm_fma(-nd, kLn2Lo, fm_add(r_hi, -r));
  const double em = fm_expm1_core(r);
  return fm_add(em, fm_fma(r_lo, em, r_lo));
}

SALF_FM_FN double exp(double x) {
  if (!(x > kExpMin)) return x != x ? x : 0.0;
  if (x > kExpMax) return INFINITY;
  int n;
  const double em = fm_expm1_reduced(x, n);
  if (n < -1021) {  // subnormal result: scale in two steps
    const double s = fm_pow2(n + 64);
    return fm_mul(fm_fma(s, em, s), 5.421010862427522e-20);  // 2^-64
  }
  if (n > 1023) {
    const double s = fm_pow2(n - 1);
    return fm_mul(fm_fma(s, em, s), 2.0);
  }
  const double s = fm_pow2(n);
  return fm_fma(s, em, s);
}

SALF_FM_FN double expm1(double x) {
  if (x != x) return x;
  if (x > -0.34657359027997264 && x < 0.34657359027997264) return fm_expm1_core(x);
  if (x < -40.0) return -1.0;  // expm1 rounds to -1 below ~ -37.4
  if (x > kExpMax) return INFINITY;
  int n;
  const double em = fm_expm1_reduced(x, n);
  if (n > 1023) {
    const double s = fm_pow2(n - 1);
    return fm_mul(fm_fma(s, em, s), 2.0);
  }
  const double s = fm_pow2(n);
  return fm_fma(s, em, fm_add(s, -1.0));
}

}  // namespace salf_fm
