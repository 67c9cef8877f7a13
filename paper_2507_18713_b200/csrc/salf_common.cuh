// salf_common.cuh -- shared device math for the SaLF render kernels (sm_100a).
//
// All fp64 expressions are written in the reference's NumPy evaluation order
// and this translation unit is compiled with --fmad=false, so a product
// followed by a sum never contracts into an FMA unless written as fma().
// Where NumPy itself uses FMA (matmul of (N,3)@(3,3) on x86 OpenBLAS) the
// kernels call fma() in the same chain order; where einsum uses its
// pairwise SIMD order ((p0 + p2) + p1 for length-3 contiguous dots,
// (p0 + p2) + (p1 + p3) for length 4) so do we.  Exactness of the integer
// outputs (tile CSR, hit lists) depends on this; float outputs agree with
// the reference to ~1e-12 (transcendentals differ by <= 1-2 ulp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/salf_b200.h"
#include "salf_fastmath.h"

namespace salf {

constexpr double kAlphaMax = 1.0 - 1e-12;           // scene.py:32
constexpr double kShC0 = 0.2820947918;              // scene.py:28
constexpr double kShC1 = 0.4886025119;              // scene.py:29
constexpr double kEpsAdvance = 1e-4;                 // octree.py:29
constexpr int kMaxRounds = 200000;                   // octree.py:31
constexpr double kDepthWeightMin = 0.5;              // render_ray.py:32
constexpr int kGradStride = 27;                      // w_s 4, w_c 9, w_sh 12, log_a, log_b

// NumPy np.maximum / np.minimum: NaN in either argument propagates.
__device__ __forceinline__ double npmax(double a, double b) { return (a != a || a > b) ? a : b; }
__device__ __forceinline__ double npmin(double a, double b) { return (a != a || a < b) ? a : b; }
__device__ __forceinline__ double npsign(double s) {
  return s > 0.0 ? 1.0 : (s < 0.0 ? -1.0 : (s == 0.0 ? 0.0 : s));
}

// ray_box_range (octree.py:175-194) for one ray against one box, NumPy
// semantics including the zero-direction override.  Returns t_in, t_out.
__device__ __forceinline__ void ray_box(const double o[3], const double d[3], const double bmin[3],
                                        const double bmax[3], double &t_in, double &t_out) {
  double ti = -INFINITY, to = INFINITY;
  bool first = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double nk, fk;
    if (d[k] == 0.0) {
      bool inside = (o[k] >= bmin[k]) && (o[k] <= bmax[k]);
      nk = inside ? -INFINITY : INFINITY;
      fk = inside ? INFINITY : -INFINITY;
    } else {
      double inv = 1.0 / d[k];
      double ta = __dmul_rn(__dsub_rn(bmin[k], o[k]), inv);
      double tb = __dmul_rn(__dsub_rn(bmax[k], o[k]), inv);
      nk = npmin(ta, tb);
      fk = npmax(ta, tb);
    }
    if (first) { ti = nk; to = fk; first = false; }
    else { ti = npmax(ti, nk); to = npmin(to, fk); }
  }
  t_in = ti;
  t_out = to;
}

// 32-byte read-only load of a double4 (two 16-byte LDG.E.128.CONSTANT).
__device__ __forceinline__ double4 ldg_d4(const double *p) {
  const double2 a = __ldg(reinterpret_cast<const double2 *>(p));
  const double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Field parameters of one voxel, fp32 as stored (SALF_PRM_STRIDE floats).
struct VoxPrm {
  float ws[4];
  float wc[9];
  float wsh[12];
};

__device__ __forceinline__ void load_prm(const float *__restrict__ prm, int64_t v, VoxPrm &p) {
  const float4 *q = reinterpret_cast<const float4 *>(prm + v * SALF_PRM_STRIDE);
  float4 a = __ldg(q + 0), b = __ldg(q + 1), c = __ldg(q + 2), e = __ldg(q + 3), f = __ldg(q + 4),
         g = __ldg(q + 5), h = __ldg(q + 6);
  p.ws[0] = a.x; p.ws[1] = a.y; p.ws[2] = a.z; p.ws[3] = a.w;
  p.wc[0] = b.x; p.wc[1] = b.y; p.wc[2] = b.z; p.wc[3] = b.w;
  p.wc[4] = c.x; p.wc[5] = c.y; p.wc[6] = c.z; p.wc[7] = c.w;
  p.wc[8] = e.x; p.wsh[0] = e.y; p.wsh[1] = e.z; p.wsh[2] = e.w;
  p.wsh[3] = f.x; p.wsh[4] = f.y; p.wsh[5] = f.z; p.wsh[6] = f.w;
  p.wsh[7] = g.x; p.wsh[8] = g.y; p.wsh[9] = g.z; p.wsh[10] = g.w;
  p.wsh[11] = h.x;
}

// eval_sdf (scene.py:229-232): einsum dot in (p0 + p2) + p1 order, + bias.
__device__ __forceinline__ double eval_sdf(const VoxPrm &p, const double x[3]) {
  double p0 = __dmul_rn((double)p.ws[0], x[0]);
  double p1 = __dmul_rn((double)p.ws[1], x[1]);
  double p2 = __dmul_rn((double)p.ws[2], x[2]);
  return __dadd_rn(__dadd_rn(__dadd_rn(p0, p2), p1), (double)p.ws[3]);
}

// sdf_to_density (scene.py:235-242) / raw exp (scene.py:250-252), with the
// per-voxel reciprocal 1/b precomputed (x * (1/b) vs x / b: <= 1 ulp).
// Also returns e = exp(-|s|/b) for the backward.
__device__ __forceinline__ double density(int mode, double s, double a, double inv_b, double &e) {
  if (mode == SALF_DENSITY_RAW) {
    e = 0.0;
    return salf_fm::exp(s);
  }
  e = salf_fm::exp(__dmul_rn(-fabs(s), inv_b));
  double inner = __dadd_rn(1.0, __dmul_rn(npsign(s), __dsub_rn(1.0, e)));
  return __dmul_rn(__dmul_rn(0.5, a), inner);
}

// segment_opacity (scene.py:282-284) -> clamped alpha and its complement
// 1 - alpha = exp(-sigma delta) from the same expm1 (no cancellation).
__device__ __forceinline__ double seg_alpha(double sigma, double delta, double &one_minus) {
  const double em = salf_fm::expm1(__dmul_rn(-sigma, delta));
  const double a = -em;
  if (a != a) { one_minus = a; return a; }
  if (a >= kAlphaMax) { one_minus = 1.0 - kAlphaMax; return kAlphaMax; }
  if (a <= 0.0) { one_minus = 1.0; return 0.0; }  // np.clip(alpha, 0, .) (alpha >= 0 anyway)
  one_minus = __dadd_rn(1.0, em);
  return a;
}

// MUFU exp (ex2.approx of x log2 e): relative error ~2^-22 + |x| 2^-24.
__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}

// MUFU reciprocal (rcp.approx.ftz, ~1 ulp; rcp(inf) = 0) for the fp32
// sigmoid -- the IEEE __frcp_rn adds a Newton step and a slow-path branch.
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// eval_color (scene.py:270-279), fp64: z = W_c x + W_sh gamma, sigmoid.
__device__ __forceinline__ void eval_color64(const VoxPrm &p, const double x[3], const double om[3],
                                             double c[3]) {
  const double g0 = kShC0, g1 = __dmul_rn(kShC1, om[1]), g2 = __dmul_rn(kShC1, om[2]),
               g3 = __dmul_rn(kShC1, om[0]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double a0 = __dmul_rn((double)p.wc[3 * i + 0], x[0]);
    double a1 = __dmul_rn((double)p.wc[3 * i + 1], x[1]);
    double a2 = __dmul_rn((double)p.wc[3 * i + 2], x[2]);
    double zc = __dadd_rn(__dadd_rn(a0, a2), a1);
    double b0 = __dmul_rn((double)p.wsh[4 * i + 0], g0);
    double b1 = __dmul_rn((double)p.wsh[4 * i + 1], g1);
    double b2 = __dmul_rn((double)p.wsh[4 * i + 2], g2);
    double b3 = __dmul_rn((double)p.wsh[4 * i + 3], g3);
    double zs = __dadd_rn(__dadd_rn(b0, b2), __dadd_rn(b1, b3));
    double z = __dadd_rn(zc, zs);
    c[i] = 1.0 / (1.0 + exp(-z));
  }
}

// Same field in fp32 (values only flow into the colour accumulators; no
// threshold decision depends on them).
__device__ __forceinline__ void eval_color32(const VoxPrm &p, const double xd[3], const double od[3],
                                             double c[3]) {
  const float x0 = (float)xd[0], x1 = (float)xd[1], x2 = (float)xd[2];
  const float g0 = (float)kShC0, g1 = (float)kShC1 * (float)od[1], g2 = (float)kShC1 * (float)od[2],
              g3 = (float)kShC1 * (float)od[0];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float z = __fmaf_rn(p.wc[3 * i + 2], x2, __fmaf_rn(p.wc[3 * i + 1], x1, p.wc[3 * i] * x0));
    z = __fmaf_rn(p.wsh[4 * i + 0], g0, z);
    z = __fmaf_rn(p.wsh[4 * i + 1], g1, z);
    z = __fmaf_rn(p.wsh[4 * i + 2], g2, z);
    z = __fmaf_rn(p.wsh[4 * i + 3], g3, z);
    c[i] = (double)fast_rcp(1.0f + fast_exp(-z));
  }
}

// expm1(x) for x <= 0 in fp32 without cancellation: degree-7 Taylor on
// (-0.25, 0] (truncation |x|^8/8! < 4e-10 relative), exp(x) - 1 below it
// (|expm1| >= 0.22 there, so the MUFU error stays ~1e-7 relative).  Branchless.
__device__ __forceinline__ float expm1_neg(float x) {
  float p = __fmaf_rn(x, 1.0f / 5040.0f, 1.0f / 720.0f);
  p = __fmaf_rn(x, p, 1.0f / 120.0f);
  p = __fmaf_rn(x, p, 1.0f / 24.0f);
  p = __fmaf_rn(x, p, 1.0f / 6.0f);
  p = __fmaf_rn(x, p, 0.5f);
  const float small = __fmaf_rn(x * x, p, x);
  return x > -0.25f ? small : fast_exp(x) - 1.0f;
}

#ifndef SALF_COLOR_PACK
#define SALF_COLOR_PACK 1  // red and green channels in fp32x2 (FFMA2 with broadcast x / gam)
#endif

// fp32 colour with a precomputed per-ray SH basis gam = (C0, C1 y, C1 z, C1 x).
// With SALF_COLOR_PACK the red and green dot products run as one fp32x2 chain
// (FMUL2 / FFMA2, the x and gam operands broadcast): each half performs the
// scalar chain's IEEE operations in the same order, so c is bit-identical.
__device__ __forceinline__ void eval_color32g(const VoxPrm &p, const float x[3], const float gam[4], float c[3]) {
#if SALF_COLOR_PACK
  {
    float2 z = __fmul2_rn(make_float2(p.wc[0], p.wc[3]), make_float2(x[0], x[0]));
    z = __ffma2_rn(make_float2(p.wc[1], p.wc[4]), make_float2(x[1], x[1]), z);
    z = __ffma2_rn(make_float2(p.wc[2], p.wc[5]), make_float2(x[2], x[2]), z);
#pragma unroll
    for (int k = 0; k < 4; ++k) z = __ffma2_rn(make_float2(p.wsh[k], p.wsh[4 + k]), make_float2(gam[k], gam[k]), z);
    const float2 t = __fmul2_rn(make_float2(-z.x, -z.y), make_float2(1.4426950408889634f, 1.4426950408889634f));
    float2 E;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(E.x) : "f"(t.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(E.y) : "f"(t.y));
    const float2 d = __fadd2_rn(make_float2(1.0f, 1.0f), E);
    c[0] = fast_rcp(d.x);
    c[1] = fast_rcp(d.y);
  }
  {
    float z = __fmaf_rn(p.wc[8], x[2], __fmaf_rn(p.wc[7], x[1], p.wc[6] * x[0]));
    z = __fmaf_rn(p.wsh[8], gam[0], z);
    z = __fmaf_rn(p.wsh[9], gam[1], z);
    z = __fmaf_rn(p.wsh[10], gam[2], z);
    z = __fmaf_rn(p.wsh[11], gam[3], z);
    c[2] = fast_rcp(1.0f + fast_exp(-z));
  }
#else
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float z = __fmaf_rn(p.wc[3 * i + 2], x[2], __fmaf_rn(p.wc[3 * i + 1], x[1], p.wc[3 * i] * x[0]));
    z = __fmaf_rn(p.wsh[4 * i + 0], gam[0], z);
    z = __fmaf_rn(p.wsh[4 * i + 1], gam[1], z);
    z = __fmaf_rn(p.wsh[4 * i + 2], gam[2], z);
    z = __fmaf_rn(p.wsh[4 * i + 3], gam[3], z);
    c[i] = fast_rcp(1.0f + fast_exp(-z));
  }
#endif
}

// (N,3) @ (3,3) as NumPy/OpenBLAS computes it on x86: fma(a2, b2, fma(a1, b1, a0*b0)).
// r is row-major; `transposed` selects a @ r.T (dot with row i) vs a @ r (column i).
__device__ __forceinline__ double mm_row(const double a[3], const double *r, int i) {
  return fma(a[2], r[3 * i + 2], fma(a[1], r[3 * i + 1], __dmul_rn(a[0], r[3 * i + 0])));
}
__device__ __forceinline__ double mm_col(const double a[3], const double *r, int j) {
  return fma(a[2], r[6 + j], fma(a[1], r[3 + j], __dmul_rn(a[0], r[j])));
}

// Orderable 64-bit key of a double (ascending), NaN last.
__device__ __forceinline__ uint64_t order_key(double z) {
  uint64_t u = (uint64_t)__double_as_longlong(z);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// Transposed warp reduction of a 32-vector held by every lane: five xor
// steps, each lane sending half of what it still holds (16 + 8 + 4 + 2 + 1 =
// 31 shuffles instead of 32 x 5).  Afterwards lane l holds the warp sum of
// component l.  fp32 partial sums (<= 32 terms; relative error ~1e-7 of the
// warp's contribution) -- the global accumulation is fp64.
// PRECONDITION: all 32 lanes converged.
__device__ __forceinline__ float warp_transpose_reduce(float v[32]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = upper ? v[i] : v[i + n / 2];
      const float keep = upper ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(full, send, off);
    }
  }
  return v[0];
}

// Gradient of one included segment (reference backward.py:52-100): the 27
// parameter components, written as fp32 into g[0..26] (g[27..31] = 0).  The
// scalar chain (g_alpha, g_sigma, ds, gz) is fp64; the outer products are
// fp32 -- they only feed fp32 warp partial sums of an fp64 accumulation.
//   A = dL/dw, tb = T_before, w = tb * alpha, suffix = sum_{j>i} A_j w_j,
//   tail = (dC . background) * T_final.
__device__ __forceinline__ void segment_grad(int mode, double delta, double sigma, double alpha, double om,
                                             double s, double e, double a, double inv_b, const double x[3],
                                             const double c[3], const double dir[3], double A, double tb,
                                             double w, double suffix, double tail, const double dC[3],
                                             float g[32]) {
  const double g_alpha = __dsub_rn(__dmul_rn(A, tb), __ddiv_rn(__dadd_rn(suffix, tail), __dsub_rn(1.0, alpha)));
  // exp(-sigma delta) = 1 - alpha (unclamped) from the forward's expm1
  const double g_sigma = __dmul_rn(__dmul_rn(g_alpha, delta),
                                   alpha >= kAlphaMax ? salf_fm::exp(__dmul_rn(-sigma, delta)) : om);
  double ds;
  if (mode == SALF_DENSITY_SDF) {
    const double k2 = __dmul_rn(__dmul_rn(a, 0.5), inv_b);
    ds = (s == 0.0) ? 0.0 : __dmul_rn(__dmul_rn(g_sigma, k2), e);
    g[25] = (float)__dmul_rn(g_sigma, sigma);
    g[26] = (float)__dmul_rn(g_sigma, __dmul_rn(__dmul_rn(-k2, s), e));
  } else {
    ds = __dmul_rn(g_sigma, sigma);
    g[25] = 0.0f;
    g[26] = 0.0f;
  }
  const float fx[3] = {(float)x[0], (float)x[1], (float)x[2]};
  const float fds = (float)ds;
  g[0] = fds * fx[0]; g[1] = fds * fx[1]; g[2] = fds * fx[2]; g[3] = fds;
  const float gam[4] = {(float)kShC0, (float)(kShC1 * dir[1]), (float)(kShC1 * dir[2]), (float)(kShC1 * dir[0])};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float gz = (float)__dmul_rn(__dmul_rn(__dmul_rn(dC[i], w), c[i]), __dsub_rn(1.0, c[i]));
#pragma unroll
    for (int j = 0; j < 3; ++j) g[4 + 3 * i + j] = gz * fx[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) g[13 + 4 * i + j] = gz * gam[j];
  }
#pragma unroll
  for (int k = kGradStride; k < 32; ++k) g[k] = 0.0f;
}

// One ray segment's fp32 fields, shared BIT FOR BIT by the certified ray
// forward (k_ray_forward_fast) and the mixed ray backward: the backward
// recovers the reference's suffix sums S_i = sum_{j>i} A_j w_j
// (backward.py:26-32, :62-64) as differences of the forward's fp64 totals of
// the exact fp32 products (w, w c, w t_mid) and its own running fp64 sums of
// the same products -- identical values, so the differences carry only fp64
// rounding (no fp32 "total - prefix" cancellation).
constexpr float kYClampF = 27.631021115928547f;  // -ln(1 - kAlphaMax) (scene.py:32)

struct SegF32 {
  float s, sigma, ee, yr, y, alpha;
};

template <bool kSdf>
__device__ __forceinline__ void seg_fields_f32(const VoxPrm &p, float a, float inv_b, const float x[3], float delta,
                                               SegF32 &o) {
  o.s = __fmaf_rn(p.ws[2], x[2], __fmaf_rn(p.ws[1], x[1], __fmaf_rn(p.ws[0], x[0], p.ws[3])));
  if (kSdf) {
    // a/2 (1 + sign(s)(1 - e)): a - a/2 e for s > 0, a/2 e otherwise (scene.py:235-242)
    o.ee = fast_exp(-fabsf(o.s) * inv_b);
    const float he = 0.5f * a * o.ee;
    o.sigma = o.s > 0.f ? a - he : he;
  } else {
    o.ee = 0.f;
    o.sigma = fast_exp(o.s);
  }
  o.yr = o.sigma * delta;
  const bool cl = o.yr >= kYClampF;
  o.y = cl ? kYClampF : o.yr;                   // -log1p(-clip(alpha))
  o.alpha = cl ? 1.f : -expm1_neg(-o.yr);      // segment_opacity (scene.py:282-284)
}

// Neumaier compensated fp32 sum h + c (+= y, y >= 0).
__device__ __forceinline__ void neumaier_add(float &h, float &c, float y) {
  const float t = h + y;
  c += fabsf(h) >= y ? (h - t) + y : (y - t) + h;
  h = t;
}

// fp32 colour + its complement without cancellation: c = 1 / (1 + E),
// 1 - c = E c (E = e^-z); c is eval_color32g's value bit for bit.
__device__ __forceinline__ void eval_color32c(const VoxPrm &p, const float x[3], const float gam[4], float c[3],
                                              float omc[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float z = __fmaf_rn(p.wc[3 * i + 2], x[2], __fmaf_rn(p.wc[3 * i + 1], x[1], p.wc[3 * i] * x[0]));
    z = __fmaf_rn(p.wsh[4 * i + 0], gam[0], z);
    z = __fmaf_rn(p.wsh[4 * i + 1], gam[1], z);
    z = __fmaf_rn(p.wsh[4 * i + 2], gam[2], z);
    z = __fmaf_rn(p.wsh[4 * i + 3], gam[3], z);
    const float E = fast_exp(-z);
    c[i] = fast_rcp(1.0f + E);
    omc[i] = E * c[i];
  }
}

// Mixed-precision gradient of one included ray segment (backward.py:52-100).
// Running state per ray: Y = Yh + Yc before this segment (the forward's
// compensated sum, advanced here), the fp64 prefix sums P = (w c[3], w, w t)
// of the exact fp32 products, and the forward's totals Acc of the same sums.
// kColor = false: depth-only seeds (LiDAR), the colour terms are compile-time zeros.
struct RayBwdState {
  float Yh, Yc;
  double Pc[3], Pw, Pwt;
  double Ac[3], Aw, Awt;
};

// kFeat (LiDAR intensity / ray-drop extension): the blended feature enters A
// like a colour without background, fdot = dF . f of this segment; its suffix
// sum is CF - PF with CF = dF . (forward's fp64 feature totals) and PF the
// running fp64 sum of w fdot.  Returns w.
template <bool kSdf, bool kColor = true, bool kFeat = false>
__device__ __forceinline__ float seg_grad_f32(const VoxPrm &p, float a, float inv_b, const float x[3], float delta,
                                              double tm, double D, const float gam[4], bool want_color,
                                              const float dC[3], float dws, float tail, RayBwdState &r, float g[32],
                                              double fdot = 0.0, double *PF = nullptr, double CF = 0.0) {
  SegF32 f;
  seg_fields_f32<kSdf>(p, a, inv_b, x, delta, f);
  const float om = fast_exp(-f.yr);                   // exp(-sigma delta), unclamped (backward.py:66)
  const float omc = f.alpha >= 1.f ? 1e-12f : om;     // 1 - alpha as the reference clamps it
  const float T = fast_exp(-(r.Yh + r.Yc));           // T_before, the forward's value
  const float w = T * f.alpha;
  float col[3] = {0.f, 0.f, 0.f}, ocol[3] = {0.f, 0.f, 0.f};
  if (kColor && want_color) eval_color32c(p, x, gam, col, ocol);
  const double wd = (double)w;
  if (kColor) {
#pragma unroll
    for (int k = 0; k < 3; ++k) r.Pc[k] = fma(wd, (double)col[k], r.Pc[k]);
  }
  r.Pw = __dadd_rn(r.Pw, wd);
  r.Pwt = fma(wd, tm, r.Pwt);
  // S = sum_{j>i} A_j w_j = dC . (Ac - Pc) + dD / ws ((Awt - Pwt) - D (Aw - Pw))
  const double sw = __dsub_rn(r.Aw, r.Pw), swt = __dsub_rn(r.Awt, r.Pwt);
  double S = (double)dws * __dsub_rn(swt, __dmul_rn(D, sw));
  if (kColor) {
#pragma unroll
    for (int k = 0; k < 3; ++k) S = fma((double)dC[k], __dsub_rn(r.Ac[k], r.Pc[k]), S);
  }
  if (kFeat) {
    *PF = fma(wd, fdot, *PF);
    S = __dadd_rn(S, __dsub_rn(CF, *PF));
  }
  const float dq = (float)__dsub_rn(tm, D);
  float A = kColor ? __fmaf_rn(dC[2], col[2], __fmaf_rn(dC[1], col[1], __fmaf_rn(dC[0], col[0], dws * dq)))
                   : dws * dq;
  if (kFeat) A += (float)fdot;
  const float g_alpha = __fmaf_rn(A, T, -((float)S + tail) * fast_rcp(omc));
  const float g_sigma = g_alpha * delta * om;
  float ds, ga, gb;
  if (kSdf) {
    const float k2e = 0.5f * a * inv_b * f.ee;
    ds = (f.s == 0.f) ? 0.f : g_sigma * k2e;
    ga = g_sigma * f.sigma;
    gb = -g_sigma * k2e * f.s;
  } else {
    ds = g_sigma * f.sigma;
    ga = 0.f;
    gb = 0.f;
  }
  g[0] = ds * x[0]; g[1] = ds * x[1]; g[2] = ds * x[2]; g[3] = ds;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float gz = kColor ? dC[i] * (w * col[i]) * ocol[i] : 0.f;  // dC w c (1 - c)
#pragma unroll
    for (int k = 0; k < 3; ++k) g[4 + 3 * i + k] = kColor ? gz * x[k] : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) g[13 + 4 * i + k] = kColor ? gz * gam[k] : 0.f;
  }
  g[25] = ga;
  g[26] = gb;
#pragma unroll
  for (int k = kGradStride; k < 32; ++k) g[k] = 0.f;
  neumaier_add(r.Yh, r.Yc, f.y);
  return w;
}

// Warp-aggregated gradient scatter.  PRECONDITION: called by all 32 lanes
// of a converged warp.  Lanes holding the same voxel id form a group
// (__match_any_sync).  Lanes in groups of fewer than 4 add their non-zero
// components directly -- all such lanes in the same 27 (predicated) RED
// instructions, so distinct voxels never serialise; each group of >= 4
// lanes is summed with one transposed reduction, after which lanes 0..26
// issue one coalesced fp64 atomic per component.  g is consumed.
__device__ __forceinline__ void scatter_grad(double *__restrict__ grad, int64_t vid, bool active, float g[32]) {
  const unsigned full = 0xffffffffu;
  if (!__ballot_sync(full, active)) return;
  const int lane = threadIdx.x & 31;
  const long long key = active ? (long long)vid : -1ll;
  const unsigned peers = __match_any_sync(full, key);
  const bool big = active && __popc(peers) >= 4;
  if (active && !big) {
    double *dst = grad + key * kGradStride;
#pragma unroll
    for (int k = 0; k < kGradStride; ++k)
      if (g[k] != 0.0f) atomicAdd(dst + k, (double)g[k]);
  }
  unsigned pending = __ballot_sync(full, big);
  while (pending) {
    const int L = __ffs(pending) - 1;
    const long long lkey = __shfl_sync(full, key, L);
    const bool mem = big && key == lkey;
    pending &= ~__ballot_sync(full, mem);
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = mem ? g[k] : 0.0f;
    const float tot = warp_transpose_reduce(v);
    if (lane < kGradStride && tot != 0.0f) atomicAdd(grad + lkey * kGradStride + lane, (double)tot);
  }
}

}  // namespace salf
