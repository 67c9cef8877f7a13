// salf_ray.cu -- linear-octree ray path (reference octree.py, render_ray.py).
//
// One thread per ray runs the reference's epsilon-marching state machine
// (octree.py:214-273) in fp64 with the reference's operation order and no FMA
// contraction, so the ray/voxel hit list is bit-identical to march_batch.
// The fused forward shades each leaf segment as it is found (fp64 opacity
// chain, fp32 or fp64 colour), applies the product-of-(1 - alpha) early stop
// of render_ray.py:154-157 and composites front to back (render_ray.py:86-114)
// without materialising any per-segment record.  The backward re-marches the
// same rays warp-synchronously and scatters per-voxel gradients with
// warp-aggregated atomics.
#include <stdlib.h>

#include <type_traits>

#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {

struct OctDev {
  const int32_t *nodes;
  double rmin[3], rmax[3];
  double root_edge;
  int max_depth;
  // jump table (salf_octree_jump_build): words after jk levels, corners per axis
  int jk;
  const int32_t *jump;
  const double *jcorner;  // [3][2^jk]
  double jedge;           // root_edge * 0.5^jk (exact)
  double inv_root;        // RN(1 / root_edge), host IEEE division
};

constexpr int32_t kJumpNone = INT32_MIN;  // the descent ends above depth K
constexpr int kJumpMaxLevels = 8;

static size_t jump_words(int k) { return (size_t)1 << (3 * k); }
static size_t jump_corner_offset(int k) { return (jump_words(k) * sizeof(int32_t) + 15) & ~(size_t)15; }

static OctDev make_oct(const salf_octree_t *t) {
  OctDev o;
  o.nodes = t->nodes;
  for (int k = 0; k < 3; ++k) {
    o.rmin[k] = t->root_min[k];
    o.rmax[k] = t->root_min[k] + t->root_edge;  // buffer.root_min + buffer.root_edge (octree.py:232)
  }
  o.root_edge = t->root_edge;
  o.max_depth = t->max_depth;
  o.jk = (t->jump && t->jump_levels > 0 && t->jump_levels <= kJumpMaxLevels) ? t->jump_levels : 0;
  o.jump = o.jk ? (const int32_t *)t->jump : nullptr;
  o.jcorner = o.jk ? (const double *)((const char *)t->jump + jump_corner_offset(o.jk)) : nullptr;
  double e = t->root_edge;
  for (int l = 0; l < o.jk; ++l) e *= 0.5;  // the descent's edge halving, exact
  o.jedge = e;
  o.inv_root = 1.0 / t->root_edge;
  return o;
}

enum : int32_t { kStatusRoundCap = 1, kStatusOutsideRoot = 2, kStatusOrder = 4, kStatusRedo = 8 };

#ifndef SALF_MARCH_INTBITS
#define SALF_MARCH_INTBITS 1
#endif
#ifndef SALF_DIV_MARKSTEIN
#define SALF_DIV_MARKSTEIN 1
#endif
// (p - root_min) / root_edge, correctly rounded (== __ddiv_rn).  The divisor
// is fixed per tree, so its correctly rounded reciprocal y comes from the
// host; q0 = RN(x y) is within 1 ulp of x / e, r = x - q0 e is exact (FMA),
// and RN(q0 + r y) = RN(x / e) (Markstein's theorem; x is 0 or >= ~1e-17 in
// magnitude here, so nothing underflows).  Saves __ddiv_rn's per-call
// reciprocal refinement and slow-path test: 3 divisions per march round.
__device__ __forceinline__ double div_root(double x, const OctDev &t) {
#if SALF_DIV_MARKSTEIN
  const double q0 = __dmul_rn(x, t.inv_root);
  const double r = fma(-q0, t.root_edge, x);
  return fma(r, t.inv_root, q0);
#else
  return __ddiv_rn(x, t.root_edge);
#endif
}

// query_batch for one point (octree.py:136-166).  Returns node word
// (-1 empty, <= -2 leaf), writes corner/edge of the node.
__device__ __forceinline__ int32_t query_point(const OctDev &t, const double p[3], double corner[3], double &edge,
                                               bool &outside) {
  double u[3];
  outside = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    u[k] = div_root(__dsub_rn(p[k], t.rmin[k]), t);
    if (u[k] < -1e-9 || u[k] > 1.0 + 1e-9) outside = true;
    u[k] = npmin(npmax(u[k], 0.0), 1.0);
    corner[k] = t.rmin[k];
  }
  edge = t.root_edge;
  int32_t w = __ldg(t.nodes);
#if SALF_MARCH_INTBITS
  // The reference's iterate u <- 2u - bit is exact, so the bit taken at
  // level l is bit (30 - l) of floor(u 2^31) (exact scaling; u == 1
  // iterates to 1, i.e. all ones; trees are < 31 levels deep).  Integer bit
  // extraction replaces the per-level fp64 compare / update; the corner
  // accumulation stays fp64 in the reference's order.
  uint32_t U[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) U[k] = min((uint32_t)__dmul_rn(u[k], 2147483648.0), 0x7fffffffu);
  int sh = 30;
  if (t.jk) {
    // jump table: the word, corner and edge the loop below reaches after jk
    // levels (built with the same operations), unless the path ends earlier
    const int s0 = 31 - t.jk;
    const uint32_t cx = U[0] >> s0, cy = U[1] >> s0, cz = U[2] >> s0;
    const int32_t wj = __ldg(t.jump + ((((cx << t.jk) | cy) << t.jk) | cz));
    if (wj != kJumpNone) {
      const int n = 1 << t.jk;
      corner[0] = __ldg(t.jcorner + cx);
      corner[1] = __ldg(t.jcorner + n + cy);
      corner[2] = __ldg(t.jcorner + 2 * n + cz);
      edge = t.jedge;
      sh = 30 - t.jk;
      w = wj;
    }
  }
  while (w >= 0) {
    const int b0 = (U[0] >> sh) & 1, b1 = (U[1] >> sh) & 1, b2 = (U[2] >> sh) & 1;
    --sh;
    edge = __dmul_rn(edge, 0.5);
    corner[0] = __dadd_rn(corner[0], b0 ? edge : 0.0);
    corner[1] = __dadd_rn(corner[1], b1 ? edge : 0.0);
    corner[2] = __dadd_rn(corner[2], b2 ? edge : 0.0);
    w = __ldg(t.nodes + w + b0 + 2 * b1 + 4 * b2);
  }
#else
  while (w >= 0) {
    const int b0 = u[0] >= 0.5, b1 = u[1] >= 0.5, b2 = u[2] >= 0.5;
    edge = __dmul_rn(edge, 0.5);
    corner[0] = __dadd_rn(corner[0], b0 ? edge : 0.0);
    corner[1] = __dadd_rn(corner[1], b1 ? edge : 0.0);
    corner[2] = __dadd_rn(corner[2], b2 ? edge : 0.0);
    // 2u - bit is exact, so one fma gives the reference's value
    u[0] = fma(2.0, u[0], -(double)b0);
    u[1] = fma(2.0, u[1], -(double)b1);
    u[2] = fma(2.0, u[2], -(double)b2);
    w = __ldg(t.nodes + w + b0 + 2 * b1 + 4 * b2);
  }
#endif
  return w;
}

// Slab test with precomputed reciprocals (1.0 / d is IEEE-exact, so caching
// it per ray changes nothing).  NumPy semantics incl. the zero-direction rule.
__device__ __forceinline__ void ray_box_inv(const double o[3], const double d[3], const double inv[3],
                                            const double bmin[3], const double bmax[3], double &t_in,
                                            double &t_out) {
  double ti = 0.0, to = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double nk, fk;
    if (d[k] == 0.0) {
      const bool inside = (o[k] >= bmin[k]) && (o[k] <= bmax[k]);
      nk = inside ? -INFINITY : INFINITY;
      fk = inside ? INFINITY : -INFINITY;
    } else {
      const double ta = __dmul_rn(__dsub_rn(bmin[k], o[k]), inv[k]);
      const double tb = __dmul_rn(__dsub_rn(bmax[k], o[k]), inv[k]);
      nk = npmin(ta, tb);
      fk = npmax(ta, tb);
    }
    if (k == 0) { ti = nk; to = fk; } else { ti = npmax(ti, nk); to = npmin(to, fk); }
  }
  t_in = ti;
  t_out = to;
}

// Exit distance only (the `far` of ray_box_range, octree.py:209-211).
__device__ __forceinline__ double ray_box_far(const double o[3], const double d[3], const double inv[3],
                                              const double bmin[3], const double bmax[3]) {
  double to = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double fk;
    if (d[k] == 0.0) {
      fk = ((o[k] >= bmin[k]) && (o[k] <= bmax[k])) ? INFINITY : -INFINITY;
    } else {
      fk = npmax(__dmul_rn(__dsub_rn(bmin[k], o[k]), inv[k]), __dmul_rn(__dsub_rn(bmax[k], o[k]), inv[k]));
    }
    to = (k == 0) ? fk : npmin(to, fk);
  }
  return to;
}

// Per-ray marcher state (BatchMarch, octree.py:222-273).  1/d is cached per
// ray (IEEE division: identical to recomputing it), exits compute only the
// far plane, and for rays whose components are all non-zero the slab faces
// are chosen by the sign of 1/d (no per-axis min/max, no NaN possible).
struct Marcher {
  double o[3], d[3], inv[3], t_max, t_cur, t_end;
  bool active, fast;
  bool pos[3];
  int rounds;

  __device__ void init(const OctDev &t, const double *orig, const double *dir, double tmax, int max_depth) {
    fast = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      o[k] = orig[k];
      d[k] = dir[k];
      inv[k] = 1.0 / d[k];
      pos[k] = inv[k] > 0.0;
      fast = fast && d[k] != 0.0 && isfinite(inv[k]);
    }
    t_max = tmax;
    double t_in, t_out;
    box(o, t.rmin, t.rmax, t_in, t_out);
    t_cur = npmax(t_in, 0.0);
    t_end = npmin(t_out, t_max);
    active = (t_out > t_cur) && (t_cur < t_max) && isfinite(t_cur);
    rounds = 0;
    (void)max_depth;
  }

  // ray_box_range for this ray (fast path: near face chosen by the sign of
  // 1/d, no min/max per axis and no NaN possible)
  __device__ __forceinline__ void box(const double p[3], const double bmin[3], const double bmax[3], double &t_in,
                                      double &t_out) const {
    if (fast) {
      double n[3], f[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        n[k] = __dmul_rn(__dsub_rn(pos[k] ? bmin[k] : bmax[k], p[k]), inv[k]);
        f[k] = __dmul_rn(__dsub_rn(pos[k] ? bmax[k] : bmin[k], p[k]), inv[k]);
      }
      const double a = n[0] > n[1] ? n[0] : n[1];
      t_in = a > n[2] ? a : n[2];
      const double b = f[0] < f[1] ? f[0] : f[1];
      t_out = b < f[2] ? b : f[2];
      return;
    }
    ray_box_inv(p, d, inv, bmin, bmax, t_in, t_out);
  }

  __device__ __forceinline__ double box_far(const double p[3], const double bmin[3], const double bmax[3]) const {
    if (fast) {
      double f[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) f[k] = __dmul_rn(__dsub_rn(pos[k] ? bmax[k] : bmin[k], p[k]), inv[k]);
      const double b = f[0] < f[1] ? f[0] : f[1];
      return b < f[2] ? b : f[2];
    }
    return ray_box_far(p, d, inv, bmin, bmax);
  }

  // query_batch for the cursor (octree.py:136-166): the reference's octant
  // iteration verbatim (u >= 0.5, corner += bit * edge, u <- 2u - bit).  An
  // integer-path descent resuming from cached ancestors was measured slower
  // on B200 (C3: 2.17 ms vs 1.82 ms) -- the loop is latency-, not load-bound.
  __device__ __forceinline__ int32_t descend(const OctDev &t, const double p[3], double corner[3], double &edge,
                                             bool &outside) const {
    return query_point(t, p, corner, edge, outside);
  }

  // One round; returns true and (vid, s0, s1) when a kept leaf segment was found.
  __device__ bool step(const OctDev &t, int64_t &vid, double &s0, double &s1, int32_t &status) {
    if (++rounds > kMaxRounds) {
      status |= kStatusRoundCap;
      active = false;
      return false;
    }
    double p[3], corner[3], edge, cmax[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __dadd_rn(o[k], __dmul_rn(t_cur, d[k]));
    bool outside;
    const int32_t w = descend(t, p, corner, edge, outside);
    if (outside) {
      status |= kStatusOutsideRoot;
      active = false;
      return false;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) cmax[k] = __dadd_rn(corner[k], edge);
    const double far = box_far(p, corner, cmax);
    t_cur = __dadd_rn(t_cur, __dadd_rn(npmax(far, 0.0), kEpsAdvance));
    bool got = false;
    if (w <= -2) {
      double a_in, a_out;
      box(o, corner, cmax, a_in, a_out);
      s0 = npmax(a_in, 0.0);
      s1 = npmin(a_out, t_max);
      if (s1 > __dadd_rn(s0, 1e-12)) {
        vid = (int64_t)(-w - 2);
        got = true;
      }
    }
    if (t_cur >= npmin(t_end, t_max)) active = false;
    return got;
  }
};

struct RaySeg {
  double tm, delta, x[3], s, e, sigma, alpha, om, c[3], a, inv_b;
};

// _evaluate_geometry (render_ray.py:117-133) + eval_color for one segment of
// the ray (o, d) in the frame of the voxel set `sc`.
template <bool kExactColor>
__device__ __forceinline__ void shade_od(const salf_scene_t &sc, const double o[3], const double d[3], int64_t vid,
                                         double s0, double s1, RaySeg &sv, bool want_color) {
  sv.tm = __dmul_rn(0.5, __dadd_rn(s0, s1));
  sv.delta = __dsub_rn(s1, s0);
  const double4 g = ldg_d4(sc.geo + 4 * vid);
  const double4 ax = ldg_d4(sc.aux + 4 * vid);  // (a, 1/b, 2/edge, 0)
  const double ctr[3] = {g.x, g.y, g.z};
  // world_to_local: (p - centre) * (2.0 / edge)  (scene.py:196-209)
#pragma unroll
  for (int k = 0; k < 3; ++k) sv.x[k] = __dmul_rn(__dsub_rn(__dadd_rn(o[k], __dmul_rn(sv.tm, d[k])), ctr[k]), ax.z);
  VoxPrm p;
  load_prm(sc.prm, vid, p);
  sv.a = ax.x;
  sv.inv_b = ax.y;
  sv.s = eval_sdf(p, sv.x);
  sv.sigma = density(sc.density_mode, sv.s, ax.x, ax.y, sv.e);
  sv.alpha = seg_alpha(sv.sigma, sv.delta, sv.om);
  if (want_color) {
    if (kExactColor) eval_color64(p, sv.x, d, sv.c);
    else eval_color32(p, sv.x, d, sv.c);
  }
}

template <bool kExactColor>
__device__ __forceinline__ void shade_seg(const salf_scene_t &sc, const Marcher &m, int64_t vid, double s0,
                                          double s1, RaySeg &sv, bool want_color) {
  shade_od<kExactColor>(sc, m.o, m.d, vid, s0, s1, sv, want_color);
}

// Extra (actor) segment records: 24 doubles each.
enum : int {
  kRecT0 = 0, kRecT1 = 1, kRecTm = 2, kRecDelta = 3, kRecX = 4, kRecS = 7, kRecE = 8, kRecSigma = 9,
  kRecAlpha = 10, kRecOm = 11, kRecC = 12, kRecA = 15, kRecInvB = 16, kRecDir = 17, kRecOwner = 20,
  kRecGvid = 21, kRecStride = 24
};

// Shade segments of rays given in the voxel set's own frame (actor segments,
// render_ray.py:178-197): one record per segment.
template <bool kExactColor>
__global__ void k_shade_segments(salf_scene_t sc, int64_t n, const double *__restrict__ so, const double *__restrict__ sd,
                                 const int64_t *__restrict__ vid, const double *__restrict__ t0,
                                 const double *__restrict__ t1, int32_t owner, int64_t vid_offset,
                                 double *__restrict__ rec) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double o[3] = {so[3 * i], so[3 * i + 1], so[3 * i + 2]}, d[3] = {sd[3 * i], sd[3 * i + 1], sd[3 * i + 2]};
  RaySeg sv;
  shade_od<kExactColor>(sc, o, d, vid[i], t0[i], t1[i], sv, true);
  double *r = rec + i * kRecStride;
  r[kRecT0] = t0[i]; r[kRecT1] = t1[i]; r[kRecTm] = sv.tm; r[kRecDelta] = sv.delta;
  r[kRecX] = sv.x[0]; r[kRecX + 1] = sv.x[1]; r[kRecX + 2] = sv.x[2];
  r[kRecS] = sv.s; r[kRecE] = sv.e; r[kRecSigma] = sv.sigma; r[kRecAlpha] = sv.alpha; r[kRecOm] = sv.om;
  r[kRecC] = sv.c[0]; r[kRecC + 1] = sv.c[1]; r[kRecC + 2] = sv.c[2];
  r[kRecA] = sv.a; r[kRecInvB] = sv.inv_b;
  r[kRecDir] = d[0]; r[kRecDir + 1] = d[1]; r[kRecDir + 2] = d[2];
  r[kRecOwner] = (double)owner; r[kRecGvid] = (double)(vid[i] + vid_offset);
  r[22] = 0.0; r[23] = 0.0;
}

// ---------------------------------------------------------------------------

__global__ void k_query(OctDev t, int64_t n, const double *__restrict__ pts, int8_t *__restrict__ flag,
                        int64_t *__restrict__ vid, double *__restrict__ corner, double *__restrict__ edge,
                        int32_t *__restrict__ outside) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]}, c[3], e;
  bool out;
  int32_t w = query_point(t, p, c, e, out);
  if (out) atomicOr(outside, 1);
  flag[i] = w >= 0 ? 0 : (w == -1 ? -1 : 1);
  vid[i] = w <= -2 ? (int64_t)(-w - 2) : -1;
  corner[3 * i] = c[0]; corner[3 * i + 1] = c[1]; corner[3 * i + 2] = c[2];
  edge[i] = e;
}

// march_batch hit list (count pass when seg_vid == nullptr, fill pass otherwise).
__global__ void k_march(OctDev t, int64_t n, const double *__restrict__ orig, const double *__restrict__ dirs,
                        const double *__restrict__ tmax, salf_scene_t sc, double keep, int early_stop,
                        int64_t *__restrict__ counts, const int64_t *__restrict__ starts, int64_t *__restrict__ seg_vid,
                        double *__restrict__ seg_t0, double *__restrict__ seg_t1, int32_t *__restrict__ status) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Marcher m;
  m.init(t, orig + 3 * i, dirs + 3 * i, tmax ? tmax[i] : INFINITY, t.max_depth);
  int64_t k = 0, off = starts ? starts[i] : 0;
  int32_t st = 0;
  double t_run = 1.0;
  while (m.active) {
    int64_t vid;
    double s0, s1;
    if (!m.step(t, vid, s0, s1, st)) continue;
    if (seg_vid) {
      seg_vid[off + k] = vid;
      seg_t0[off + k] = s0;
      seg_t1[off + k] = s1;
    }
    ++k;
    if (early_stop) {
      RaySeg sv;
      shade_seg<true>(sc, m, vid, s0, s1, sv, false);
      t_run = __dmul_rn(t_run, __dsub_rn(1.0, sv.alpha));
      if (t_run <= keep) break;
    }
  }
  if (!seg_vid) counts[i] = k;
  if (status) status[i] = st;
}

// Fused integrate_rays: march + shade + composite for one ray per thread.
struct LidarFeat {
  const float *feat;  // M x 8 per-voxel LiDAR feature (nullable)
  const float *head;  // 2 x 13: [W_f(8) | W_depth | W_dir(3) | bias] for intensity, drop
  float *out_feat;    // N x 8 alpha-blended feature (nullable)
  float *out_head;    // N x 2 (intensity, ray-drop probability)
  double *out_acc64;  // N x 8 fp64 totals of the exact products w f (nullable; the mixed feature backward's suffix sums)
};

#ifndef SALF_RAY_MINB
#define SALF_RAY_MINB 5  // LiDAR fast forward (measured: 5 beats 4 for the training instantiation)
#endif
#ifndef SALF_RAYX_MINB
#define SALF_RAYX_MINB 4  // fp64 ray forward (parity mode and the redo): 128 registers, no spills
#endif
// kLidar: depth-only rays (render_lidar_ranges never reads colour), plus the
// optional intensity / ray-drop extension.
template <bool kExactColor, bool kLidar, bool kRedo = false>
__global__ void __launch_bounds__(128, SALF_RAYX_MINB) k_ray_forward(OctDev t, salf_scene_t sc, int64_t n,
                                                     const double *__restrict__ orig, const double *__restrict__ dirs,
                                                     const uint8_t *__restrict__ valid, salf_raster_opts_t opt,
                                                     float *__restrict__ out_rgb, float *__restrict__ out_op,
                                                     float *__restrict__ out_depth, double *__restrict__ saved,
                                                     int32_t *__restrict__ status, LidarFeat lf) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (kRedo && !(status[i] & kStatusRedo)) return;  // only the rays the certified pass flagged
  const double keep = 1.0 - opt.stop_threshold;
  double acc_c[3] = {0.0, 0.0, 0.0}, acc_w = 0.0, acc_wt = 0.0, T = 1.0, t_run = 1.0, last_t0 = -INFINITY;
  float acc_f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  double acc_f64[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const bool feat = kLidar && lf.feat != nullptr;
  int64_t n_seg = 0, n_inc = 0;
  int32_t st = 0;
  const bool ok = valid ? valid[i] != 0 : true;
  if (ok) {
    Marcher m;
    m.init(t, orig + 3 * i, dirs + 3 * i, INFINITY, t.max_depth);
    bool frozen = false;
    while (m.active) {
      int64_t vid;
      double s0, s1;
      if (!m.step(t, vid, s0, s1, st)) continue;
      if (s0 < last_t0) st |= kStatusOrder;
      last_t0 = s0;
      ++n_seg;
      RaySeg sv;
      shade_seg<kExactColor>(sc, m, vid, s0, s1, sv, !frozen && !kLidar);
      if (!frozen) {
        if (T > keep) {  // included iff T_before > 1 - stop_threshold (render_ray.py:97-99)
          const double w = __dmul_rn(T, sv.alpha);
          if (!kLidar) {
#pragma unroll
            for (int k = 0; k < 3; ++k) acc_c[k] = __dadd_rn(acc_c[k], __dmul_rn(w, sv.c[k]));
          }
          if (feat) {
            const float4 f0 = __ldg(reinterpret_cast<const float4 *>(lf.feat) + 2 * vid);
            const float4 f1 = __ldg(reinterpret_cast<const float4 *>(lf.feat) + 2 * vid + 1);
            const float wf = (float)w;
            acc_f[0] = fmaf(wf, f0.x, acc_f[0]); acc_f[1] = fmaf(wf, f0.y, acc_f[1]);
            acc_f[2] = fmaf(wf, f0.z, acc_f[2]); acc_f[3] = fmaf(wf, f0.w, acc_f[3]);
            acc_f[4] = fmaf(wf, f1.x, acc_f[4]); acc_f[5] = fmaf(wf, f1.y, acc_f[5]);
            acc_f[6] = fmaf(wf, f1.z, acc_f[6]); acc_f[7] = fmaf(wf, f1.w, acc_f[7]);
            if (lf.out_acc64) {
              const float fv[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
              for (int k = 0; k < 8; ++k) acc_f64[k] = fma(w, (double)fv[k], acc_f64[k]);
            }
          }
          acc_w = __dadd_rn(acc_w, w);
          acc_wt = __dadd_rn(acc_wt, __dmul_rn(w, sv.tm));
          T = __dmul_rn(T, sv.om);
          ++n_inc;
        } else {
          frozen = true;
        }
      }
      // product-based early stop on the march (render_ray.py:154-157)
      t_run = __dmul_rn(t_run, __dsub_rn(1.0, sv.alpha));
      if (t_run <= keep) break;
    }
  }
  if (ok) {
    const double t_fin = T;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (out_rgb) out_rgb[3 * i + k] = (float)__dadd_rn(acc_c[k], __dmul_rn(t_fin, opt.background[k]));
    out_op[i] = (float)__dsub_rn(1.0, t_fin);
    out_depth[i] = acc_w > kDepthWeightMin ? (float)__ddiv_rn(acc_wt, acc_w) : NAN;
  } else {  // render_rays_image: invalid pixels keep the background (render_ray.py:280-293)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (out_rgb) out_rgb[3 * i + k] = (float)opt.background[k];
    out_op[i] = 0.0f;
    out_depth[i] = NAN;
  }
  if (saved) {
    double *s = saved + i * SALF_SAVED_STRIDE;
    s[0] = acc_c[0]; s[1] = acc_c[1]; s[2] = acc_c[2];
    s[3] = acc_w; s[4] = acc_wt; s[5] = T; s[6] = (double)n_seg; s[7] = (double)n_inc;
  }
  if (feat) {
    // linear head on [blended feature, expected depth (0 if none), view dir] + sigmoid
    const float dep = (ok && acc_w > kDepthWeightMin) ? (float)__ddiv_rn(acc_wt, acc_w) : 0.0f;
    const float dv[3] = {(float)dirs[3 * i], (float)dirs[3 * i + 1], (float)dirs[3 * i + 2]};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float *W = lf.head + 13 * j;
      float z = W[12];
#pragma unroll
      for (int k = 0; k < 8; ++k) z = fmaf(W[k], acc_f[k], z);
      z = fmaf(W[8], dep, z);
      z = fmaf(W[9], dv[0], fmaf(W[10], dv[1], fmaf(W[11], dv[2], z)));
      lf.out_head[2 * i + j] = 1.0f / (1.0f + expf(-z));
    }
    if (lf.out_feat) {
#pragma unroll
      for (int k = 0; k < 8; ++k) lf.out_feat[8 * i + k] = acc_f[k];
    }
    if (lf.out_acc64) {
#pragma unroll
      for (int k = 0; k < 8; ++k) lf.out_acc64[8 * i + k] = acc_f64[k];
    }
  }
  if (status) status[i] = st;
}

// Certified mixed-precision ray forward (default mode, no LiDAR features).
// The march (segment list) stays fp64 and bit-exact; per segment only the
// local coordinates x are fp64 (as shade_od), the fields and opacity are fp32
// (MUFU exp, cancellation-free expm1), and the transmittance is
// T = exp(-Y), Y = sum min(sigma delta, ln 1e12) as a compensated fp32 sum with
// a running bound EY on |Y - Y_exact| (model as in salf_raster.cu: x rounded
// to fp32, SDF |ds| <= |w_s|_1 (4e-7), MUFU / rounding terms).  The
// reference's decisions -- inclusion T_before > keep (render_ray.py:97-99),
// the product early stop (:154-157) and depth validity sum w > 0.5
// (:111-112) -- are certified outside the band or the ray is flagged
// (status bit 8) and recomputed by the fp64 kernel (k_ray_forward<.., kRedo>).
#ifndef SALF_RAYF_MINB_CAM
#define SALF_RAYF_MINB_CAM 6  // camera rays (colour): measured best (C4 10.9 -> 9.7 ms)
#endif
template <bool kLidar, bool kSdf, bool kFeat = false, bool kTot64 = true>
__global__ void __launch_bounds__(128, kLidar ? SALF_RAY_MINB : SALF_RAYF_MINB_CAM) k_ray_forward_fast(
    OctDev t, salf_scene_t sc, int64_t n, const double *__restrict__ orig, const double *__restrict__ dirs,
    const uint8_t *__restrict__ valid, salf_raster_opts_t opt, float *__restrict__ out_rgb,
    float *__restrict__ out_op, float *__restrict__ out_depth, double *__restrict__ saved,
    int32_t *__restrict__ status, LidarFeat lf) {
  double acc_f[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // fp64 totals of the exact products w f
  constexpr bool feat = kLidar && kFeat;  // the extension is a separate instantiation (no per-segment test)
  constexpr float kU = 5.9604645e-8f;  // 2^-24
  constexpr double kLn2 = 0.6931471805599453;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double y_stop_d = -log(1.0 - opt.stop_threshold);
  const float y_stop = (float)y_stop_d, y_stop_err = (float)fabs(y_stop_d - (double)y_stop);
  // kTot64 (a backward follows): fp64 totals of the exact fp32 products w c, w,
  // w t_mid -- the mixed backward rebuilds its suffix sums from them
  // (seg_grad_f32); without saved state (inference) plain fp32 sums.  T = exp(-Y)
  // exactly as the backward recomputes it (also for the first segment)
  using Acc = typename std::conditional<kTot64, double, float>::type;
  float T = fast_exp(-0.f), EY = 0.f, Yh = 0.f, Yc = 0.f;
  Acc acc_c[3] = {0, 0, 0}, acc_w = 0, acc_wt = 0;
  double last_t0 = -INFINITY;
  int64_t n_seg = 0, n_inc = 0;
  int32_t st = 0;
  bool flag = false;
  const bool ok = valid ? valid[i] != 0 : true;
  if (ok) {
    Marcher m;
    m.init(t, orig + 3 * i, dirs + 3 * i, INFINITY, t.max_depth);
    while (m.active) {
      int64_t vid;
      double s0, s1;
      if (!m.step(t, vid, s0, s1, st)) continue;
      if (s0 < last_t0) st |= kStatusOrder;
      last_t0 = s0;
      ++n_seg;
      // inclusion: T_before > keep  <=>  Y_before < y_stop (certified outside the band)
      const float Ys = Yh + Yc;
      const float band = __fmaf_rn(2.f, EY, __fmaf_rn(4.f * kU, Ys, y_stop_err + 1e-9f));
      if (fabsf(y_stop - Ys) <= band) flag = true;
      if (!(Ys < y_stop)) break;  // frozen: the reference's march would already have stopped
      const double tm = __dmul_rn(0.5, __dadd_rn(s0, s1));
      const float delta = (float)__dsub_rn(s1, s0);
      const double4 g = ldg_d4(sc.geo + 4 * vid);
      const double4 ax = ldg_d4(sc.aux + 4 * vid);  // (a, 1/b, 2/edge, 0)
      const double ctr[3] = {g.x, g.y, g.z};
      float x[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        x[k] = (float)__dmul_rn(__dsub_rn(__dadd_rn(m.o[k], __dmul_rn(tm, m.d[k])), ctr[k]), ax.z);
      VoxPrm p;
      load_prm(sc.prm, vid, p);
      const float wn = fabsf(p.ws[0]) + fabsf(p.ws[1]) + fabsf(p.ws[2]) + fabsf(p.ws[3]);
      const float a = (float)ax.x, inv_b = (float)ax.y;
      SegF32 f;
      seg_fields_f32<kSdf>(p, a, inv_b, x, delta, f);
      const float sigma = f.sigma, y = f.y, alpha = f.alpha;
      const float rel = kSdf ? __fmaf_rn(wn * 4e-7f, inv_b, __fmaf_rn(3e-7f, fabsf(f.s) * inv_b, 5.4e-7f))
                             : __fmaf_rn(wn, 4e-7f, __fmaf_rn(3e-7f, fabsf(f.s), 5.4e-7f));
      (void)sigma;
      const float w = T * alpha;
      const double wd = (double)w;
      if (!kLidar) {
        float col[3];
        const float gam[4] = {(float)kShC0, (float)(kShC1 * m.d[1]), (float)(kShC1 * m.d[2]),
                              (float)(kShC1 * m.d[0])};
        eval_color32g(p, x, gam, col);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if constexpr (kTot64) acc_c[k] = fma(wd, (double)col[k], acc_c[k]);
          else acc_c[k] = __fmaf_rn(w, col[k], acc_c[k]);
        }
      }
      if (feat) {  // intensity / ray-drop extension: blended 8-channel feature
        const float4 f0 = __ldg(reinterpret_cast<const float4 *>(lf.feat) + 2 * vid);
        const float4 f1 = __ldg(reinterpret_cast<const float4 *>(lf.feat) + 2 * vid + 1);
        const float fv[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) acc_f[k] = fma(wd, (double)fv[k], acc_f[k]);
      }
      if constexpr (kTot64) {
        acc_w = __dadd_rn(acc_w, wd);
        acc_wt = fma(wd, tm, acc_wt);
      } else {
        acc_w += w;
        acc_wt = __fmaf_rn(w, (float)tm, acc_wt);
      }
      EY += y * (rel + 2.f * kU);
      neumaier_add(Yh, Yc, y);
      T = fast_exp(-(Yh + Yc));
      ++n_inc;
      // product early stop after this segment: prod(1 - alpha) <= keep  <=>  Y >= y_stop
      const float Ya = Yh + Yc;
      if (fabsf(y_stop - Ya) <= __fmaf_rn(2.f, EY, __fmaf_rn(4.f * kU, Ya, y_stop_err + 1e-9f))) flag = true;
      if (Ya >= y_stop) break;
    }
  }
  const double Y = (double)Yh + (double)Yc;
  if (ok && fabs(Y - kLn2) <= (double)__fmaf_rn(2.f, EY, __fmaf_rn(4.f * kU, (float)Y, 1e-9f))) flag = true;
  const bool vdepth = ok && Y > kLn2;  // sum w = 1 - T_final > 0.5
  // the saved (raw) weight sum must take the same side of 0.5 as the certified Y
  if (ok && (acc_w > kDepthWeightMin) != vdepth) flag = true;
  if (ok) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (out_rgb) out_rgb[3 * i + k] = (float)fma((double)T, opt.background[k], (double)acc_c[k]);
    out_op[i] = (float)(-expm1(-Y));  // 1 - T without cancellation near T = 1
    out_depth[i] = vdepth ? (float)__ddiv_rn((double)acc_wt, (double)acc_w) : NAN;
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (out_rgb) out_rgb[3 * i + k] = (float)opt.background[k];
    out_op[i] = 0.0f;
    out_depth[i] = NAN;
  }
  if (saved) {
    double *sv = saved + i * SALF_SAVED_STRIDE;
    sv[0] = acc_c[0]; sv[1] = acc_c[1]; sv[2] = acc_c[2];
    sv[3] = acc_w; sv[4] = acc_wt;  // raw sums (the backward's suffix sums need them bit for bit)
    sv[5] = T; sv[6] = (double)n_seg; sv[7] = (double)n_inc;
  }
  if (feat) {
    // linear head on [blended feature, expected depth (0 if none), view dir] + sigmoid (as k_ray_forward)
    const float dep = vdepth ? (float)__ddiv_rn((double)acc_wt, (double)acc_w) : 0.0f;
    const float dv[3] = {(float)dirs[3 * i], (float)dirs[3 * i + 1], (float)dirs[3 * i + 2]};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float *W = lf.head + 13 * j;
      float z = W[12];
#pragma unroll
      for (int k = 0; k < 8; ++k) z = fmaf(W[k], (float)acc_f[k], z);
      z = fmaf(W[8], dep, z);
      z = fmaf(W[9], dv[0], fmaf(W[10], dv[1], fmaf(W[11], dv[2], z)));
      lf.out_head[2 * i + j] = 1.0f / (1.0f + expf(-z));
    }
    if (lf.out_feat) {
#pragma unroll
      for (int k = 0; k < 8; ++k) lf.out_feat[8 * i + k] = (float)acc_f[k];
    }
    if (lf.out_acc64) {
#pragma unroll
      for (int k = 0; k < 8; ++k) lf.out_acc64[8 * i + k] = acc_f[k];
    }
  }
  if (status) status[i] = st | (flag ? kStatusRedo : 0);
}

// Ray backward: warp-synchronous re-march (every lane advances one round per
// iteration, as BatchMarch does) so gradient scatters run with the full warp.
struct FeatGrad {
  const float *feat;    // M x 8 per-voxel LiDAR feature (nullptr: no feature terms)
  const double *dF;     // N x 8 dL/dF of the blended feature
  const double *Facc;   // N x 8 blended feature of the forward
  double *feat_grad;    // M x 8 dL/dfeature (accumulated)
};

// Deterministic mode: each included segment's 27-row goes to its own slot
// (row_start[ray] + k-th included segment) instead of the atomic scatter;
// salf::det_reduce_rows then sums the rows per voxel in a fixed order.
struct RowSink {
  float *rows;               // (slots, 27) or nullptr (atomic mode)
  uint32_t *row_vid;         // (slots,) voxel of each used slot (unused: n_vox)
  const int64_t *row_start;  // (n + 1,) exclusive scan of the forward's segment counts
};

// kMixed (default mode, no LiDAR features): inclusion is the forward's
// included-segment count saved[:, 7] (the certified forward's decisions equal
// the fp64 ones), the march stays fp64 and bit-exact, and the segment fields
// and gradient chain are fp32 (seg_grad_f32); kSdf selects the density.
#ifndef SALF_RAYB_MINB
#define SALF_RAYB_MINB 4  // 128 registers: measured best (5, 6 spill)
#endif
template <bool kExactColor, bool kMixed = false, bool kSdf = true, bool kColor = true, bool kFeat = false>
__global__ void __launch_bounds__(128, kMixed ? SALF_RAYB_MINB : 1) k_ray_backward(OctDev t, salf_scene_t sc, int64_t n,
                                                      const double *__restrict__ orig, const double *__restrict__ dirs,
                                                      const uint8_t *__restrict__ valid, salf_raster_opts_t opt,
                                                      const double *__restrict__ saved, const double *__restrict__ d_rgb,
                                                      const double *__restrict__ d_depth, double *__restrict__ grad,
                                                      FeatGrad fg, RowSink sink) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double keep = 1.0 - opt.stop_threshold;
  bool live = i < n && (valid ? valid[i] != 0 : true);
  Marcher m;
  m.active = false;
  double dC[3] = {0, 0, 0}, total = 0.0, tail = 0.0, D = 0.0, dd = 0.0, ws = 1.0, prefix = 0.0, T = 1.0,
         t_run = 1.0;
  double dF[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (live) {
    m.init(t, orig + 3 * i, dirs + 3 * i, INFINITY, t.max_depth);
    const double *s = saved + i * SALF_SAVED_STRIDE;
    for (int k = 0; k < 3; ++k) dC[k] = d_rgb ? d_rgb[3 * i + k] : 0.0;
    const double acc_w = s[3], acc_wt = s[4];
    const bool okd = acc_w > kDepthWeightMin;
    dd = okd ? d_depth[i] : 0.0;
    D = okd ? __ddiv_rn(acc_wt, acc_w) : 0.0;
    ws = okd ? acc_w : 1.0;
    total = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(dC[0], s[0]), __dmul_rn(dC[2], s[2])), __dmul_rn(dC[1], s[1])),
                      __ddiv_rn(__dmul_rn(dd, __dsub_rn(acc_wt, __dmul_rn(D, acc_w))), ws));
    tail = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(dC[0], opt.background[0]), __dmul_rn(dC[2], opt.background[2])),
                               __dmul_rn(dC[1], opt.background[1])),
                     s[5]);
    live = m.active && (dC[0] != 0.0 || dC[1] != 0.0 || dC[2] != 0.0 || dd != 0.0);
    if (fg.feat) {
      // the blended feature F = sum w_i f_i enters like a colour without background
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        dF[k] = fg.dF[8 * i + k];
        total = __dadd_rn(total, __dmul_rn(dF[k], fg.Facc[8 * i + k]));
        live = live || (m.active && dF[k] != 0.0);
      }
    }
  }
  // kFeat (mixed): CF = dF . Facc with Facc the forward's fp64 totals; PF runs over the segments
  double CF = 0.0, PF = 0.0;
  if (kMixed && kFeat && i < n && fg.feat) {
#pragma unroll
    for (int k = 0; k < 8; ++k) CF = fma(dF[k], fg.Facc[8 * i + k], CF);
  }
  int64_t n_inc = 0, n_done = 0;
  RayBwdState rs;
  float dCf[3] = {(float)dC[0], (float)dC[1], (float)dC[2]};
  const float dwsf = (float)(dd / ws), tailf = (float)tail;
  float gam[4] = {0.f, 0.f, 0.f, 0.f};
  if (kMixed && live) {
    const double *s = saved + i * SALF_SAVED_STRIDE;
    n_inc = (int64_t)s[7];
    if (n_inc == 0) live = false;
    rs.Yh = 0.f;
    rs.Yc = 0.f;
    rs.Pw = rs.Pwt = 0.0;
    rs.Aw = s[3];
    rs.Awt = s[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      rs.Pc[k] = 0.0;
      rs.Ac[k] = s[k];
    }
    gam[0] = (float)kShC0;
    gam[1] = (float)(kShC1 * m.d[1]);
    gam[2] = (float)(kShC1 * m.d[2]);
    gam[3] = (float)(kShC1 * m.d[0]);
  }
  int32_t st = 0;
  int64_t slot = (sink.rows && i < n) ? sink.row_start[i] : 0;
  const int64_t slot_end = (sink.rows && i < n) ? sink.row_start[i + 1] : 0;
  const bool want_color = dC[0] != 0.0 || dC[1] != 0.0 || dC[2] != 0.0;
  while (__any_sync(0xffffffffu, live)) {
    bool act = false;
    int64_t vid = 0;
    float g[32];
    if (live) {
      double s0, s1;
      if (kMixed) {
        if (m.step(t, vid, s0, s1, st)) {
          // fp64: t_mid, delta, local coordinates (shade_od); fp32 after
          const double tm = __dmul_rn(0.5, __dadd_rn(s0, s1));
          const double4 gg = ldg_d4(sc.geo + 4 * vid);
          const double4 ax = ldg_d4(sc.aux + 4 * vid);
          const double ctr[3] = {gg.x, gg.y, gg.z};
          float x[3];
#pragma unroll
          for (int k = 0; k < 3; ++k)
            x[k] = (float)__dmul_rn(__dsub_rn(__dadd_rn(m.o[k], __dmul_rn(tm, m.d[k])), ctr[k]), ax.z);
          VoxPrm p;
          load_prm(sc.prm, vid, p);
          if (kFeat) {
            const float4 f0 = __ldg(reinterpret_cast<const float4 *>(fg.feat) + 2 * vid);
            const float4 f1 = __ldg(reinterpret_cast<const float4 *>(fg.feat) + 2 * vid + 1);
            const float fv[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            double fdot = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) fdot = fma(dF[k], (double)fv[k], fdot);
            const float w = seg_grad_f32<kSdf, kColor, true>(p, (float)ax.x, (float)ax.y, x,
                                                             (float)__dsub_rn(s1, s0), tm, D, gam, want_color, dCf,
                                                             dwsf, tailf, rs, g, fdot, &PF, CF);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (dF[k] != 0.0) atomicAdd(fg.feat_grad + 8 * vid + k, __dmul_rn((double)w, dF[k]));
          } else {
            seg_grad_f32<kSdf, kColor>(p, (float)ax.x, (float)ax.y, x, (float)__dsub_rn(s1, s0), tm, D, gam,
                                       want_color, dCf, dwsf, tailf, rs, g);
          }
          act = true;
          if (++n_done >= n_inc) live = false;
        }
      } else if (m.step(t, vid, s0, s1, st)) {
        RaySeg sv;
        sv.c[0] = sv.c[1] = sv.c[2] = 0.0;  // depth-only rays (LiDAR): no colour term
        shade_seg<kExactColor>(sc, m, vid, s0, s1, sv, want_color);
        const double a = sv.alpha;
        const double tb = T;
        if (tb > keep) {
          const double w = __dmul_rn(tb, a);
          double A = __dadd_rn(
              __dadd_rn(__dadd_rn(__dmul_rn(dC[0], sv.c[0]), __dmul_rn(dC[2], sv.c[2])), __dmul_rn(dC[1], sv.c[1])),
              __ddiv_rn(__dmul_rn(dd, __dsub_rn(sv.tm, D)), ws));
          if (fg.feat) {
            const float4 f0 = __ldg(reinterpret_cast<const float4 *>(fg.feat) + 2 * vid);
            const float4 f1 = __ldg(reinterpret_cast<const float4 *>(fg.feat) + 2 * vid + 1);
            const double f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              A = __dadd_rn(A, __dmul_rn(dF[k], f[k]));
              if (dF[k] != 0.0) atomicAdd(fg.feat_grad + 8 * vid + k, __dmul_rn(w, dF[k]));
            }
          }
          prefix = __dadd_rn(prefix, __dmul_rn(A, w));
          const double suffix = __dsub_rn(total, prefix);
          segment_grad(sc.density_mode, sv.delta, sv.sigma, sv.alpha, sv.om, sv.s, sv.e, sv.a, sv.inv_b, sv.x, sv.c,
                       m.d, A, tb, w, suffix, tail, dC, g);
          act = true;
          T = __dmul_rn(T, sv.om);
          t_run = __dmul_rn(t_run, __dsub_rn(1.0, a));
          if (t_run <= keep) live = false;
        } else {
          live = false;  // every later segment is excluded
        }
      }
      if (!m.active) live = false;
    }
    if (sink.rows) {
      if (act && slot < slot_end) {
        float *dst = sink.rows + slot * kGradStride;
#pragma unroll
        for (int k = 0; k < kGradStride; ++k) dst[k] = g[k];
        sink.row_vid[slot] = (uint32_t)vid;
        ++slot;
      }
    } else {
      scatter_grad(grad, vid, act, g);
    }
  }
}


// integrate_rays with live actors (render_ray.py:161-239): the static march
// runs without early stop (:175) and is merged, in the reference's
// lexsort((vid, owner, t0, ray)) order, with the ray's pre-shaded actor
// segments (CSR ex_start / ex_rec).  Static wins ties at equal t0 (owner -1).
template <bool kExactColor>
__global__ void __launch_bounds__(128) k_ray_forward_merge(OctDev t, salf_scene_t sc, int64_t n,
                                                           const double *__restrict__ orig,
                                                           const double *__restrict__ dirs,
                                                           const uint8_t *__restrict__ valid, salf_raster_opts_t opt,
                                                           const int64_t *__restrict__ ex_start,
                                                           const double *__restrict__ ex_rec,
                                                           float *__restrict__ out_rgb, float *__restrict__ out_op,
                                                           float *__restrict__ out_depth, double *__restrict__ saved,
                                                           int32_t *__restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double keep = 1.0 - opt.stop_threshold;
  double acc_c[3] = {0.0, 0.0, 0.0}, acc_w = 0.0, acc_wt = 0.0, T = 1.0;
  int64_t n_seg = 0;
  int32_t st = 0;
  const bool ok = valid ? valid[i] != 0 : true;
  if (ok) {
    Marcher m;
    m.init(t, orig + 3 * i, dirs + 3 * i, INFINITY, t.max_depth);
    int64_t k = ex_start[i];
    const int64_t kend = ex_start[i + 1];
    bool have = false, frozen = false;
    int64_t vid = 0;
    double s0 = 0.0, s1 = 0.0;
    while (true) {
      while (!have && m.active) have = m.step(t, vid, s0, s1, st);
      const bool take_static = have && (k >= kend || !(ex_rec[k * kRecStride + kRecT0] < s0));
      if (!take_static && k >= kend) break;
      double alpha, om, tm, c[3];
      if (take_static) {
        RaySeg sv;
        shade_seg<kExactColor>(sc, m, vid, s0, s1, sv, !frozen);
        alpha = sv.alpha; om = sv.om; tm = sv.tm; c[0] = sv.c[0]; c[1] = sv.c[1]; c[2] = sv.c[2];
        have = false;
      } else {
        const double *r = ex_rec + k * kRecStride;
        alpha = r[kRecAlpha]; om = r[kRecOm]; tm = r[kRecTm]; c[0] = r[kRecC]; c[1] = r[kRecC + 1]; c[2] = r[kRecC + 2];
        ++k;
      }
      ++n_seg;
      if (!frozen) {
        if (T > keep) {
          const double w = __dmul_rn(T, alpha);
#pragma unroll
          for (int q = 0; q < 3; ++q) acc_c[q] = __dadd_rn(acc_c[q], __dmul_rn(w, c[q]));
          acc_w = __dadd_rn(acc_w, w);
          acc_wt = __dadd_rn(acc_wt, __dmul_rn(w, tm));
          T = __dmul_rn(T, om);
        } else {
          frozen = true;  // later segments are excluded; keep marching for the status only
          break;
        }
      }
    }
  }
  if (ok) {
#pragma unroll
    for (int q = 0; q < 3; ++q) out_rgb[3 * i + q] = (float)__dadd_rn(acc_c[q], __dmul_rn(T, opt.background[q]));
    out_op[i] = (float)__dsub_rn(1.0, T);
    out_depth[i] = acc_w > kDepthWeightMin ? (float)__ddiv_rn(acc_wt, acc_w) : NAN;
  } else {
#pragma unroll
    for (int q = 0; q < 3; ++q) out_rgb[3 * i + q] = (float)opt.background[q];
    out_op[i] = 0.0f;
    out_depth[i] = NAN;
  }
  if (saved) {
    double *s = saved + i * SALF_SAVED_STRIDE;
    s[0] = acc_c[0]; s[1] = acc_c[1]; s[2] = acc_c[2];
    s[3] = acc_w; s[4] = acc_wt; s[5] = T; s[6] = (double)n_seg; s[7] = 0.0;
  }
  if (status) status[i] = st;
}

// Backward of k_ray_forward_merge: static segments re-marched (grad), actor
// segments from their records (ex_grad, indexed by the global actor voxel id).
// Warp-synchronous: each iteration a lane either advances its marcher or
// consumes one segment.
template <bool kExactColor>
__global__ void __launch_bounds__(128) k_ray_backward_merge(OctDev t, salf_scene_t sc, int64_t n,
                                                            const double *__restrict__ orig,
                                                            const double *__restrict__ dirs,
                                                            const uint8_t *__restrict__ valid, salf_raster_opts_t opt,
                                                            const int64_t *__restrict__ ex_start,
                                                            const double *__restrict__ ex_rec,
                                                            const double *__restrict__ saved,
                                                            const double *__restrict__ d_rgb,
                                                            const double *__restrict__ d_depth,
                                                            double *__restrict__ grad, double *__restrict__ ex_grad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double keep = 1.0 - opt.stop_threshold;
  bool live = i < n && (valid ? valid[i] != 0 : true);
  Marcher m;
  m.active = false;
  double dC[3] = {0, 0, 0}, total = 0.0, tail = 0.0, D = 0.0, dd = 0.0, ws = 1.0, prefix = 0.0, T = 1.0;
  int64_t k = 0, kend = 0;
  if (live) {
    m.init(t, orig + 3 * i, dirs + 3 * i, INFINITY, t.max_depth);
    k = ex_start[i];
    kend = ex_start[i + 1];
    const double *s = saved + i * SALF_SAVED_STRIDE;
    for (int q = 0; q < 3; ++q) dC[q] = d_rgb[3 * i + q];
    const double acc_w = s[3], acc_wt = s[4];
    const bool okd = acc_w > kDepthWeightMin;
    dd = okd ? d_depth[i] : 0.0;
    D = okd ? __ddiv_rn(acc_wt, acc_w) : 0.0;
    ws = okd ? acc_w : 1.0;
    total = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(dC[0], s[0]), __dmul_rn(dC[2], s[2])), __dmul_rn(dC[1], s[1])),
                      __ddiv_rn(__dmul_rn(dd, __dsub_rn(acc_wt, __dmul_rn(D, acc_w))), ws));
    tail = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(dC[0], opt.background[0]), __dmul_rn(dC[2], opt.background[2])),
                               __dmul_rn(dC[1], opt.background[1])),
                     s[5]);
    live = (m.active || k < kend) && (dC[0] != 0.0 || dC[1] != 0.0 || dC[2] != 0.0 || dd != 0.0);
  }
  int32_t st = 0;
  bool have = false;
  int64_t svid = 0;
  double s0 = 0.0, s1 = 0.0;
  while (__any_sync(0xffffffffu, live)) {
    bool act_s = false, act_x = false;
    int64_t gv = 0;
    float g[32];
    if (live) {
      if (!have && m.active) {
        have = m.step(t, svid, s0, s1, st);  // marcher advance only this iteration
      } else {
        const bool take_static = have && (k >= kend || !(ex_rec[k * kRecStride + kRecT0] < s0));
        if (!take_static && k >= kend) {
          live = false;
        } else {
          double tm, delta, x[3], ss, e, sigma, a, om, c[3], aa, ib, dir[3];
          if (take_static) {
            RaySeg sv;
            shade_seg<kExactColor>(sc, m, svid, s0, s1, sv, true);
            tm = sv.tm; delta = sv.delta; ss = sv.s; e = sv.e; sigma = sv.sigma; a = sv.alpha; om = sv.om;
            aa = sv.a; ib = sv.inv_b;
            for (int q = 0; q < 3; ++q) { x[q] = sv.x[q]; c[q] = sv.c[q]; dir[q] = m.d[q]; }
            gv = svid;
            have = false;
          } else {
            const double *r = ex_rec + k * kRecStride;
            tm = r[kRecTm]; delta = r[kRecDelta]; ss = r[kRecS]; e = r[kRecE]; sigma = r[kRecSigma];
            a = r[kRecAlpha]; om = r[kRecOm]; aa = r[kRecA]; ib = r[kRecInvB];
            for (int q = 0; q < 3; ++q) { x[q] = r[kRecX + q]; c[q] = r[kRecC + q]; dir[q] = r[kRecDir + q]; }
            gv = (int64_t)r[kRecGvid];
            ++k;
          }
          if (T > keep) {
            const double w = __dmul_rn(T, a);
            const double A = __dadd_rn(
                __dadd_rn(__dadd_rn(__dmul_rn(dC[0], c[0]), __dmul_rn(dC[2], c[2])), __dmul_rn(dC[1], c[1])),
                __ddiv_rn(__dmul_rn(dd, __dsub_rn(tm, D)), ws));
            prefix = __dadd_rn(prefix, __dmul_rn(A, w));
            const double suffix = __dsub_rn(total, prefix);
            segment_grad(sc.density_mode, delta, sigma, a, om, ss, e, aa, ib, x, c, dir, A, T, w, suffix, tail, dC, g);
            if (take_static) act_s = true; else act_x = true;
            T = __dmul_rn(T, om);
          } else {
            live = false;
          }
        }
      }
    }
    scatter_grad(grad, gv, act_s, g);
    scatter_grad(ex_grad, gv, act_x, g);
  }
}

}  // namespace salf

using namespace salf;

// Jump table for the descent (see salf_b200.h): one thread per depth-K cell
// walks the reference's levels (child = b0 + 2 b1 + 4 b2, octree.py:152-163);
// thread 0..3*2^K-1 of the second kernel accumulate the per-axis corners in
// the descent's order (edge halved, then corner += bit ? edge : 0).
__global__ void k_jump_words(const int32_t *__restrict__ nodes, int K, int32_t *__restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ((int64_t)1 << (3 * K))) return;
  const uint32_t mask = (1u << K) - 1;
  const uint32_t cx = (uint32_t)(c >> (2 * K)) & mask, cy = (uint32_t)(c >> K) & mask, cz = (uint32_t)c & mask;
  int32_t w = nodes[0];
  for (int l = 0; l < K; ++l) {
    if (w < 0) {
      w = kJumpNone;
      break;
    }
    const int sh = K - 1 - l;
    w = nodes[w + ((cx >> sh) & 1) + 2 * ((cy >> sh) & 1) + 4 * ((cz >> sh) & 1)];
  }
  out[c] = w;
}

__global__ void k_jump_corners(double r0, double r1, double r2, double root_edge, int K, double *__restrict__ out) {
  const int n = 1 << K;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  const int axis = i / n, pre = i - axis * n;
  double corner = axis == 0 ? r0 : (axis == 1 ? r1 : r2), edge = root_edge;
  for (int l = 0; l < K; ++l) {
    edge = __dmul_rn(edge, 0.5);
    corner = __dadd_rn(corner, ((pre >> (K - 1 - l)) & 1) ? edge : 0.0);
  }
  out[i] = corner;
}

extern "C" int salf_octree_query(const salf_octree_t *tree, int64_t n, const double *p, int8_t *flag, int64_t *vid,
                                 double *corner, double *edge, int32_t *out_of_root, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    OctDev t = make_oct(tree);
    k_query<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(t, n, p, flag, vid, corner, edge,
                                                                             out_of_root);
    return check_cuda("salf_octree_query");
  }
  SALF_CATCH
}

extern "C" int salf_march(const salf_octree_t *tree, int64_t n, const double *origins, const double *dirs,
                          const double *t_max, const salf_scene_t *scene, double stop_threshold, int32_t early_stop,
                          int64_t *counts, const int64_t *starts, int64_t *seg_vid, double *seg_t0, double *seg_t1,
                          int32_t *status, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    OctDev t = make_oct(tree);
    salf_scene_t sc = scene ? *scene : salf_scene_t{};
    if (early_stop && !scene) return set_error(SALF_EINVAL, "early stop needs the scene");
    k_march<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        t, n, origins, dirs, t_max, sc, 1.0 - stop_threshold, early_stop, counts, starts, seg_vid, seg_t0, seg_t1,
        status);
    return check_cuda("salf_march");
  }
  SALF_CATCH
}

extern "C" int salf_ray_forward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n, const double *origins,
                                const double *dirs, const uint8_t *valid, const salf_raster_opts_t *opts,
                                float *out_rgb, float *out_opacity, float *out_depth, double *saved, int32_t *status,
                                void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    LidarFeat lf{nullptr, nullptr, nullptr, nullptr, nullptr};
    if (opts->exact_color)
      k_ray_forward<true, false><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, valid, *opts,
                                                                           out_rgb, out_opacity, out_depth, saved,
                                                                           status, lf);
    else {
      // certified mixed precision, then fp64 recomputation of the flagged rays
      if (!status) return set_error(SALF_EINVAL, "the mixed-precision ray forward needs a status buffer");
      cudaStream_t st = (cudaStream_t)stream;
      const bool sdf = scene->density_mode == SALF_DENSITY_SDF;
      if (!saved) {  // inference (no backward follows): fp32 totals
        if (sdf)
          k_ray_forward_fast<false, true, false, false><<<grid, 128, 0, st>>>(
              t, *scene, n, origins, dirs, valid, *opts, out_rgb, out_opacity, out_depth, nullptr, status, lf);
        else
          k_ray_forward_fast<false, false, false, false><<<grid, 128, 0, st>>>(
              t, *scene, n, origins, dirs, valid, *opts, out_rgb, out_opacity, out_depth, nullptr, status, lf);
      } else if (sdf) {
        k_ray_forward_fast<false, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, valid, *opts, out_rgb,
                                                              out_opacity, out_depth, saved, status, lf);
      } else {
        k_ray_forward_fast<false, false><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, valid, *opts, out_rgb,
                                                               out_opacity, out_depth, saved, status, lf);
      }
      static const bool no_redo = getenv("SALF_NO_REDO") && getenv("SALF_NO_REDO")[0] == '1';  // diagnostics
      if (!no_redo)
        k_ray_forward<false, false, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, valid, *opts, out_rgb,
                                                                out_opacity, out_depth, saved, status, lf);
    }
    return check_cuda("salf_ray_forward");
  }
  SALF_CATCH
}

extern "C" int salf_lidar_forward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                  const double *origins, const double *dirs, const salf_raster_opts_t *opts,
                                  const float *feat, const float *head, float *out_depth, float *out_opacity,
                                  float *out_feat, float *out_head, double *feat_acc64, double *saved,
                                  int32_t *status, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    if (feat && !head) return set_error(SALF_EINVAL, "LiDAR features need the 2 x 13 head");
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    LidarFeat lf{feat, head, out_feat, out_head, feat_acc64};
    cudaStream_t st = (cudaStream_t)stream;
    if (status && !opts->exact_color) {
      // certified mixed precision + fp64 redo of flagged rays (features blended in fp32 either way)
      const bool sdf = scene->density_mode == SALF_DENSITY_SDF;
      if (feat) {
        if (sdf)
          k_ray_forward_fast<true, true, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, nullptr, *opts,
                                                                     nullptr, out_opacity, out_depth, saved, status, lf);
        else
          k_ray_forward_fast<true, false, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, nullptr, *opts,
                                                                      nullptr, out_opacity, out_depth, saved, status, lf);
      } else if (!saved) {  // inference (no backward follows): fp32 totals
        if (sdf)
          k_ray_forward_fast<true, true, false, false><<<grid, 128, 0, st>>>(
              t, *scene, n, origins, dirs, nullptr, *opts, nullptr, out_opacity, out_depth, nullptr, status, lf);
        else
          k_ray_forward_fast<true, false, false, false><<<grid, 128, 0, st>>>(
              t, *scene, n, origins, dirs, nullptr, *opts, nullptr, out_opacity, out_depth, nullptr, status, lf);
      } else if (sdf) {
        k_ray_forward_fast<true, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, nullptr, *opts, nullptr,
                                                             out_opacity, out_depth, saved, status, lf);
      } else {
        k_ray_forward_fast<true, false><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, nullptr, *opts, nullptr,
                                                              out_opacity, out_depth, saved, status, lf);
      }
      static const bool no_redo = getenv("SALF_NO_REDO") && getenv("SALF_NO_REDO")[0] == '1';  // diagnostics
      if (!no_redo)
        k_ray_forward<false, true, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, nullptr, *opts, nullptr,
                                                               out_opacity, out_depth, saved, status, lf);
    } else {
      k_ray_forward<false, true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, nullptr, *opts, nullptr,
                                                       out_opacity, out_depth, saved, status, lf);
    }
    return check_cuda("salf_lidar_forward");
  }
  SALF_CATCH
}

// Mixed-precision ray backward: density mode and colour seeds (d_rgb == NULL:
// depth-only, e.g. LiDAR) select the instantiation.
static void launch_ray_backward_mixed(bool sdf, bool color, unsigned grid, cudaStream_t st, const OctDev &t,
                                      const salf_scene_t &sc, int64_t n, const double *o, const double *d,
                                      const uint8_t *valid, const salf_raster_opts_t &opts, const double *saved,
                                      const double *d_rgb, const double *d_depth, double *grad, FeatGrad fg,
                                      RowSink sink) {
  if (sdf && color)
    k_ray_backward<false, true, true, true><<<grid, 128, 0, st>>>(t, sc, n, o, d, valid, opts, saved, d_rgb, d_depth,
                                                                  grad, fg, sink);
  else if (sdf)
    k_ray_backward<false, true, true, false><<<grid, 128, 0, st>>>(t, sc, n, o, d, valid, opts, saved, d_rgb,
                                                                   d_depth, grad, fg, sink);
  else if (color)
    k_ray_backward<false, true, false, true><<<grid, 128, 0, st>>>(t, sc, n, o, d, valid, opts, saved, d_rgb,
                                                                   d_depth, grad, fg, sink);
  else
    k_ray_backward<false, true, false, false><<<grid, 128, 0, st>>>(t, sc, n, o, d, valid, opts, saved, d_rgb,
                                                                    d_depth, grad, fg, sink);
}

extern "C" int salf_ray_backward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                 const double *origins, const double *dirs, const uint8_t *valid,
                                 const salf_raster_opts_t *opts, const double *saved, const double *d_rgb,
                                 const double *d_depth, double *grad, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    FeatGrad fg{nullptr, nullptr, nullptr, nullptr};
    if (opts->exact_color)
      k_ray_backward<true><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, valid, *opts, saved,
                                                                     d_rgb, d_depth, grad, fg, RowSink{});
    else
      launch_ray_backward_mixed(scene->density_mode == SALF_DENSITY_SDF, d_rgb != nullptr, grid,
                                (cudaStream_t)stream, t, *scene, n, origins, dirs, valid, *opts, saved, d_rgb,
                                d_depth, grad, fg, RowSink{});
    return check_cuda("salf_ray_backward");
  }
  SALF_CATCH
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

__global__ void k_fill_u32(int64_t n, uint32_t v, uint32_t *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

extern "C" size_t salf_ray_backward_det_workspace_bytes(int64_t n_slots, int64_t n_voxels) {
  const int64_t ns = std::max<int64_t>(n_slots, 1);
  return align256(sizeof(float) * kGradStride * ns) + align256(sizeof(uint32_t) * ns) +
         det_reduce_workspace_bytes(ns, n_voxels);
}

extern "C" int salf_ray_backward_deterministic(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                               const double *origins, const double *dirs, const uint8_t *valid,
                                               const salf_raster_opts_t *opts, const double *saved,
                                               const double *d_rgb, const double *d_depth, double *grad,
                                               const int64_t *row_start, int64_t n_slots, void *workspace,
                                               size_t workspace_bytes, void *stream) {
  SALF_TRY {
    if (n == 0 || n_slots <= 0) return SALF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t a = align256(sizeof(float) * kGradStride * n_slots), b = align256(sizeof(uint32_t) * n_slots);
    if (workspace_bytes < a + b) return set_error(SALF_EWORKSPACE, "deterministic ray backward workspace too small");
    RowSink sink{(float *)workspace, (uint32_t *)((char *)workspace + a), row_start};
    k_fill_u32<<<(unsigned)((n_slots + 255) / 256), 256, 0, st>>>(n_slots, (uint32_t)scene->n, sink.row_vid);
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    FeatGrad fg{nullptr, nullptr, nullptr, nullptr};
    if (opts->exact_color)
      k_ray_backward<true><<<grid, 128, 0, st>>>(t, *scene, n, origins, dirs, valid, *opts, saved, d_rgb, d_depth,
                                                 grad, fg, sink);
    else
      launch_ray_backward_mixed(scene->density_mode == SALF_DENSITY_SDF, d_rgb != nullptr, grid, st, t, *scene, n,
                                origins, dirs, valid, *opts, saved, d_rgb, d_depth, grad, fg, sink);
    const int rc = check_cuda("salf_ray_backward_deterministic");
    if (rc != SALF_OK) return rc;
    return det_reduce_rows(n_slots, sink.row_vid, sink.rows, scene->n, grad, (char *)workspace + a + b,
                           workspace_bytes - a - b, st);
  }
  SALF_CATCH
}

extern "C" int salf_lidar_backward(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                   const double *origins, const double *dirs, const salf_raster_opts_t *opts,
                                   const double *saved, const double *d_depth, const float *feat, const double *dF,
                                   const double *Facc, double *grad, double *feat_grad, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    if (feat && (!dF || !Facc || !feat_grad)) return set_error(SALF_EINVAL, "feature backward needs dF, F and a buffer");
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    // colour is not part of the LiDAR model: no colour seeds (d_rgb = nullptr)
    FeatGrad fg{feat, dF, Facc, feat_grad};
    if (opts->exact_color)
      k_ray_backward<false><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, nullptr, *opts, saved,
                                                                      nullptr, d_depth, grad, fg, RowSink{});
    else if (feat && scene->density_mode == SALF_DENSITY_SDF)
      k_ray_backward<false, true, true, false, true><<<grid, 128, 0, (cudaStream_t)stream>>>(
          t, *scene, n, origins, dirs, nullptr, *opts, saved, nullptr, d_depth, grad, fg, RowSink{});
    else if (feat)
      k_ray_backward<false, true, false, false, true><<<grid, 128, 0, (cudaStream_t)stream>>>(
          t, *scene, n, origins, dirs, nullptr, *opts, saved, nullptr, d_depth, grad, fg, RowSink{});
    else
      launch_ray_backward_mixed(scene->density_mode == SALF_DENSITY_SDF, false, grid, (cudaStream_t)stream, t,
                                *scene, n, origins, dirs, nullptr, *opts, saved, nullptr, d_depth, grad, fg,
                                RowSink{});
    return check_cuda("salf_lidar_backward");
  }
  SALF_CATCH
}

// Rays into one actor's canonical frame (render_ray.py:180-190): per ray the
// pose of its timestamp (pose table row pose_idx[i]: translation, then the
// row-major rotation matrix R, evaluated by the host for the batch's distinct
// timestamps with the reference's own NumPy), o_a = R^T (o - pos) and
// d_a = R^T d in np.einsum("nji,nj->ni") order ((p0 + p1) + p2, plain products;
// this file is compiled with --fmad=false), then ray_box_range against the
// actor box +-half (octree.py:175-194: reciprocal multiply, zero-direction
// override, NaN-propagating min / max) and the reference's hit rule
// (t_out > max(t_in, 0)) & (max(t_in, 0) < t_max = inf).
__global__ void k_actor_rays(int64_t n, const double *__restrict__ o, const double *__restrict__ d,
                             const int64_t *__restrict__ pose_idx, const double *__restrict__ poses, double hx,
                             double hy, double hz, double *__restrict__ o_a, double *__restrict__ d_a,
                             uint8_t *__restrict__ hit) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double *P = poses + 12 * (pose_idx ? pose_idx[i] : 0);
  const double v[3] = {__dsub_rn(o[3 * i], P[0]), __dsub_rn(o[3 * i + 1], P[1]), __dsub_rn(o[3 * i + 2], P[2])};
  const double w[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  const double *R = P + 3;
  const double half[3] = {hx, hy, hz};
  double oa[3], da[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    oa[k] = __dadd_rn(__dadd_rn(__dmul_rn(R[k], v[0]), __dmul_rn(R[3 + k], v[1])), __dmul_rn(R[6 + k], v[2]));
    da[k] = __dadd_rn(__dadd_rn(__dmul_rn(R[k], w[0]), __dmul_rn(R[3 + k], w[1])), __dmul_rn(R[6 + k], w[2]));
    o_a[3 * i + k] = oa[k];
    d_a[3 * i + k] = da[k];
  }
  double t_in = 0.0, t_out = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double nk, fk;
    if (da[k] == 0.0) {
      const bool inside = (oa[k] >= -half[k]) && (oa[k] <= half[k]);
      nk = inside ? -INFINITY : INFINITY;
      fk = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = 1.0 / da[k];
      const double ta = __dmul_rn(__dsub_rn(-half[k], oa[k]), inv), tb = __dmul_rn(__dsub_rn(half[k], oa[k]), inv);
      nk = npmin(ta, tb);
      fk = npmax(ta, tb);
    }
    t_in = k ? npmax(t_in, nk) : nk;
    t_out = k ? npmin(t_out, fk) : fk;
  }
  const double t0 = npmax(t_in, 0.0);
  hit[i] = (t_out > t0) && (t0 < INFINITY);
}

extern "C" int salf_actor_rays(int64_t n, const double *origins, const double *dirs, const int64_t *pose_idx,
                               const double *poses, const double *half_extents, double *o_actor, double *d_actor,
                               uint8_t *hit, void *stream) {
  SALF_TRY {
    if (n <= 0) return SALF_OK;
    k_actor_rays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, origins, dirs, pose_idx, poses, half_extents[0], half_extents[1], half_extents[2], o_actor, d_actor, hit);
    return check_cuda("salf_actor_rays");
  }
  SALF_CATCH
}

extern "C" int salf_shade_segments(const salf_scene_t *scene, int64_t n, const double *seg_origin,
                                   const double *seg_dir, const int64_t *seg_vid, const double *seg_t0,
                                   const double *seg_t1, int32_t owner, int64_t vid_offset, int32_t exact_color,
                                   double *records, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (exact_color)
      k_shade_segments<true><<<grid, 128, 0, (cudaStream_t)stream>>>(*scene, n, seg_origin, seg_dir, seg_vid, seg_t0,
                                                                       seg_t1, owner, vid_offset, records);
    else
      k_shade_segments<false><<<grid, 128, 0, (cudaStream_t)stream>>>(*scene, n, seg_origin, seg_dir, seg_vid, seg_t0,
                                                                        seg_t1, owner, vid_offset, records);
    return check_cuda("salf_shade_segments");
  }
  SALF_CATCH
}

extern "C" int salf_ray_forward_merge(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                      const double *origins, const double *dirs, const uint8_t *valid,
                                      const salf_raster_opts_t *opts, const int64_t *ex_start, const double *ex_rec,
                                      float *out_rgb, float *out_opacity, float *out_depth, double *saved,
                                      int32_t *status, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (opts->exact_color)
      k_ray_forward_merge<true><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, valid, *opts,
                                                                          ex_start, ex_rec, out_rgb, out_opacity,
                                                                          out_depth, saved, status);
    else
      k_ray_forward_merge<false><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, valid, *opts,
                                                                           ex_start, ex_rec, out_rgb, out_opacity,
                                                                           out_depth, saved, status);
    return check_cuda("salf_ray_forward_merge");
  }
  SALF_CATCH
}

extern "C" int salf_ray_backward_merge(const salf_octree_t *tree, const salf_scene_t *scene, int64_t n,
                                       const double *origins, const double *dirs, const uint8_t *valid,
                                       const salf_raster_opts_t *opts, const int64_t *ex_start, const double *ex_rec,
                                       const double *saved, const double *d_rgb, const double *d_depth, double *grad,
                                       double *ex_grad, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    OctDev t = make_oct(tree);
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (opts->exact_color)
      k_ray_backward_merge<true><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, valid, *opts,
                                                                           ex_start, ex_rec, saved, d_rgb, d_depth,
                                                                           grad, ex_grad);
    else
      k_ray_backward_merge<false><<<grid, 128, 0, (cudaStream_t)stream>>>(t, *scene, n, origins, dirs, valid, *opts,
                                                                            ex_start, ex_rec, saved, d_rgb, d_depth,
                                                                            grad, ex_grad);
    return check_cuda("salf_ray_backward_merge");
  }
  SALF_CATCH
}

extern "C" size_t salf_octree_jump_bytes(int32_t levels) {
  if (levels <= 0 || levels > kJumpMaxLevels) return 0;
  return jump_corner_offset(levels) + sizeof(double) * 3 * ((size_t)1 << levels);
}

extern "C" int salf_octree_jump_build(const salf_octree_t *tree, int32_t levels, void *jump, void *stream) {
  SALF_TRY {
    if (levels <= 0 || levels > kJumpMaxLevels)
      return set_error(SALF_EINVAL, "jump table levels must be in 1..%d, got %d", kJumpMaxLevels, (int)levels);
    if (tree->n_nodes <= 0) return set_error(SALF_EINVAL, "empty octree");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nw = (int64_t)jump_words(levels);
    k_jump_words<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(tree->nodes, levels, (int32_t *)jump);
    const int nc = 3 << levels;
    k_jump_corners<<<(nc + 127) / 128, 128, 0, st>>>(tree->root_min[0], tree->root_min[1], tree->root_min[2],
                                                     tree->root_edge, levels,
                                                     (double *)((char *)jump + jump_corner_offset(levels)));
    return check_cuda("salf_octree_jump_build");
  }
  SALF_CATCH
}
