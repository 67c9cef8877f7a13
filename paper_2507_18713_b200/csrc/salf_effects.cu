// salf_effects.cu -- secondary-ray effects with injected analytic spheres
// (reference render_ray.py:310-489, trace_effects).
//
// The reference runs a wavefront loop: every wave renders its rays through
// the volume (integrate_rays), intersects them with the spheres, and either
// composites the volume colour (sun-shadowed by the spheres) or spawns the
// next wave from the sphere interaction (mirror reflection; glass
// Schlick-weighted reflection + Snell refraction; opaque albedo).  The volume
// part is the fused ray kernel (salf_ray.cu); this file is one kernel per
// wave for everything else: sphere hits, the volume/sphere decision, shadow
// rays, accumulation into the image and the next wave (at most two children
// per ray, written to slots 2i / 2i + 1 so a stable compaction keeps a
// deterministic order).  fp64 throughout, reference operation order.
#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {

constexpr double kTMinHit = 1e-6;       // render_ray.py:333
constexpr double kShadowFactor = 0.5;   // :334
constexpr double kMinWeight = 1e-4;     // :452, :464

// einsum("ni,ni->n") of length 3: (p0 + p2) + p1
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[2], b[2])), __dmul_rn(a[1], b[1]));
}

// _sphere_hits (render_ray.py:337-357): nearest positive hit (t, index), (inf, -1) on miss.
__device__ __forceinline__ int sphere_hit(const double o[3], const double d[3], int n_sph,
                                          const salf_sphere_t *__restrict__ sph, double &best_t) {
  best_t = INFINITY;
  int best_s = -1;
  for (int si = 0; si < n_sph; ++si) {
    const salf_sphere_t &sp = sph[si];
    double oc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) oc[k] = __dsub_rn(o[k], sp.center[k]);
    const double b = dot3(oc, d);
    const double c = __dsub_rn(dot3(oc, oc), __dmul_rn(sp.radius, sp.radius));
    const double disc = __dsub_rn(__dmul_rn(b, b), c);
    const bool ok = disc >= 0.0;
    const double sq = sqrt(ok ? disc : 0.0);
    const double t_near = __dsub_rn(-b, sq), t_far = __dadd_rn(-b, sq);
    const double t = t_near > kTMinHit ? t_near : t_far;  // inside: take the exit
    const bool hit = ok && t > kTMinHit;
    if (hit && t < best_t) {
      best_t = t;
      best_s = si;
    }
  }
  return best_s;
}

__device__ __forceinline__ void emit(int64_t slot, const double o[3], const double d[3], double ts, double w,
                                     int32_t budget, int64_t pix, double *__restrict__ no, double *__restrict__ nd,
                                     double *__restrict__ nts, double *__restrict__ nw, int32_t *__restrict__ nb,
                                     int64_t *__restrict__ npix, uint8_t *__restrict__ nflag) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    no[3 * slot + k] = o[k];
    nd[3 * slot + k] = d[k];
  }
  nts[slot] = ts;
  nw[slot] = w;
  nb[slot] = budget;
  npix[slot] = pix;
  nflag[slot] = 1;
}

__global__ void k_effects_wave(int64_t n, const double *__restrict__ o_in, const double *__restrict__ d_in,
                               const double *__restrict__ ts_in, const double *__restrict__ w_in,
                               const int32_t *__restrict__ b_in, const int64_t *__restrict__ pix_in,
                               const float *__restrict__ vol_rgb, const double *__restrict__ vol_saved, int n_sph,
                               const salf_sphere_t *__restrict__ sph, double sx, double sy, double sz,
                               double *__restrict__ out, double *__restrict__ no, double *__restrict__ nd,
                               double *__restrict__ nts, double *__restrict__ nw, int32_t *__restrict__ nb,
                               int64_t *__restrict__ npix, uint8_t *__restrict__ nflag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  nflag[2 * i] = 0;
  nflag[2 * i + 1] = 0;
  const double o[3] = {o_in[3 * i], o_in[3 * i + 1], o_in[3 * i + 2]};
  const double d[3] = {d_in[3 * i], d_in[3 * i + 1], d_in[3 * i + 2]};
  const double w = w_in[i], ts = ts_in[i];
  const int32_t budget = b_in[i];
  const int64_t pix = pix_in[i];
  double hit_t = INFINITY;
  const int hit_s = n_sph ? sphere_hit(o, d, n_sph, sph, hit_t) : -1;
  // rec.depth: weighted mean t_mid where the weight sum exceeds 0.5, else NaN (render_ray.py:111-112)
  const double *sv = vol_saved + i * SALF_SAVED_STRIDE;
  const double vdepth = sv[3] > kDepthWeightMin ? __ddiv_rn(sv[4], sv[3]) : NAN;
  const bool sphere_wins = budget > 0 && hit_s >= 0 && (vdepth != vdepth || hit_t < vdepth);
  double *dst = out + 3 * pix;
  if (!sphere_wins) {
    // volume colour, darkened where a sphere occludes the surface point from the sun (:391-403)
    double col[3] = {(double)vol_rgb[3 * i], (double)vol_rgb[3 * i + 1], (double)vol_rgb[3 * i + 2]};
    if (n_sph && vdepth == vdepth) {
      double surf[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) surf[k] = __dadd_rn(o[k], __dmul_rn(vdepth, d[k]));
      const double sun[3] = {sx, sy, sz};
      double st;
      if (sphere_hit(surf, sun, n_sph, sph, st) >= 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) col[k] = __dmul_rn(col[k], kShadowFactor);
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(dst + k, __dmul_rn(w, col[k]));
    return;
  }
  const salf_sphere_t &sp = sph[hit_s];
  double p[3], nrm[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    p[k] = __dadd_rn(o[k], __dmul_rn(hit_t, d[k]));
    nrm[k] = __ddiv_rn(__dsub_rn(p[k], sp.center[k]), sp.radius);
  }
  if (sp.material == SALF_SPHERE_OPAQUE) {
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(dst + k, __dmul_rn(w, sp.albedo[k]));
    return;
  }
  if (sp.material == SALF_SPHERE_MIRROR) {  // :426-434
    const double dn = dot3(d, nrm);
    double r[3], q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      r[k] = __dsub_rn(d[k], __dmul_rn(__dmul_rn(2.0, dn), nrm[k]));
      q[k] = __dadd_rn(p[k], __dmul_rn(1e-6, r[k]));
    }
    emit(2 * i, q, r, ts, w, budget - 1, pix, no, nd, nts, nw, nb, npix, nflag);
    return;
  }
  // glass (:435-472): orient the normal against the incident ray, swap media inside
  double cos_i = -dot3(d, nrm);
  const bool entering = cos_i > 0.0;
  double n_o[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) n_o[k] = entering ? nrm[k] : -nrm[k];
  cos_i = fabs(cos_i);
  const double n1 = entering ? 1.0 : sp.ior, n2 = entering ? sp.ior : 1.0;
  const double eta = __ddiv_rn(n1, n2);
  const double k = __dsub_rn(1.0, __dmul_rn(__dmul_rn(eta, eta), __dsub_rn(1.0, __dmul_rn(cos_i, cos_i))));
  const bool tir = k < 0.0;
  double fres;
  if (tir) {
    fres = 1.0;
  } else if (sp.ior == 1.0) {
    fres = 0.0;
  } else {
    const double f = __ddiv_rn(__dsub_rn(1.0, sp.ior), __dadd_rn(1.0, sp.ior));
    const double f0 = __dmul_rn(f, f);
    const double m = __dsub_rn(1.0, cos_i);
    const double m5 = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(m, m), m), m), m);
    fres = __dadd_rn(f0, __dmul_rn(__dsub_rn(1.0, f0), m5));
  }
  const double refl_w = __dmul_rn(w, fres);
  if (refl_w > kMinWeight) {
    double r[3], q[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = __dadd_rn(d[c], __dmul_rn(__dmul_rn(2.0, cos_i), n_o[c]));
      q[c] = __dadd_rn(p[c], __dmul_rn(1e-6, r[c]));
    }
    emit(2 * i, q, r, ts, refl_w, budget - 1, pix, no, nd, nts, nw, nb, npix, nflag);
  }
  const double refr_w = __dmul_rn(w, __dsub_rn(1.0, fres));
  if (!tir && refr_w > kMinWeight) {
    const double s = __dsub_rn(__dmul_rn(eta, cos_i), sqrt(k > 0.0 ? k : 0.0));
    double r[3], q[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] = __dadd_rn(__dmul_rn(eta, d[c]), __dmul_rn(s, n_o[c]));
    const double len = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(r[0], r[0]), __dmul_rn(r[1], r[1])), __dmul_rn(r[2], r[2])));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = __ddiv_rn(r[c], len);
      q[c] = __dadd_rn(p[c], __dmul_rn(1e-6, r[c]));
    }
    emit(2 * i + 1, q, r, ts, refr_w, budget - 1, pix, no, nd, nts, nw, nb, npix, nflag);
  }
}

}  // namespace salf

using namespace salf;

extern "C" int salf_effects_wave(int64_t n, const double *origins, const double *dirs, const double *t_stamps,
                                 const double *weight, const int32_t *budget, const int64_t *pix,
                                 const float *vol_rgb, const double *vol_saved, int32_t n_spheres,
                                 const salf_sphere_t *spheres, const double *sun_dir, double *out,
                                 double *next_origins, double *next_dirs, double *next_t_stamps, double *next_weight,
                                 int32_t *next_budget, int64_t *next_pix, uint8_t *next_flag, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_effects_wave<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        n, origins, dirs, t_stamps, weight, budget, pix, vol_rgb, vol_saved, n_spheres, spheres, sun_dir[0],
        sun_dir[1], sun_dir[2], out, next_origins, next_dirs, next_t_stamps, next_weight, next_budget, next_pix,
        next_flag);
    return check_cuda("salf_effects_wave");
  }
  SALF_CATCH
}
