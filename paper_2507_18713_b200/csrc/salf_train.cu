// salf_train.cu -- the rest of the training step on the device (SURVEY §8f
// rank 1): Adam (reference optim.py:48-62), the scene refresh after an update,
// and the parameter regularisers eikonal / empty-space / LiDAR opacity
// (reference losses.py:49-60, :188-249).  All fp64, reference operation order.
//
// Parameter block: (M, 27) f64 rows = w_s[4] w_c[9] w_sh[12] log_a log_b
// (the gradient buffer's layout).
#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {

// Adam with the reference's expression order:
//   m = b1 m + (1 - b1) g ; v = b2 v + (1 - b2) g g
//   p -= lr * (m / bias1) / (sqrt(v / bias2) + eps)
__global__ void k_adam(int64_t n, double *__restrict__ p, const double *__restrict__ g, double *__restrict__ m,
                       double *__restrict__ v, double lr, double b1, double b2, double eps, double bias1,
                       double bias2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double gi = g[i];
  const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dsub_rn(1.0, b1), gi));
  const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), gi), gi));
  m[i] = mi;
  v[i] = vi;
  const double mh = __ddiv_rn(mi, bias1), vh = __ddiv_rn(vi, bias2);
  p[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(sqrt(vh), eps)));
}

// Device scene refresh from the parameter block: prm (f32 fields), aux a, 1/b.
__global__ void k_refresh(int64_t n, const double *__restrict__ p, float *__restrict__ prm, double *__restrict__ aux) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double *r = p + i * kGradStride;
  float *q = prm + i * SALF_PRM_STRIDE;
#pragma unroll
  for (int k = 0; k < 25; ++k) q[k] = (float)r[k];
  aux[4 * i + 0] = exp(r[25]);
  aux[4 * i + 1] = 1.0 / exp(r[26]);
}

// loss_eikonal (losses.py:49-60): mean | ||W_s[:3]|| - 1 | over `idx`.
__global__ void k_eikonal(int64_t n_idx, const int64_t *__restrict__ idx, const double *__restrict__ p,
                          double *__restrict__ grad, double *__restrict__ loss_sum, double inv_n) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_idx) return;
  const int64_t v = idx[j];
  const double *r = p + v * kGradStride;
  const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(r[0], r[0]), __dmul_rn(r[1], r[1])), __dmul_rn(r[2], r[2])));
  atomicAdd(loss_sum, fabs(__dsub_rn(nrm, 1.0)));
  if (nrm > 1e-12) {
    const double s = __dmul_rn(npsign(__dsub_rn(nrm, 1.0)), inv_n);
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(grad + v * kGradStride + k, __dmul_rn(s, __ddiv_rn(r[k], nrm)));
  }
}

// density at the voxel centre (x = 0 -> s = bias) and its opacity over the edge
// (losses.py:216-228).
__global__ void k_center_alpha(int64_t n_idx, const int64_t *__restrict__ idx, const double *__restrict__ p,
                               const double *__restrict__ geo, int mode, double *__restrict__ alpha_out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_idx) return;
  const int64_t v = idx[j];
  const double *r = p + v * kGradStride;
  const double s = r[3], edge = geo[4 * v + 3];
  double e;
  const double sigma = density(mode, s, exp(r[25]), 1.0 / exp(r[26]), e);
  alpha_out[j] = -expm1(__dmul_rn(-sigma, edge));
}

// loss_empty gradient (losses.py:230-249) for the k selected (lowest-alpha) outer voxels.
__global__ void k_empty_grad(int64_t k, const int64_t *__restrict__ sel, const double *__restrict__ p,
                             const double *__restrict__ geo, int mode, double *__restrict__ grad) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int64_t v = sel[j];
  const double *r = p + v * kGradStride;
  const double s = r[3], edge = geo[4 * v + 3];
  const double a = exp(r[25]), b = exp(r[26]);
  double e;
  const double sigma = density(mode, s, a, 1.0 / b, e);
  const double g_alpha = 1.0 / (double)k;
  const double g_sigma = __dmul_rn(__dmul_rn(g_alpha, edge), exp(__dmul_rn(-sigma, edge)));
  double *gr = grad + v * kGradStride;
  if (mode == SALF_DENSITY_SDF) {
    const double k2 = __ddiv_rn(a, __dmul_rn(2.0, b));
    const double ee = exp(__ddiv_rn(-fabs(s), b));
    const double ds = (s == 0.0) ? 0.0 : __dmul_rn(__dmul_rn(g_sigma, k2), ee);
    atomicAdd(gr + 3, ds);
    atomicAdd(gr + 25, __dmul_rn(g_sigma, sigma));
    atomicAdd(gr + 26, __dmul_rn(g_sigma, __dmul_rn(__dmul_rn(-k2, s), ee)));
  } else {
    atomicAdd(gr + 3, __dmul_rn(g_sigma, sigma));
  }
}

// loss_opacity_lidar gradient (losses.py:188-226) for points already located
// in leaves (vid >= 0): opacity over a 20 cm traversal driven towards 1.
__global__ void k_opacity_lidar(int64_t n, const double *__restrict__ pts, const int64_t *__restrict__ vid,
                                const double *__restrict__ p, const double *__restrict__ geo, int mode,
                                double *__restrict__ grad, double *__restrict__ loss_sum) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t v = vid[j];
  const double *r = p + v * kGradStride;
  const double4 g = make_double4(geo[4 * v], geo[4 * v + 1], geo[4 * v + 2], geo[4 * v + 3]);
  const double sc2 = __ddiv_rn(2.0, g.w);
  const double x[3] = {__dmul_rn(__dsub_rn(pts[3 * j], g.x), sc2), __dmul_rn(__dsub_rn(pts[3 * j + 1], g.y), sc2),
                       __dmul_rn(__dsub_rn(pts[3 * j + 2], g.z), sc2)};
  const double s = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(r[0], x[0]), __dmul_rn(r[2], x[2])), __dmul_rn(r[1], x[1])),
                             r[3]);
  const double a = exp(r[25]), b = exp(r[26]);
  double e;
  const double sigma = density(mode, s, a, 1.0 / b, e);
  const double delta = 0.2;  // LIDAR_OPACITY_DELTA (losses.py:17)
  const double alpha = -expm1(__dmul_rn(-sigma, delta));
  atomicAdd(loss_sum, __dsub_rn(1.0, alpha));
  const double g_sigma = __ddiv_rn(__dmul_rn(-delta, exp(__dmul_rn(-sigma, delta))), (double)n);
  double *gr = grad + v * kGradStride;
  double ds;
  if (mode == SALF_DENSITY_SDF) {
    const double k2 = __ddiv_rn(a, __dmul_rn(2.0, b));
    const double ee = exp(__ddiv_rn(-fabs(s), b));
    ds = (s == 0.0) ? 0.0 : __dmul_rn(__dmul_rn(g_sigma, k2), ee);
    atomicAdd(gr + 25, __dmul_rn(g_sigma, sigma));
    atomicAdd(gr + 26, __dmul_rn(g_sigma, __dmul_rn(__dmul_rn(-k2, s), ee)));
  } else {
    ds = __dmul_rn(g_sigma, sigma);
  }
  atomicAdd(gr + 0, __dmul_rn(ds, x[0]));
  atomicAdd(gr + 1, __dmul_rn(ds, x[1]));
  atomicAdd(gr + 2, __dmul_rn(ds, x[2]));
  atomicAdd(gr + 3, ds);
}

// loss_smooth (losses.py:95-185): one thread per (face pair, face corner).
// Corners of the finer voxel's face in its local frame; the coarse side sees
// the same world point in its own frame; SDF and colour (view = face normal)
// differences, L1, gradients into both voxels.
__global__ void k_smooth(int64_t n_pairs, const int64_t *__restrict__ fine, const int64_t *__restrict__ coarse,
                         const int32_t *__restrict__ axis, const double *__restrict__ sgn,
                         const double *__restrict__ p, const double *__restrict__ geo, double inv_ns, double inv_nc,
                         double *__restrict__ grad, double *__restrict__ loss_sums) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pairs * 4) return;
  const int64_t q = t >> 2;
  const int corner = (int)(t & 3);
  const int64_t f = fine[q], c = coarse[q];
  const int ax = axis[q];
  const double sg = sgn[q];
  const int o0 = ax == 0 ? 1 : 0, o1 = ax == 2 ? 1 : 2;  // the two in-face axes
  // corners [(-1,-1), (-1,1), (1,-1), (1,1)] over (o0, o1)
  double xf[3];
  xf[ax] = sg;
  xf[o0] = (corner & 2) ? 1.0 : -1.0;
  xf[o1] = (corner & 1) ? 1.0 : -1.0;
  const double *gf = geo + 4 * f, *gc = geo + 4 * c;
  const double hf = __ddiv_rn(gf[3], 2.0), sc2 = __ddiv_rn(2.0, gc[3]);
  double xc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double wpt = __dadd_rn(gf[k], __dmul_rn(xf[k], hf));  // local_to_world (scene.py:211-219)
    xc[k] = __dmul_rn(__dsub_rn(wpt, gc[k]), sc2);            // world_to_local (scene.py:196-209)
  }
  const double *pf = p + f * kGradStride, *pc = p + c * kGradStride;
  auto sdf = [](const double *r, const double x[3]) {
    return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(r[0], x[0]), __dmul_rn(r[2], x[2])), __dmul_rn(r[1], x[1])), r[3]);
  };
  const double om[3] = {ax == 0 ? sg : 0.0, ax == 1 ? sg : 0.0, ax == 2 ? sg : 0.0};
  const double gam[4] = {kShC0, __dmul_rn(kShC1, om[1]), __dmul_rn(kShC1, om[2]), __dmul_rn(kShC1, om[0])};
  auto color = [&](const double *r, const double x[3], double out[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double *wc = r + 4 + 3 * i, *ws = r + 13 + 4 * i;
      const double zc = __dadd_rn(__dadd_rn(__dmul_rn(wc[0], x[0]), __dmul_rn(wc[2], x[2])), __dmul_rn(wc[1], x[1]));
      const double zs = __dadd_rn(__dadd_rn(__dmul_rn(ws[0], gam[0]), __dmul_rn(ws[2], gam[2])),
                                  __dadd_rn(__dmul_rn(ws[1], gam[1]), __dmul_rn(ws[3], gam[3])));
      out[i] = 1.0 / (1.0 + exp(-__dadd_rn(zc, zs)));
    }
  };
  const double ds = __dsub_rn(sdf(pf, xf), sdf(pc, xc));
  double cf[3], cc[3];
  color(pf, xf, cf);
  color(pc, xc, cc);
  double l_c = 0.0;
  const double gs = __dmul_rn(npsign(ds), inv_ns);
  double *Gf = grad + f * kGradStride, *Gc = grad + c * kGradStride;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    atomicAdd(Gf + k, __dmul_rn(gs, xf[k]));
    atomicAdd(Gc + k, -__dmul_rn(gs, xc[k]));
  }
  atomicAdd(Gf + 3, gs);
  atomicAdd(Gc + 3, -gs);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double dci = __dsub_rn(cf[i], cc[i]);
    l_c = __dadd_rn(l_c, fabs(dci));
    const double gci = __dmul_rn(npsign(dci), inv_nc);
    const double gzf = __dmul_rn(__dmul_rn(gci, cf[i]), __dsub_rn(1.0, cf[i]));
    const double gzc = __dmul_rn(__dmul_rn(-gci, cc[i]), __dsub_rn(1.0, cc[i]));
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      atomicAdd(Gf + 4 + 3 * i + j, __dmul_rn(gzf, xf[j]));
      atomicAdd(Gc + 4 + 3 * i + j, __dmul_rn(gzc, xc[j]));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      atomicAdd(Gf + 13 + 4 * i + j, __dmul_rn(gzf, gam[j]));
      atomicAdd(Gc + 13 + 4 * i + j, __dmul_rn(gzc, gam[j]));
    }
  }
  atomicAdd(loss_sums, fabs(ds));
  atomicAdd(loss_sums + 1, l_c);
}

// L1 loss seed + value (losses.py:22-31): d[i] = sign(pred - gt) * scale on
// selected elements (mask[i / group] != 0, or all when mask is NULL), 0
// elsewhere; loss_sum += sum |pred - gt| over the selection.
template <typename G>
__global__ void __launch_bounds__(256) k_l1_seed(int64_t n, const float *__restrict__ pred, const G *__restrict__ gt,
                                                 const uint8_t *__restrict__ mask, int group, double scale,
                                                 double *__restrict__ d, double *__restrict__ loss_sum) {
  // grid-stride over elements; the loss is reduced per warp, then per block,
  // with one fp64 atomic per block (not per warp: a single address)
  __shared__ double part[8];
  double l = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool sel = mask == nullptr || mask[i / group] != 0;
    const double diff = (double)pred[i] - (double)gt[i];
    d[i] = sel ? __dmul_rn(npsign(diff), scale) : 0.0;
    l += sel ? fabs(diff) : 0.0;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = l;
  __syncthreads();
  if (threadIdx.x == 0 && loss_sum) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    if (t != 0.0) atomicAdd(loss_sum, t);
  }
}

}  // namespace salf

using namespace salf;

extern "C" int salf_loss_smooth(const double *params, const double *geo, int64_t n_pairs, const int64_t *fine,
                                const int64_t *coarse, const int32_t *axis, const double *sign, double *grad,
                                double *loss_sums, void *stream) {
  SALF_TRY {
    if (n_pairs == 0) return SALF_OK;
    const int64_t n = n_pairs * 4;
    k_smooth<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        n_pairs, fine, coarse, axis, sign, params, geo, 1.0 / (double)(4 * n_pairs), 1.0 / (double)(12 * n_pairs), grad,
        loss_sums);
    return check_cuda("salf_loss_smooth");
  }
  SALF_CATCH
}

extern "C" int salf_loss_opacity_lidar(const double *params, const double *geo, int32_t density_mode, int64_t n,
                                       const double *points, const int64_t *vid, double *grad, double *loss_sum,
                                       void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_opacity_lidar<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, points, vid, params, geo,
                                                                                   density_mode, grad, loss_sum);
    return check_cuda("salf_loss_opacity_lidar");
  }
  SALF_CATCH
}

extern "C" int salf_adam_step(int64_t n, double *params, const double *grad, double *m, double *v, double lr,
                              double beta1, double beta2, double eps, int64_t step, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    const double bias1 = 1.0 - pow(beta1, (double)step), bias2 = 1.0 - pow(beta2, (double)step);
    k_adam<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, params, grad, m, v, lr, beta1, beta2,
                                                                          eps, bias1, bias2);
    return check_cuda("salf_adam_step");
  }
  SALF_CATCH
}

extern "C" int salf_scene_refresh(const double *params, int64_t n, float *prm, double *aux, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_refresh<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, params, prm, aux);
    return check_cuda("salf_scene_refresh");
  }
  SALF_CATCH
}

extern "C" int salf_loss_eikonal(const double *params, int64_t n_idx, const int64_t *idx, double *grad,
                                 double *loss_sum, void *stream) {
  SALF_TRY {
    if (n_idx == 0) return SALF_OK;
    k_eikonal<<<(unsigned)((n_idx + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_idx, idx, params, grad, loss_sum,
                                                                                 1.0 / (double)n_idx);
    return check_cuda("salf_loss_eikonal");
  }
  SALF_CATCH
}

extern "C" int salf_center_alpha(const double *params, const double *geo, int32_t density_mode, int64_t n_idx,
                                 const int64_t *idx, double *alpha, void *stream) {
  SALF_TRY {
    if (n_idx == 0) return SALF_OK;
    k_center_alpha<<<(unsigned)((n_idx + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_idx, idx, params, geo,
                                                                                       density_mode, alpha);
    return check_cuda("salf_center_alpha");
  }
  SALF_CATCH
}

extern "C" int salf_loss_empty_grad(const double *params, const double *geo, int32_t density_mode, int64_t k,
                                    const int64_t *sel, double *grad, void *stream) {
  SALF_TRY {
    if (k == 0) return SALF_OK;
    k_empty_grad<<<(unsigned)((k + 255) / 256), 256, 0, (cudaStream_t)stream>>>(k, sel, params, geo, density_mode,
                                                                                grad);
    return check_cuda("salf_loss_empty_grad");
  }
  SALF_CATCH
}

extern "C" int salf_l1_seed(int64_t n, const float *pred, const void *gt, int32_t gt_f64, const uint8_t *mask,
                            int32_t group, double scale, double *d_out, double *loss_sum, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    if (group < 1) return set_error(SALF_EINVAL, "group must be >= 1");
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (gt_f64)
      k_l1_seed<double><<<g, 256, 0, (cudaStream_t)stream>>>(n, pred, (const double *)gt, mask, group, scale, d_out,
                                                             loss_sum);
    else
      k_l1_seed<float><<<g, 256, 0, (cudaStream_t)stream>>>(n, pred, (const float *)gt, mask, group, scale, d_out,
                                                            loss_sum);
    return check_cuda("salf_l1_seed");
  }
  SALF_CATCH
}
