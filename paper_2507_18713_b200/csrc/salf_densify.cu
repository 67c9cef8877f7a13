// salf_densify.cu -- the densify / prune round on the device (SURVEY §8f
// rank 1; reference densify.py:39-94, optim.py:35-40, trainer.py:194-206).
//
//   k_densify_flags   centre opacity (densify.py:39-46, reference fp64 order),
//                     prune = opacity < threshold, eligible = kept and not at
//                     the finest level (:68-70)
//   k_grad_norm_acc   grad_acc += ||dL/dW_c|| per voxel (trainer.py:193)
//   k_densify_apply   the new voxel arrays: kept rows in index order, then
//                     8 children per split voxel (child offsets x fastest,
//                     :28-30, :76-86) inheriting every parameter; Adam
//                     moments carried for kept rows and zeroed for children
//                     (optim.py:35-40)
// The ranking and compaction between the two (lexsort by gradient norm,
// ties by index; flatnonzero) are stable sorts / selections on the host
// side of the ABI (paper_2507_18713_b200/densify.py).
#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {

__global__ void k_densify_flags(int64_t n, const double *__restrict__ p, const double *__restrict__ geo,
                                const uint8_t *__restrict__ level, int mode, double prune_opacity, int max_levels,
                                uint8_t *__restrict__ flags, double *__restrict__ opacity) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double *r = p + i * kGradStride;
  const double s = r[3], edge = geo[4 * i + 3];
  double sigma;
  if (mode == SALF_DENSITY_SDF) {
    // 0.5 * a * (1.0 + sign(s) * (1.0 - exp(-|s| / b)))  (scene.py:242)
    const double a = salf_fm::exp(r[25]), b = salf_fm::exp(r[26]);
    const double e = salf_fm::exp(__ddiv_rn(-fabs(s), b));
    sigma = __dmul_rn(__dmul_rn(0.5, a), __dadd_rn(1.0, __dmul_rn(npsign(s), __dsub_rn(1.0, e))));
  } else {
    sigma = salf_fm::exp(s);
  }
  const double op = -salf_fm::expm1(__dmul_rn(-sigma, edge));
  const bool prune = op < prune_opacity;
  const bool eligible = !prune && (int)level[i] < max_levels - 1;
  flags[i] = (uint8_t)((prune ? 1 : 0) | (eligible ? 2 : 0));
  if (opacity) opacity[i] = op;
}

// np.linalg.norm(w_c.reshape(M, 9), axis=1): sqrt of NumPy's pairwise sum of
// the 9 squares ((0+1)+(2+3)) + ((4+5)+(6+7)), then + 8.
__global__ void k_grad_norm_acc(int64_t n, const double *__restrict__ g, double *__restrict__ acc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double *r = g + i * kGradStride + 4;
  double q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) q[k] = __dmul_rn(r[k], r[k]);
  const double s = __dadd_rn(__dadd_rn(__dadd_rn(q[0], q[1]), __dadd_rn(q[2], q[3])),
                             __dadd_rn(__dadd_rn(q[4], q[5]), __dadd_rn(q[6], q[7])));
  acc[i] = __dadd_rn(acc[i], sqrt(__dadd_rn(s, q[8])));
}

// One thread per (output row, column) of the 27-wide blocks; column 27 of
// the index space carries level / ijk.
__global__ void k_densify_apply(int64_t n_keep, const int64_t *__restrict__ keep_idx, int64_t n_split,
                                const int64_t *__restrict__ split_idx, const uint8_t *__restrict__ level,
                                const int32_t *__restrict__ ijk, const double *__restrict__ p,
                                const double *__restrict__ m, const double *__restrict__ v,
                                uint8_t *__restrict__ level_out, int32_t *__restrict__ ijk_out,
                                double *__restrict__ p_out, double *__restrict__ m_out, double *__restrict__ v_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rows = n_keep + 8 * n_split;
  if (t >= rows * (kGradStride + 1)) return;
  const int64_t row = t / (kGradStride + 1);
  const int col = (int)(t - row * (kGradStride + 1));
  const bool child = row >= n_keep;
  const int64_t src = child ? split_idx[(row - n_keep) >> 3] : keep_idx[row];
  if (col < kGradStride) {
    const int64_t o = row * kGradStride + col, s = src * kGradStride + col;
    p_out[o] = p[s];
    if (m_out) m_out[o] = child ? 0.0 : m[s];
    if (v_out) v_out[o] = child ? 0.0 : v[s];
    return;
  }
  if (!child) {
    level_out[row] = level[src];
#pragma unroll
    for (int k = 0; k < 3; ++k) ijk_out[3 * row + k] = ijk[3 * src + k];
  } else {
    const int c = (int)((row - n_keep) & 7);  // child offset (x, y, z) = bits (0, 1, 2)
    level_out[row] = (uint8_t)(level[src] + 1);
#pragma unroll
    for (int k = 0; k < 3; ++k) ijk_out[3 * row + k] = 2 * ijk[3 * src + k] + ((c >> k) & 1);
  }
}

// Voxel geometry from (level, ijk) in the reference's rounding
// (scene.py:186-194): edge = base / 2^level, centre = aabb_min + (ijk + 0.5) edge;
// aux = (exp(log_a), 1 / exp(log_b), 2 / edge) as DeviceScene holds it.
__global__ void k_voxel_geometry(int64_t n, const uint8_t *__restrict__ level, const int32_t *__restrict__ ijk,
                                 double ax, double ay, double az, double base_edge, const double *__restrict__ p,
                                 double *__restrict__ geo, double *__restrict__ aux, float *__restrict__ prm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double edge = __ddiv_rn(base_edge, ldexp(1.0, (int)level[i]));
  const double lo[3] = {ax, ay, az};
#pragma unroll
  for (int k = 0; k < 3; ++k) geo[4 * i + k] = __dadd_rn(lo[k], __dmul_rn(__dadd_rn((double)ijk[3 * i + k], 0.5), edge));
  geo[4 * i + 3] = edge;
  const double *r = p + i * kGradStride;
  aux[4 * i + 0] = exp(r[25]);
  aux[4 * i + 1] = 1.0 / exp(r[26]);
  aux[4 * i + 2] = __ddiv_rn(2.0, edge);
  aux[4 * i + 3] = 0.0;
  float *q = prm + i * SALF_PRM_STRIDE;
#pragma unroll
  for (int k = 0; k < 25; ++k) q[k] = (float)r[k];
#pragma unroll
  for (int k = 25; k < SALF_PRM_STRIDE; ++k) q[k] = 0.f;
}

}  // namespace salf

using namespace salf;

extern "C" int salf_densify_flags(int64_t n, const double *params, const double *geo, const uint8_t *level,
                                  int32_t density_mode, double prune_opacity, int32_t max_levels, uint8_t *flags,
                                  double *opacity, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_densify_flags<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, params, geo, level, density_mode, prune_opacity, max_levels, flags, opacity);
    return check_cuda("salf_densify_flags");
  }
  SALF_CATCH
}

extern "C" int salf_grad_norm_acc(int64_t n, const double *grad, double *acc, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_grad_norm_acc<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, grad, acc);
    return check_cuda("salf_grad_norm_acc");
  }
  SALF_CATCH
}

extern "C" int salf_densify_apply(int64_t n_keep, const int64_t *keep_idx, int64_t n_split, const int64_t *split_idx,
                                  const uint8_t *level, const int32_t *ijk, const double *params, const double *m,
                                  const double *v, uint8_t *level_out, int32_t *ijk_out, double *params_out,
                                  double *m_out, double *v_out, void *stream) {
  SALF_TRY {
    const int64_t total = (n_keep + 8 * n_split) * (kGradStride + 1);
    if (total == 0) return SALF_OK;
    if ((m_out && !m) || (v_out && !v)) return set_error(SALF_EINVAL, "moment outputs need moment inputs");
    k_densify_apply<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n_keep, keep_idx, n_split, split_idx, level, ijk, params, m, v, level_out, ijk_out, params_out, m_out, v_out);
    return check_cuda("salf_densify_apply");
  }
  SALF_CATCH
}

extern "C" int salf_voxel_geometry(int64_t n, const uint8_t *level, const int32_t *ijk, const double *aabb_min,
                                   double base_edge, const double *params, double *geo, double *aux, float *prm,
                                   void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_voxel_geometry<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, level, ijk, aabb_min[0], aabb_min[1], aabb_min[2], base_edge, params, geo, aux, prm);
    return check_cuda("salf_voxel_geometry");
  }
  SALF_CATCH
}

// ---------------------------------------------------------------------------
// salf.v1 voxel records straight into the device layout (container.py:27-35,
// :91-100).  Record (121 B, little endian, unaligned):
// u8 level | i32 ijk[3] | f32 w_s[4] | f32 w_c[9] | f32 w_sh[12] | f32 log_a | f32 log_b.
// A warp stages 32 records (3872 B = 242 x 16 B, 16-B aligned because
// 32 x 121 = 3872) with vector loads into shared memory, then each lane
// decodes its record: level / ijk, the (27) f64 parameter row, geo / aux /
// prm (k_voxel_geometry's arithmetic), and flags non-finite fields
// (bit f of *bad for field f = w_s, w_c, w_sh, log_a, log_b).
namespace salf {
constexpr int kRecBytes = 121;

__device__ __forceinline__ float rec_f32(const uint8_t *r, int off) {
  const uint32_t u = (uint32_t)r[off] | ((uint32_t)r[off + 1] << 8) | ((uint32_t)r[off + 2] << 16) |
                     ((uint32_t)r[off + 3] << 24);
  return __uint_as_float(u);
}

__global__ void __launch_bounds__(128) k_decode_records(int64_t n, const uint8_t *__restrict__ rec, double ax,
                                                        double ay, double az, double base_edge,
                                                        uint8_t *__restrict__ level, int32_t *__restrict__ ijk,
                                                        double *__restrict__ params, double *__restrict__ geo,
                                                        double *__restrict__ aux, float *__restrict__ prm,
                                                        int32_t *__restrict__ bad) {
  __shared__ __align__(16) uint8_t stage[4][32 * kRecBytes];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t first = ((int64_t)blockIdx.x * 4 + warp) * 32;
  if (first >= n) return;
  const int cnt = (int)min((int64_t)32, n - first);
  const uint8_t *src = rec + first * kRecBytes;
  uint8_t *buf = stage[warp];
  if (cnt == 32) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);  // 16-B aligned (see above)
    uint4 *d4 = reinterpret_cast<uint4 *>(buf);
    for (int k = lane; k < 32 * kRecBytes / 16; k += 32) d4[k] = __ldg(s4 + k);
  } else {
    for (int k = lane; k < cnt * kRecBytes; k += 32) buf[k] = src[k];
  }
  __syncwarp();
  if (lane >= cnt) return;
  const int64_t i = first + lane;
  const uint8_t *r = buf + lane * kRecBytes;
  const uint8_t lv = r[0];
  level[i] = lv;
  int32_t c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = (int32_t)__float_as_uint(rec_f32(r, 1 + 4 * k));
    ijk[3 * i + k] = c[k];
  }
  double p[27];
  int flags = 0;
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    const float f = rec_f32(r, 13 + 4 * k);
    p[k] = (double)f;
    const int field = k < 4 ? 0 : (k < 13 ? 1 : (k < 25 ? 2 : k - 22));
    if (!isfinite(f)) flags |= 1 << field;
    params[i * kGradStride + k] = p[k];
  }
  if (flags) atomicOr(bad, flags);
  const double edge = __ddiv_rn(base_edge, ldexp(1.0, (int)lv));
  const double lo[3] = {ax, ay, az};
#pragma unroll
  for (int k = 0; k < 3; ++k) geo[4 * i + k] = __dadd_rn(lo[k], __dmul_rn(__dadd_rn((double)c[k], 0.5), edge));
  geo[4 * i + 3] = edge;
  aux[4 * i + 0] = exp(p[25]);
  aux[4 * i + 1] = 1.0 / exp(p[26]);
  aux[4 * i + 2] = __ddiv_rn(2.0, edge);
  aux[4 * i + 3] = 0.0;
  float *q = prm + i * SALF_PRM_STRIDE;
#pragma unroll
  for (int k = 0; k < 25; ++k) q[k] = (float)p[k];
#pragma unroll
  for (int k = 25; k < SALF_PRM_STRIDE; ++k) q[k] = 0.f;
}
}  // namespace salf

extern "C" int salf_decode_records(int64_t n, const uint8_t *records, const double *aabb_min, double base_edge,
                                   uint8_t *level, int32_t *ijk, double *params, double *geo, double *aux,
                                   float *prm, int32_t *bad, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    if (((uintptr_t)records & 15) != 0) return set_error(SALF_EINVAL, "record buffer must be 16-byte aligned");
    const int64_t warps = (n + 31) / 32;
    k_decode_records<<<(unsigned)((warps + 3) / 4), 128, 0, (cudaStream_t)stream>>>(
        n, records, aabb_min[0], aabb_min[1], aabb_min[2], base_edge, level, ijk, params, geo, aux, prm, bad);
    return check_cuda("salf_decode_records");
  }
  SALF_CATCH
}
