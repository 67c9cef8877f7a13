// salf_raster.cu -- tile rasterizer for pinhole cameras (reference render_raster.py).
//
// Pipeline per frame (all on one stream):
//   k_project      fp64 corner projection, cull, reference + tightened tile spans,
//                  orderable depth keys                         (render_raster.py:97-176)
//   depth rank     visible voxels only (non-empty span): stable radix sort of
//                  (z_center key, index) -> ties break by voxel index exactly
//                  like lexsort                                      (:177)
//   k_emit         instances written in depth-rank order, key = tile id
//   radix sort     stable sort by tile id (ceil(log2 T) bits, 2 passes at
//                  C2) -> per-tile lists in (z, index) order
//   k_offsets      CSR offsets per tile                              (:180-181)
//   k_composite    one CTA per tile, one thread per pixel: staged entries in
//                  shared memory, fp64 slab test + exact-order fp64 opacity chain,
//                  early exit when every pixel of the tile is frozen  (:201-301)
//   k_backward     replay of k_composite producing per-voxel gradients with
//                  warp-aggregated atomics (definition: DESIGN.md §raster backward)
#include "salf_common.cuh"
#include "salf_internal.h"
#include "salf_sort.cuh"

namespace salf {

struct PinholeDev {
  int width, height, tile, tiles_x, tiles_y;
  double fx, fy, cx, cy;
  double pos[3];
  double rot[9];
  double near;
};

static PinholeDev make_pinhole(const salf_camera_t *cam, double near, int tile) {
  PinholeDev p;
  p.width = cam->width;
  p.height = cam->height;
  p.tile = tile;
  p.tiles_x = (cam->width + tile - 1) / tile;
  p.tiles_y = (cam->height + tile - 1) / tile;
  p.fx = cam->fx; p.fy = cam->fy; p.cx = cam->cx; p.cy = cam->cy;
  for (int k = 0; k < 3; ++k) p.pos[k] = cam->position[k];
  for (int k = 0; k < 9; ++k) p.rot[k] = cam->rot[k];
  p.near = near;
  return p;
}

// ---------------------------------------------------------------------------
// projection + spans

__device__ __forceinline__ void span_from_rect(double umin, double vmin, double umax, double vmax,
                                               const PinholeDev &c, bool culled, int4 &span) {
  // cull_and_bin pixel-centre coverage (render_raster.py:151-166)
  double u_lo = npmax(ceil(umin - 0.5), 0.0);
  double u_hi = npmin(floor(umax - 0.5), (double)(c.width - 1));
  double v_lo = npmax(ceil(vmin - 0.5), 0.0);
  double v_hi = npmin(floor(vmax - 0.5), (double)(c.height - 1));
  bool vis = !culled && (u_lo <= u_hi) && (v_lo <= v_hi);
  if (!vis) {
    span = make_int4(1, 1, 0, 0);
    return;
  }
  span = make_int4((int)u_lo / c.tile, (int)v_lo / c.tile, (int)u_hi / c.tile, (int)v_hi / c.tile);
}

// Packed conservative pixel-row range of a voxel's footprint (lo | hi << 16,
// clamped to the image; lo > hi when it covers no pixel row).
__device__ __forceinline__ int32_t pack_rows(double v0, double v1, int height) {
  const double lo = npmax(ceil(v0 - 0.5), 0.0), hi = npmin(floor(v1 - 0.5), (double)(height - 1));
  if (!(lo <= hi)) return 1;  // lo = 1, hi = 0: empty
  return (int32_t)lo | ((int32_t)hi << 16);
}

__global__ void k_project(int64_t n, const double4 *__restrict__ geo, const double *__restrict__ vrot, PinholeDev c,
                          double4 *__restrict__ rect, double *__restrict__ zc_out,
                          uint8_t *__restrict__ culled_out, int4 *__restrict__ span_ref,
                          int4 *__restrict__ span_fit, uint64_t *__restrict__ zkey,
                          int32_t *__restrict__ vrange) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 g = geo[i];
  const double ctr[3] = {g.x, g.y, g.z};
  double pc[8][3];
  int n_front = 0, n_back = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    // corner = centre + offset * edge; offsets x fastest (render_raster.py:32-34, :106-109)
    const double off[3] = {(k & 1) ? 0.5 : -0.5, (k & 2) ? 0.5 : -0.5, (k & 4) ? 0.5 : -0.5};
    double ofs[3] = {__dmul_rn(off[0], g.w), __dmul_rn(off[1], g.w), __dmul_rn(off[2], g.w)};
    if (vrot) {  // rotated voxels: offs = R . offs, einsum("nij,nkj->nki") order (p0 + p2) + p1
      const double *R = vrot + 9 * i;
      double r3[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        r3[a] = __dadd_rn(__dadd_rn(__dmul_rn(R[3 * a], ofs[0]), __dmul_rn(R[3 * a + 2], ofs[2])), __dmul_rn(R[3 * a + 1], ofs[1]));
      ofs[0] = r3[0]; ofs[1] = r3[1]; ofs[2] = r3[2];
    }
    double rel[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) rel[j] = __dsub_rn(__dadd_rn(ctr[j], ofs[j]), c.pos[j]);
#pragma unroll
    for (int j = 0; j < 3; ++j) pc[k][j] = mm_col(rel, c.rot, j);  // (corners - pos) @ R
    if (pc[k][2] <= c.near) ++n_back; else ++n_front;
  }
  double relc[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) relc[j] = __dsub_rn(ctr[j], c.pos[j]);
  const double zc = mm_col(relc, c.rot, 2);
  const bool culled = (n_back == 8);
  const bool straddle = !culled && n_back > 0;
  double umin = INFINITY, vmin = INFINITY, umax = -INFINITY, vmax = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (pc[k][2] > c.near) {
      // cam.fx * p_cam[..., 0] / z + cam.cx  (render_raster.py:117-118)
      double u = __dadd_rn(__ddiv_rn(__dmul_rn(c.fx, pc[k][0]), pc[k][2]), c.cx);
      double v = __dadd_rn(__ddiv_rn(__dmul_rn(c.fy, pc[k][1]), pc[k][2]), c.cy);
      umin = npmin(umin, u); umax = npmax(umax, u);
      vmin = npmin(vmin, v); vmax = npmax(vmax, v);
    }
  }
  double r0 = umin, r1 = vmin, r2 = umax, r3 = vmax;
  if (straddle) { r0 = 0.0; r1 = 0.0; r2 = (double)c.width; r3 = (double)c.height; }
  if (culled) { r0 = r1 = r2 = r3 = NAN; }
  if (rect) rect[i] = make_double4(r0, r1, r2, r3);
  if (zc_out) zc_out[i] = zc;
  if (culled_out) culled_out[i] = culled ? 1 : 0;
  int4 sref;
  span_from_rect(r0, r1, r2, r3, c, culled, sref);
  if (span_ref) span_ref[i] = sref;
  // conservative footprint rows widened by one pixel (front voxels: the
  // corner hull; straddlers: the near-plane-clipped hull below)
  if (vrange && !straddle) {
    vrange[2 * i] = culled ? 1 : pack_rows(vmin - 1.0, vmax + 1.0, c.height);
    vrange[2 * i + 1] = culled ? 1 : pack_rows(umin - 1.0, umax + 1.0, c.width);  // columns, same packing
  }
  if (span_fit || vrange) {
    int4 sfit = sref;
    if (straddle && sref.x <= sref.z) {
      // Tight footprint of cube ∩ {z_cam >= near}: the projection of its
      // vertices (front corners + edge crossings of the near plane), widened
      // by one pixel.  Pixels outside it cannot produce t1 > t0 for this
      // voxel, so dropping it from their tiles leaves every sum unchanged.
      double fu0 = umin, fv0 = vmin, fu1 = umax, fv1 = vmax;
#pragma unroll
      for (int e = 0; e < 12; ++e) {
        // 12 cube edges: 4 along each axis
        const int axis = e >> 2, w = e & 3;
        int a, b;
        if (axis == 0) { a = (w & 1) * 2 + (w >> 1) * 4; b = a + 1; }
        else if (axis == 1) { a = (w & 1) + (w >> 1) * 4; b = a + 2; }
        else { a = (w & 1) + (w >> 1) * 2; b = a + 4; }
        const double za = pc[a][2], zb = pc[b][2];
        if ((za <= c.near) != (zb <= c.near)) {
          const double s = (c.near - za) / (zb - za);
          const double x = pc[a][0] + s * (pc[b][0] - pc[a][0]);
          const double y = pc[a][1] + s * (pc[b][1] - pc[a][1]);
          const double u = c.fx * x / c.near + c.cx, v = c.fy * y / c.near + c.cy;
          fu0 = fmin(fu0, u); fu1 = fmax(fu1, u);
          fv0 = fmin(fv0, v); fv1 = fmax(fv1, v);
        }
      }
      int4 t;
      span_from_rect(fu0 - 1.0, fv0 - 1.0, fu1 + 1.0, fv1 + 1.0, c, false, t);
      sfit = t;
      if (vrange) {
        vrange[2 * i] = pack_rows(fv0 - 1.0, fv1 + 1.0, c.height);
        vrange[2 * i + 1] = pack_rows(fu0 - 1.0, fu1 + 1.0, c.width);
      }
    } else if (straddle && vrange) {
      vrange[2 * i] = vrange[2 * i + 1] = 1;  // no pixel
    }
    if (span_fit) span_fit[i] = sfit;
  }
  if (zkey) zkey[i] = order_key(zc);
}

// ---------------------------------------------------------------------------
// binning

// Visible voxels (non-empty span) in ascending index order, their depth keys
// and instance counts, in one pass: CTA tile of 2048 voxels (warp w owns 256
// consecutive voxels, ballots give the in-warp order), decoupled look-back for
// the tile's output position.  nums[0] = visible voxels (written by the last
// tile), nums[1] = instances (atomic).
__global__ void __launch_bounds__(sortk::kBlock) k_select_vis(int64_t n, const int4 *__restrict__ span,
                                                              const uint64_t *__restrict__ zkey,
                                                              int64_t *__restrict__ cnt, int32_t *__restrict__ vis_idx,
                                                              uint64_t *__restrict__ zk_vis,
                                                              uint64_t *__restrict__ status,
                                                              uint32_t *__restrict__ ticket, int64_t *__restrict__ nums) {
  using namespace sortk;
  __shared__ uint32_t s_tile;
  __shared__ int64_t s_w[kWarps + 1];
  __shared__ int64_t s_c[kWarps];
  __shared__ int64_t s_base;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t wbase = (int64_t)tile * kScanTile + (int64_t)w * (32 * kScanItems);
  uint32_t ball[kScanItems];
  int wcount = 0;
  int64_t csum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t idx = wbase + 32 * k + lane;
    int64_t c = 0;
    if (idx < n) {
      const int4 s = span[idx];
      c = (s.x <= s.z && s.y <= s.w) ? (int64_t)(s.z - s.x + 1) * (s.w - s.y + 1) : 0;
      cnt[idx] = c;
    }
    ball[k] = __ballot_sync(0xffffffffu, c > 0);
    wcount += __popc(ball[k]);
    csum += c;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  if (lane == 0) {
    s_w[w] = wcount;
    s_c[w] = csum;
  }
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0, inst = 0;
    for (int i = 0; i < kWarps; ++i) {
      const int64_t c = s_w[i];
      s_w[i] = run;
      run += c;
      inst += s_c[i];
    }
    if (inst) atomicAdd(reinterpret_cast<unsigned long long *>(nums + 1), (unsigned long long)inst);
    const int64_t pre = (int64_t)lookback64(status, tile, (uint64_t)run);
    s_base = pre;
    if ((int64_t)(tile + 1) * kScanTile >= n) nums[0] = pre + run;
  }
  __syncthreads();
  int64_t pos = s_base + s_w[w];
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (ball[k] >> lane & 1u) {
      const int64_t idx = wbase + 32 * k + lane;
      const int64_t q = pos + __popc(ball[k] & lt);
      vis_idx[q] = (int32_t)idx;
      zk_vis[q] = zkey[idx];
    }
    pos += __popc(ball[k]);
  }
}

// base_r[r] = exclusive prefix of the instance counts in depth-rank order
// (r < nums[0]); thread t owns 8 consecutive ranks, look-back across CTAs.
__global__ void __launch_bounds__(sortk::kBlock) k_scan_ranked(const int64_t *__restrict__ nums,
                                                               const int32_t *__restrict__ sorted_vis,
                                                               const int64_t *__restrict__ cnt,
                                                               int64_t *__restrict__ base_r,
                                                               uint64_t *__restrict__ status,
                                                               uint32_t *__restrict__ ticket) {
  using namespace sortk;
  __shared__ uint32_t s_tile;
  __shared__ int64_t s_w[kWarps + 1];
  __shared__ int64_t s_pre;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t n = nums[0];
  const int64_t r0 = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  if ((int64_t)tile * kScanTile >= n) return;  // uniform
  int64_t c[kScanItems], sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    c[k] = (r0 + k < n) ? cnt[sorted_vis[r0 + k]] : 0;
    sum += c[k];
  }
  int64_t total;
  int64_t ex = block_excl_scan(sum, s_w, total);
  if (threadIdx.x == 0) s_pre = (int64_t)lookback64(status, tile, (uint64_t)total);
  __syncthreads();
  ex += s_pre;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (r0 + k < n) base_r[r0 + k] = ex;
    ex += c[k];
  }
}

// One group of kEmitLanes lanes per visible voxel, in global depth-rank order:
// its instances are written at base_r[rank] with the tile id as the (only)
// sort key, so a stable sort by tile leaves every tile's list in (z, index)
// order.  Lanes stride over the voxel's tiles (spans can be the full image for
// straddling voxels in reference mode).  Instances past `cap` are not written
// (the caller sees nums[1] > cap and re-bins with a larger capacity).
constexpr int kEmitLanes = 8;

__global__ void k_emit(const int64_t *__restrict__ nums, const int32_t *__restrict__ sorted_vis,
                       const int4 *__restrict__ span, const int64_t *__restrict__ base_r, int tiles_x, int64_t cap,
                       uint32_t *__restrict__ keys, int32_t *__restrict__ vals) {
  // ~11 instances per visible voxel at C2; a span covers at most the tile
  // grid, so the 32-bit row/column split is exact.  Grid-stride over the ranks
  // (the visible count is only known on the device).
  const int lane = threadIdx.x % kEmitLanes;
  const int64_t n_vis = nums[0];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / kEmitLanes;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kEmitLanes; r < n_vis; r += stride) {
    const int32_t v = sorted_vis[r];
    const int4 s = span[v];
    const int nx = s.z - s.x + 1;
    const int cnt = nx * (s.w - s.y + 1);
    const int64_t b = base_r[r];
    // past the capacity: write the part that fits, so every slot below the capacity holds a real
    // (tile, voxel) instance -- the truncated lists are composited (then re-binned) and must only
    // name real voxels
    if (b >= cap) continue;
    const int lim = (int)min((int64_t)cnt, cap - b);
    int ty = s.y + lane / nx, tx = s.x + lane % nx;
    const int dy = kEmitLanes / nx, dx = kEmitLanes % nx;
    for (int k = lane; k < lim; k += kEmitLanes) {
      keys[b + k] = (uint32_t)(ty * tiles_x + tx);
      vals[b + k] = v;
      tx += dx;  // advance by kEmitLanes instances in row-major order
      ty += dy;
      if (tx > s.z) {
        tx -= nx;
        ++ty;
      }
    }
  }
}

__global__ void k_offsets(int n_tiles, const int64_t *__restrict__ nums, int64_t cap,
                          const uint32_t *__restrict__ keys, int64_t *__restrict__ offsets) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n_tiles) return;
  const int64_t n_inst = min(nums[1], cap);
  // lower_bound of tile t in the sorted keys
  int64_t lo = 0, hi = n_inst;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < (uint32_t)t) lo = mid + 1; else hi = mid;
  }
  offsets[t] = lo;
}

static inline int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------------------
// composite

struct Entry {
  double o[3];   // camera position - voxel centre
  double lo[3];  // (-half) - o
  double hi[3];  //   half  - o
  double half;   // 0.5 * edge
  double inv_half;
  double a, inv_b;  // density transfer (aux)
  int64_t vid;
  VoxPrm p;       // field parameters, staged once per tile chunk
  int rot;        // rotated voxel (flattened actor): R is read from scene.rot
};

struct PixelRay {
  double d[3], inv[3], t_near;
  float gam[4];  // SH basis of the pixel direction (fp32 colour path)
  bool zero[3];
  bool pos[3];  // inv > 0: the slab's near face is the low face (no per-pair min/max)
  bool fast;    // all components non-zero with finite reciprocals (no NaN can arise)
};

__device__ __forceinline__ void pixel_ray(const PinholeDev &c, int px, int py, PixelRay &r) {
  // gen_camera_rays pinhole (sensors.py:131-151) + t_near (render_raster.py:214-215)
  const double u = (double)px + 0.5, v = (double)py + 0.5;
  double dc[3] = {__ddiv_rn(__dsub_rn(u, c.cx), c.fx), __ddiv_rn(__dsub_rn(v, c.cy), c.fy), 1.0};
  const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dc[0], dc[0]), __dmul_rn(dc[1], dc[1])),
                                    __dmul_rn(dc[2], dc[2])));
#pragma unroll
  for (int k = 0; k < 3; ++k) dc[k] = __ddiv_rn(dc[k], nrm);
#pragma unroll
  for (int k = 0; k < 3; ++k) r.d[k] = mm_row(dc, c.rot, k);  // d_cam @ R.T
  const double dz = mm_col(r.d, c.rot, 2);                   // (dirs @ R)[:, 2]
  r.t_near = __ddiv_rn(c.near, dz);
  r.gam[0] = (float)kShC0;
  r.gam[1] = (float)(kShC1 * r.d[1]);
  r.gam[2] = (float)(kShC1 * r.d[2]);
  r.gam[3] = (float)(kShC1 * r.d[0]);
  r.fast = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.zero[k] = (r.d[k] == 0.0);
    r.inv[k] = 1.0 / r.d[k];
    r.pos[k] = r.inv[k] > 0.0;
    r.fast = r.fast && !r.zero[k] && isfinite(r.inv[k]);
  }
}

// The pixel ray seen in a rotated voxel's frame: d' = R^T d in the reference's
// einsum("nji,nj->ni") order (render_raster.py:191-196); t_near is unchanged.
__device__ __forceinline__ void rotate_ray(const PixelRay &r, const double *R, PixelRay &out) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    out.d[i] = __dadd_rn(__dadd_rn(__dmul_rn(R[i], r.d[0]), __dmul_rn(R[3 + i], r.d[1])), __dmul_rn(R[6 + i], r.d[2]));
  out.t_near = r.t_near;
  out.gam[0] = (float)kShC0;
  out.gam[1] = (float)(kShC1 * out.d[1]);
  out.gam[2] = (float)(kShC1 * out.d[2]);
  out.gam[3] = (float)(kShC1 * out.d[0]);
  out.fast = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    out.zero[k] = (out.d[k] == 0.0);
    out.inv[k] = 1.0 / out.d[k];
    out.pos[k] = out.inv[k] > 0.0;
    out.fast = out.fast && !out.zero[k] && isfinite(out.inv[k]);
  }
}

__device__ __forceinline__ double fmax_sel(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double fmin_sel(double a, double b) { return a < b ? a : b; }

// slab test of a pixel ray against a staged entry -> (t0, t_out, hit)
__device__ __forceinline__ bool pair_hit(const PixelRay &r, const Entry &e, double &t0, double &t1) {
  if (r.fast) {
    // lo < hi, so for inv > 0 the reference's min(ta, tb) is ta = lo * inv
    // exactly (rounding is monotone) and max is tb; no NaN is possible.
    const double n0 = __dmul_rn(r.pos[0] ? e.lo[0] : e.hi[0], r.inv[0]);
    const double f0 = __dmul_rn(r.pos[0] ? e.hi[0] : e.lo[0], r.inv[0]);
    const double n1 = __dmul_rn(r.pos[1] ? e.lo[1] : e.hi[1], r.inv[1]);
    const double f1 = __dmul_rn(r.pos[1] ? e.hi[1] : e.lo[1], r.inv[1]);
    const double n2 = __dmul_rn(r.pos[2] ? e.lo[2] : e.hi[2], r.inv[2]);
    const double f2 = __dmul_rn(r.pos[2] ? e.hi[2] : e.lo[2], r.inv[2]);
    const double ti = fmax_sel(fmax_sel(n0, n1), n2);
    t1 = fmin_sel(fmin_sel(f0, f1), f2);
    t0 = fmax_sel(fmax_sel(ti, r.t_near), 0.0);
    return t1 > __dadd_rn(t0, 1e-12);
  }
  double ti = 0.0, to = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double nk, fk;
    if (r.zero[k]) {
      const bool inside = (e.o[k] >= -e.half) && (e.o[k] <= e.half);
      nk = inside ? -INFINITY : INFINITY;
      fk = inside ? INFINITY : -INFINITY;
    } else {
      const double ta = __dmul_rn(e.lo[k], r.inv[k]);
      const double tb = __dmul_rn(e.hi[k], r.inv[k]);
      nk = npmin(ta, tb);
      fk = npmax(ta, tb);
    }
    if (k == 0) { ti = nk; to = fk; }
    else { ti = npmax(ti, nk); to = npmin(to, fk); }
  }
  t0 = npmax(npmax(ti, r.t_near), 0.0);
  t1 = to;
  return t1 > __dadd_rn(t0, 1e-12);
}

struct SegVals {
  double tm, delta, x[3], s, e, sigma, alpha, om, c[3], a, inv_b;
  double dir[3];  // view direction in the voxel's frame
  float cf[3];    // fp32 colour (fast mode)
};

// Fields of one hit pair (render_raster.py:239-253), with the ray direction
// `dir` in the voxel's frame (the pixel ray, or R^T d for rotated voxels).
// Divisions by 0.5*edge and by b are multiplications by precomputed
// reciprocals (<= 1 ulp).
template <bool kExactColor>
__device__ __forceinline__ void shade_pair(const salf_scene_t &sc, const double dir[3], const float gam[4],
                                           const Entry &e, double t0, double t1, SegVals &sv) {
  sv.delta = __dsub_rn(t1, t0);
  sv.tm = __dmul_rn(0.5, __dadd_rn(t0, t1));
#pragma unroll
  for (int k = 0; k < 3; ++k) sv.x[k] = __dmul_rn(__dadd_rn(e.o[k], __dmul_rn(sv.tm, dir[k])), e.inv_half);
  sv.dir[0] = dir[0]; sv.dir[1] = dir[1]; sv.dir[2] = dir[2];
  sv.a = e.a;
  sv.inv_b = e.inv_b;
  sv.s = eval_sdf(e.p, sv.x);
  sv.sigma = density(sc.density_mode, sv.s, e.a, e.inv_b, sv.e);
  sv.alpha = seg_alpha(sv.sigma, sv.delta, sv.om);
  if (kExactColor) {
    eval_color64(e.p, sv.x, dir, sv.c);
  } else {
    const float xf[3] = {(float)sv.x[0], (float)sv.x[1], (float)sv.x[2]};
    eval_color32g(e.p, xf, gam, sv.cf);
    sv.c[0] = sv.cf[0]; sv.c[1] = sv.cf[1]; sv.c[2] = sv.cf[2];
  }
}

// Pair test + fields for one staged entry; rotated entries (flattened actor
// voxels) are tested and shaded with the ray in the voxel's frame.  One
// shading instance serves both cases (only the slab test is duplicated).
template <bool kExactColor, bool kRot>
__device__ __forceinline__ bool hit_and_shade(const salf_scene_t &sc, const PixelRay &r, const Entry &e, SegVals &sv) {
  double t0, t1;
  if (!kRot) {
    if (!pair_hit(r, e, t0, t1)) return false;
    shade_pair<kExactColor>(sc, r.d, r.gam, e, t0, t1, sv);
    return true;
  }
  PixelRay rr;
  bool hit;
  if (!e.rot) {
    hit = pair_hit(r, e, t0, t1);
  } else {
    rotate_ray(r, sc.rot + 9 * e.vid, rr);
    hit = pair_hit(rr, e, t0, t1);
  }
  if (!hit) return false;
  double dir[3];
  float gam[4];
#pragma unroll
  for (int k = 0; k < 3; ++k) dir[k] = e.rot ? rr.d[k] : r.d[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) gam[k] = e.rot ? rr.gam[k] : r.gam[k];
  shade_pair<kExactColor>(sc, dir, gam, e, t0, t1, sv);
  return true;
}

template <bool kRot>
__device__ __forceinline__ void stage_entry(const salf_scene_t &sc, const PinholeDev &c, int32_t vid,
                                            Entry &e) {
  const double4 g = ldg_d4(sc.geo + 4 * (int64_t)vid);
  const double2 ab = __ldg(reinterpret_cast<const double2 *>(sc.aux + 4 * (int64_t)vid));
  e.vid = vid;
  e.a = ab.x;
  e.inv_b = ab.y;
  load_prm(sc.prm, vid, e.p);
  e.half = __dmul_rn(0.5, g.w);
  e.inv_half = 1.0 / e.half;
  e.o[0] = __dsub_rn(c.pos[0], g.x);
  e.o[1] = __dsub_rn(c.pos[1], g.y);
  e.o[2] = __dsub_rn(c.pos[2], g.z);
  e.rot = 0;
  if (kRot) {
    const double *R = sc.rot + 9 * (int64_t)vid;
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (R[k] != ((k % 4 == 0) ? 1.0 : 0.0)) e.rot = 1;
    if (e.rot) {  // o' = R^T o (einsum "nji,nj->ni", render_raster.py:195)
      double o2[3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        o2[i] = __dadd_rn(__dadd_rn(__dmul_rn(R[i], e.o[0]), __dmul_rn(R[3 + i], e.o[1])), __dmul_rn(R[6 + i], e.o[2]));
      e.o[0] = o2[0]; e.o[1] = o2[1]; e.o[2] = o2[2];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e.lo[k] = __dsub_rn(-e.half, e.o[k]);
    e.hi[k] = __dsub_rn(e.half, e.o[k]);
  }
}

#ifndef SALF_CHUNK
#define SALF_CHUNK 64
#endif
#ifndef SALF_CHUNKB
#define SALF_CHUNKB 32
#endif
constexpr int kChunk = SALF_CHUNK;    // forward: entries staged per step in shared memory
// Hit words (forward -> backward): bit b of word w of pixel slot p of a tile is
// "list position 32 w + b of the tile is an included hit of that pixel"
// (the reference's hit AND inclusion decisions, as certified by the forward or
// recomputed by the fp64 redo).  Tile t's words start at 256 (off[t] / 32 + t):
// ceil(len / 32) <= floor(off[t+1] / 32) - floor(off[t] / 32) + 1, so tiles never
// overlap and the whole array is 256 (I / 32 + T + 1) words.
constexpr int kHitSlots = 256;  // pixel slots per tile word row (tile <= 16)
__device__ __forceinline__ int64_t hit_word_base(int64_t beg, int tile_id) {
  return (int64_t)kHitSlots * (beg / 32 + tile_id);
}
constexpr int kChunkB = SALF_CHUNKB;  // backward: + a kChunkB x warps x 27 fp32 reduction buffer

// fp64 parity-mode composite (exact_color=True): the reference-order
// arithmetic everywhere, fp64 colour.
template <bool kRot>
__global__ void __launch_bounds__(256, 3) k_composite(salf_scene_t sc, PinholeDev c, salf_raster_opts_t opt,
                                                   const int64_t *__restrict__ offsets,
                                                   const int32_t *__restrict__ entries, float *__restrict__ out_rgb,
                                                   float *__restrict__ out_op, float *__restrict__ out_depth,
                                                   double *__restrict__ saved) {
  __shared__ Entry sm[kChunk];
  const int tile_id = blockIdx.x;
  const int tx = tile_id % c.tiles_x, ty = tile_id / c.tiles_x;
  const int lx = threadIdx.x % c.tile, ly = threadIdx.x / c.tile;
  const int px = tx * c.tile + lx, py = ty * c.tile + ly;
  const bool inside = px < c.width && py < c.height && threadIdx.x < c.tile * c.tile;
  const int64_t beg = offsets[tile_id], end = offsets[tile_id + 1];
  const double keep = 1.0 - opt.stop_threshold;

  PixelRay r;
  if (inside) pixel_ray(c, px, py, r);
  // transmittance kept as a running product of (1 - alpha) (the reference's
  // exp(cumsum(log1p(-alpha))), render_raster.py:258-274, to ~1e-15)
  double acc_c[3] = {0.0, 0.0, 0.0}, acc_w = 0.0, acc_wt = 0.0, T = 1.0;
  bool alive = inside;
  int64_t n_stop = end - beg;
  int n_inc = 0;  // included segments of this pixel (work statistics, saved[7])
  const int nthreads = blockDim.x;

  for (int64_t base = beg; base < end; base += kChunk) {
    const int cn = (int)min((int64_t)kChunk, end - base);
    __syncthreads();
    for (int j = threadIdx.x; j < cn; j += nthreads) stage_entry<kRot>(sc, c, entries[base + j], sm[j]);
    __syncthreads();
    if (alive) {
      for (int j = 0; j < cn; ++j) {
        SegVals sv;
        if (!hit_and_shade<true, kRot>(sc, r, sm[j], sv)) continue;
        if (T > keep) {  // included iff T_before > 1 - stop_threshold
          const double w = __dmul_rn(T, sv.alpha);
#pragma unroll
          for (int k = 0; k < 3; ++k) acc_c[k] = __dadd_rn(acc_c[k], __dmul_rn(w, sv.c[k]));
          acc_w = __dadd_rn(acc_w, w);
          acc_wt = __dadd_rn(acc_wt, __dmul_rn(w, sv.tm));
          T = __dmul_rn(T, sv.om);
          ++n_inc;
        } else {
          alive = false;
          n_stop = base - beg + j;
          break;
        }
      }
    }
    if (!__syncthreads_or(alive)) break;
  }
  if (!inside) return;
  const int64_t pix = (int64_t)py * c.width + px;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    out_rgb[pix * 3 + k] = (float)__dadd_rn(acc_c[k], __dmul_rn(T, opt.background[k]));
  out_op[pix] = (float)__dsub_rn(1.0, T);
  out_depth[pix] = acc_w > kDepthWeightMin ? (float)__ddiv_rn(acc_wt, acc_w) : NAN;
  if (saved) {
    double *s = saved + pix * SALF_SAVED_STRIDE;
    s[0] = acc_c[0]; s[1] = acc_c[1]; s[2] = acc_c[2];
    s[3] = acc_w; s[4] = acc_wt; s[5] = T; s[6] = (double)n_stop; s[7] = (double)n_inc;
  }
}

// ---------------------------------------------------------------------------
// backward

// fp64 parity-mode backward (exact_color=True), reference operation order.
template <bool kRot>
#ifndef SALF_BWD_MINB
#define SALF_BWD_MINB 2
#endif
__global__ void __launch_bounds__(256, SALF_BWD_MINB) k_backward(salf_scene_t sc, PinholeDev c, salf_raster_opts_t opt,
                                                  const int64_t *__restrict__ offsets,
                                                  const int32_t *__restrict__ entries,
                                                  const double *__restrict__ saved, const double *__restrict__ d_rgb,
                                                  const double *__restrict__ d_depth, double *__restrict__ grad,
                                                  float *__restrict__ partial) {
  __shared__ Entry sm[kChunkB];
  const int tile_id = blockIdx.x;
  const int tx = tile_id % c.tiles_x, ty = tile_id / c.tiles_x;
  const int lx = threadIdx.x % c.tile, ly = threadIdx.x / c.tile;
  const int px = tx * c.tile + lx, py = ty * c.tile + ly;
  const bool inside = px < c.width && py < c.height && threadIdx.x < c.tile * c.tile;
  const int64_t beg = offsets[tile_id];
  const double keep = 1.0 - opt.stop_threshold;
  const int nthreads = blockDim.x;

  PixelRay r;
  double dC[3] = {0, 0, 0}, total = 0.0, tail = 0.0, D = 0.0, dd = 0.0, ws = 1.0, prefix = 0.0, T = 1.0;
  int64_t n_stop = 0;
  if (inside) {
    pixel_ray(c, px, py, r);
    const int64_t pix = (int64_t)py * c.width + px;
    const double *s = saved + pix * SALF_SAVED_STRIDE;
    for (int k = 0; k < 3; ++k) dC[k] = d_rgb[pix * 3 + k];
    const double acc_w = s[3], acc_wt = s[4];
    // depth_valid / depth_safe / wsum_safe (backward.py:46-49)
    const bool ok = acc_w > kDepthWeightMin;
    dd = (ok && d_depth) ? d_depth[pix] : 0.0;
    D = ok ? __ddiv_rn(acc_wt, acc_w) : 0.0;
    ws = ok ? acc_w : 1.0;
    // sum_j A_j w_j = dC . acc_rgb + dD (acc_wt - D acc_w) / ws  (suffix sums by subtraction)
    total = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(dC[0], s[0]), __dmul_rn(dC[2], s[2])), __dmul_rn(dC[1], s[1])),
                      __ddiv_rn(__dmul_rn(dd, __dsub_rn(acc_wt, __dmul_rn(D, acc_w))), ws));
    // tail = (dC . background) * T_final  (backward.py:62)
    tail = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(dC[0], opt.background[0]), __dmul_rn(dC[2], opt.background[2])),
                               __dmul_rn(dC[1], opt.background[1])),
                     s[5]);
    n_stop = (int64_t)s[6];
  }
  int64_t max_stop = n_stop;
  // CTA-wide bound on the entries any pixel still needs
  __shared__ long long s_max;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  atomicMax(&s_max, (long long)max_stop);
  __syncthreads();
  const int64_t lim = beg + (int64_t)s_max;

  // Two-level reduction: each warp reduces its lanes' 27-vectors for entry j
  // (transposed shuffle reduction) into red[j][warp][.]; after the chunk the
  // CTA sums its warps and issues one fp64 atomic per (entry, component).
  __shared__ float red[kChunkB][8][kGradStride];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = nthreads >> 5;
  for (int64_t base = beg; base < lim; base += kChunkB) {
    const int cn = (int)min((int64_t)kChunkB, lim - base);
    __syncthreads();
    for (int j = threadIdx.x; j < cn; j += nthreads) stage_entry<kRot>(sc, c, entries[base + j], sm[j]);
    __syncthreads();
    for (int j = 0; j < cn; ++j) {
      const int64_t jj = base - beg + j;
      float g[32];
      bool act = false;
      SegVals sv;
      if (inside && jj < n_stop && hit_and_shade<true, kRot>(sc, r, sm[j], sv)) {
        if (T > keep) {
          const double w = __dmul_rn(T, sv.alpha);
          // A = dC . c + dD (t_mid - D) / ws   (backward.py:52-59, einsum order (0+2)+1)
          const double A = __dadd_rn(
              __dadd_rn(__dadd_rn(__dmul_rn(dC[0], sv.c[0]), __dmul_rn(dC[2], sv.c[2])), __dmul_rn(dC[1], sv.c[1])),
              __ddiv_rn(__dmul_rn(dd, __dsub_rn(sv.tm, D)), ws));
          prefix = __dadd_rn(prefix, __dmul_rn(A, w));
          const double suffix = __dsub_rn(total, prefix);
          segment_grad(sc.density_mode, sv.delta, sv.sigma, sv.alpha, sv.om, sv.s, sv.e, sv.a, sv.inv_b, sv.x, sv.c,
                       sv.dir, A, T, w, suffix, tail, dC, g);
          act = true;
          T = __dmul_rn(T, sv.om);
        }
      }
      // every active lane of this warp holds entry j's voxel: one group
      float tot = 0.0f;
      if (__ballot_sync(0xffffffffu, act)) {
#pragma unroll
        for (int k = 0; k < 32; ++k) g[k] = act ? g[k] : 0.0f;
        tot = warp_transpose_reduce(g);
      }
      if (lane < kGradStride) red[j][warp][lane] = tot;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < cn * kGradStride; q += nthreads) {
      const int j = q / kGradStride, k = q - j * kGradStride;
      float sum = 0.0f;
      for (int w = 0; w < nwarps; ++w) sum += red[j][w][k];
      if (partial) partial[(base + j) * kGradStride + k] = sum;  // deterministic mode
      else if (sum != 0.0f) atomicAdd(grad + sm[j].vid * kGradStride + k, (double)sum);
    }
  }
  (void)keep;
}

// Mixed-precision backward (default, fast mode).  Which entries a pixel
// includes is fixed by the forward: the hits before its saved stop index
// n_stop (inclusion is monotone in T), so no fp64 transmittance is needed to
// reproduce it.  What stays fp64 is what is ill-conditioned at driving-scene
// distances (camera-voxel distance ~1000x the voxel edge): the slab test,
// delta, t_mid, the local coordinates x and t_mid - D.  Everything after x
// (SDF, density, alpha, colour, the gradient chain) is fp32; the prefix sum
// of A w stays fp64 because the suffix is recovered by subtraction.
// Segment fields in the reference's order: backward.py:52-100.
//
// Each thread owns NP pixels of the tile (rows ly, ly + rows/NP, ...): their
// 27-vectors are summed in registers before the warp's transposed
// reduction, so the shuffle reduction, the staged-entry reads and the loop
// overhead are paid once per NP pixels.

// Pixel ray for the mixed-precision pair test: fp64 direction (for the
// closest-approach parameter), fp32 direction / reciprocals / SH basis.
struct RayF {
  double d[3];
  double tn0;  // max(t_near, 0)
  float df[3], dl[3], inv[3], gam[4];  // d = df + dl (two-float split)
  float tn0f;
  float refine;  // backward: chords shorter than refine * h/2 are re-derived in fp64 (pair_hit_bwd)
  bool fast;   // no zero component (else the fp64 reference slab test runs)
};

#ifndef SALF_REFINE_MIN
#define SALF_REFINE_MIN 0.0f
#endif
#ifndef SALF_REFINE_K
#define SALF_REFINE_K 0.05f
#endif
#ifdef SALF_DIAG_CHORD
__device__ unsigned long long g_diag[4];
#endif
#ifndef SALF_REFTOL
#define SALF_REFTOL 5e-5f
#endif
constexpr float kRefTol = SALF_REFTOL;  // fp64 chord when the fp32 chord's bound exceeds this relative error
#ifndef SALF_CHORD_INLINE
#define SALF_CHORD_INLINE __forceinline__
#endif
__device__ __forceinline__ void rayf_from_dir(const double d[3], double t_near, RayF &r) {
  r.fast = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.d[k] = d[k];
    r.df[k] = (float)d[k];
    r.dl[k] = (float)(d[k] - (double)r.df[k]);
    r.inv[k] = 1.0f / r.df[k];
    r.fast = r.fast && d[k] != 0.0 && isfinite(r.inv[k]);
  }
  r.tn0 = t_near > 0.0 ? t_near : 0.0;
  r.tn0f = (float)r.tn0;
  r.refine = fmaxf(SALF_REFINE_MIN, SALF_REFINE_K * fmaxf(fabsf(r.inv[0]), fmaxf(fabsf(r.inv[1]), fabsf(r.inv[2]))));
  r.gam[0] = (float)kShC0;
  r.gam[1] = (float)(kShC1 * d[1]);
  r.gam[2] = (float)(kShC1 * d[2]);
  r.gam[3] = (float)(kShC1 * d[0]);
}

// Staged entry of the mixed-precision backward.
// Layout: the 25 field parameters first (16-B aligned: LDS.128 reads), then
// the scalars, then the fp64 geometry.
struct __align__(16) EntryF {
  VoxPrm p;
  float wn;         // |w_s| 1-norm (error bound of the fp32 SDF)
  float hf, inv_hf; // fp32 half edge and its reciprocal
  float a, inv_b;
  int vid, rot;
  double o[3];      // camera position - voxel centre (fp64)
  double half;      // 0.5 * edge (fp64, for the reference slab test fallback)
  float oh[3], ol[3];  // o = oh + ol (two-float split)
  int vlo, vhi;        // conservative footprint pixel rows (vlo > vhi: none)
  int ulo, uhi;        // and columns
};

template <bool kRot>
__device__ __forceinline__ void stage_entry_f(const salf_scene_t &sc, const PinholeDev &c, int32_t vid, EntryF &e,
                                              const int32_t *__restrict__ vrange) {
  if (vrange) {
    const int2 r = __ldg(reinterpret_cast<const int2 *>(vrange) + vid);
    e.vlo = r.x & 0xffff;
    e.vhi = (r.x >> 16) & 0xffff;
    e.ulo = r.y & 0xffff;
    e.uhi = (r.y >> 16) & 0xffff;
  } else {
    e.vlo = e.ulo = 0;
    e.vhi = e.uhi = 0x7fff;
  }
  const double4 g = ldg_d4(sc.geo + 4 * (int64_t)vid);
  const double2 ab = __ldg(reinterpret_cast<const double2 *>(sc.aux + 4 * (int64_t)vid));
  e.vid = vid;
  e.a = (float)ab.x;
  e.inv_b = (float)ab.y;
  load_prm(sc.prm, vid, e.p);
  e.wn = fabsf(e.p.ws[0]) + fabsf(e.p.ws[1]) + fabsf(e.p.ws[2]) + fabsf(e.p.ws[3]);
  e.half = 0.5 * g.w;
  e.hf = (float)e.half;
  e.inv_hf = (float)(1.0 / e.half);
  e.o[0] = c.pos[0] - g.x;
  e.o[1] = c.pos[1] - g.y;
  e.o[2] = c.pos[2] - g.z;
  e.rot = 0;
  if (kRot) {
    const double *R = sc.rot + 9 * (int64_t)vid;
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (R[k] != ((k % 4 == 0) ? 1.0 : 0.0)) e.rot = 1;
    if (e.rot) {  // o' = R^T o (render_raster.py:195)
      double o2[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) o2[i] = R[i] * e.o[0] + R[3 + i] * e.o[1] + R[6 + i] * e.o[2];
      e.o[0] = o2[0]; e.o[1] = o2[1]; e.o[2] = o2[2];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e.oh[k] = (float)e.o[k];
    e.ol[k] = (float)(e.o[k] - (double)e.oh[k]);
  }
}

// Short chords (grazing pairs): the fp32 slab values carry ~2^-24 h |1/d|
// each, a large RELATIVE error of a chord of length delta << h -- enough to
// turn an fp64 miss into an fp32 hit with y ~ 1e-7 (an opacity of 5e-7 where
// the reference has 0) or to skew a grazing segment's alpha and gradient by
// 1e-3.  The certified forward flags every pixel with a hit whose fp32 chord
// is within its error band of zero (fp64 redo decides it); the backward
// re-derives every chord whose fp32 length is not accurate to ~1e-6 from the
// three slabs and the near plane in fp64 (1/d by one Newton step on the fp32
// reciprocal, |err| ~ 2^-46), kept iff t1 > t0 + 1e-12 (render_raster.py:241),
// so both passes see the reference's hits.
#ifndef SALF_BWD_REFINE
#define SALF_BWD_REFINE 1  // A/B only: 0 keeps every fp32 chord (not parity-safe)
#endif

__device__ SALF_CHORD_INLINE bool chord64(const RayF &r, const EntryF &e, double ts, double &u0, double &u1) {
  u0 = r.tn0 - ts;
  u1 = INFINITY;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double qk = fma(ts, r.d[k], e.o[k]);
    double iv = (double)r.inv[k];
    iv = fma(iv, fma(-r.d[k], iv, 1.0), iv);
    const double hi = fabs(e.half * iv), qi = qk * iv;
    u0 = fmax(u0, -hi - qi);
    u1 = fmin(u1, hi - qi);
  }
  return u1 > u0 + 1e-12;
}

// Error bound of an fp32 chord [u0, u1] from pair_hit_f / pair_hit_bwd,
// evaluated only for chords the cheap whole-ray bound (max_k |1/d_k|) cannot
// certify.  Each slab value -/+ h|1/d_k| - q_k/d_k carries at most
// e_k = (12 u h + 2e-12) |1/d_k| (u = 2^-24; q's two-float / fp64->fp32 error
// included), the near-plane value tn0 - t* at most 2u(|tn0| + |t*|).  The
// computed max (min) can differ from the exact one only through faces whose
// values lie within their errors of it, so |du0| <= E0 = max e_k over the
// near faces k with n_k + e_k >= u0 - e(argmax), and likewise E1 for u1.
// (A ray nearly parallel to one axis has a huge |1/d_k| there, but that face
// is far from deciding the chord, so E0 + E1 stays ~1e-6 h |1/d_active|.)
__device__ __forceinline__ float chord_err(const float inv[3], float hf, const float q[3], float u_near, float u0,
                                        float u1, float t_abs) {
  constexpr float u = 5.9604645e-8f;
  const float ek = __fmaf_rn(12.f * u, hf, 2e-12f);
  const float en = 2.f * u * t_abs;  // error of the near-plane value u_near = tn0 - t*
  float nk[3], fk[3], er[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float qi = q[k] * inv[k], a = fabsf(inv[k]);
    nk[k] = __fmaf_rn(-hf, a, -qi);
    fk[k] = __fmaf_rn(hf, a, -qi);
    er[k] = ek * a;
  }
  // errors of the values that produced u0 and u1
  float e0 = u_near == u0 ? en : 0.f, e1 = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (nk[k] == u0) e0 = fmaxf(e0, er[k]);
    if (fk[k] == u1) e1 = fmaxf(e1, er[k]);
  }
  // every value within reach of the computed max / min
  float E0 = e0, E1 = e1;
  if (u_near + en >= u0 - e0) E0 = fmaxf(E0, en);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (nk[k] + er[k] >= u0 - e0) E0 = fmaxf(E0, er[k]);
    if (fk[k] - er[k] <= u1 + e1) E1 = fmaxf(E1, er[k]);
  }
  return E0 + E1;
}

// Pair test in closest-approach coordinates.  With t* ~ -(o . d) (any
// value near the closest approach to the voxel centre) the ray is q + u d
// with q = o + t* d (|q| ~ the voxel size for any pair that can hit) and
// u = t - t*, so the slab test, delta, t_mid - t* and the local coordinates
// are well-conditioned in fp32 even though |o| ~ 1000 voxel edges.  q is
// evaluated in two-float arithmetic (o = oh + ol, d = dh + dl):
// q = fma(t*, dh, oh) + fma(t*, dl, ol), |dq| <= 2^-23 |q| + 1e-12; t* itself
// is fp32 (its error only moves the reference point along the ray).  No fp64
// and no fp64<->fp32 conversion per pair.  Rays with a zero direction
// component use the fp64 reference slab test (octree.py:184-194).
#ifndef SALF_PAIR_PACK
#define SALF_PAIR_PACK 1  // forward pair test: x and y slabs in fp32x2
#endif
__device__ __forceinline__ bool pair_hit_f(const RayF &r, const EntryF &e, float q[3], float &u0, float &u1,
                                           float &ts) {
  if (r.fast) {
    ts = -__fmaf_rn(e.oh[2], r.df[2], __fmaf_rn(e.oh[1], r.df[1], e.oh[0] * r.df[0]));
    // slab k: u in [(-s h - q) / d, (s h - q) / d], s = sign(d): h |1/d| -/+ q/d
#if SALF_PAIR_PACK
    // axes x and y as fp32x2 (each half the scalar chain's IEEE operations), z scalar
    const float2 tt = make_float2(ts, ts);
    const float2 q01 = __fadd2_rn(__ffma2_rn(tt, make_float2(r.df[0], r.df[1]), make_float2(e.oh[0], e.oh[1])),
                                  __ffma2_rn(tt, make_float2(r.dl[0], r.dl[1]), make_float2(e.ol[0], e.ol[1])));
    q[0] = q01.x;
    q[1] = q01.y;
    q[2] = __fmaf_rn(ts, r.df[2], e.oh[2]) + __fmaf_rn(ts, r.dl[2], e.ol[2]);
    const float2 nqi01 = __fmul2_rn(q01, make_float2(-r.inv[0], -r.inv[1]));  // -q/d (exact negation)
    const float2 ai01 = make_float2(fabsf(r.inv[0]), fabsf(r.inv[1]));
    const float2 n01 = __ffma2_rn(make_float2(-e.hf, -e.hf), ai01, nqi01);
    const float2 f01 = __ffma2_rn(make_float2(e.hf, e.hf), ai01, nqi01);
    const float qi2 = q[2] * r.inv[2];
    const float n2 = __fmaf_rn(-e.hf, fabsf(r.inv[2]), -qi2), f2v = __fmaf_rn(e.hf, fabsf(r.inv[2]), -qi2);
    const float un = fmaxf(fmaxf(fmaxf(-INFINITY, n01.x), n01.y), n2);
    const float uf = fminf(fminf(fminf(INFINITY, f01.x), f01.y), f2v);
#else
    float un = -INFINITY, uf = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      q[k] = __fmaf_rn(ts, r.df[k], e.oh[k]) + __fmaf_rn(ts, r.dl[k], e.ol[k]);
      const float qi = q[k] * r.inv[k];
      un = fmaxf(un, __fmaf_rn(-e.hf, fabsf(r.inv[k]), -qi));
      uf = fminf(uf, __fmaf_rn(e.hf, fabsf(r.inv[k]), -qi));
    }
#endif
    u0 = fmaxf(un, r.tn0f - ts);
    u1 = uf;
    return u1 > u0;
  }
  const double tsd = -fma(e.o[2], r.d[2], fma(e.o[1], r.d[1], e.o[0] * r.d[0]));
  ts = (float)tsd;
  const double t_ref = (double)ts;  // u relative to the fp32 reference point
  double ti = 0.0, to = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    q[k] = (float)fma(t_ref, r.d[k], e.o[k]);
    const double lo = -e.half - e.o[k], hi = e.half - e.o[k];
    double nk, fk;
    if (r.d[k] == 0.0) {
      const bool inside = (e.o[k] >= -e.half) && (e.o[k] <= e.half);
      nk = inside ? -INFINITY : INFINITY;
      fk = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = 1.0 / r.d[k];
      const double ta = lo * inv, tb = hi * inv;
      nk = npmin(ta, tb);
      fk = npmax(ta, tb);
    }
    if (k == 0) { ti = nk; to = fk; }
    else { ti = npmax(ti, nk); to = npmin(to, fk); }
  }
  const double t0 = npmax(ti, r.tn0);
  if (!(to > t0 + 1e-12)) return false;
  u0 = (float)(t0 - t_ref);
  u1 = (float)(to - t_ref);
  return true;
}

// The backward's variant: t* and q in fp64 (6 DFMA), rounded to fp32 once
// for the hit test.  (The two-float form above measured slower in the
// issue-bound backward.)  A chord whose fp32 length is not accurate to ~5e-6
// (delta < refine h/2 with r.refine = 0.05 max_k |1/d_k|; the fp32 slab
// values carry ~1.2e-7 h/2 |1/d_k| each) is re-derived in fp64 (chord64;
// kExact: every chord).  A superset of the chords the forward flags
// (delta <= 2 dd ~ 1.4e-6 h/2 max|1/d|), so both passes see the reference's
// hits.  Outputs delta and um = t_mid - t*.
template <bool kExact>
__device__ __forceinline__ bool pair_hit_bwd(const RayF &r, const EntryF &e, float q[3], float &delta, float &um,
                                           double &ts) {
  ts = -fma(e.o[2], r.d[2], fma(e.o[1], r.d[1], e.o[0] * r.d[0]));
  if (r.fast) {
    // slab k: u in [(-s h - q) / d, (s h - q) / d], s = sign(d): h |1/d| -/+ q/d
    float un = -INFINITY, uf = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      q[k] = (float)fma(ts, r.d[k], e.o[k]);
      const float qi = q[k] * r.inv[k];
      un = fmaxf(un, __fmaf_rn(-e.hf, fabsf(r.inv[k]), -qi));
      uf = fminf(uf, __fmaf_rn(e.hf, fabsf(r.inv[k]), -qi));
    }
    const float u0f = fmaxf(un, (float)(r.tn0 - ts));
    if (!(uf > u0f)) return false;
#ifdef SALF_DIAG_CHORD
    atomicAdd(&g_diag[0], 1ull);
    if (uf - u0f < e.hf * r.refine) {
      atomicAdd(&g_diag[1], 1ull);
      if (chord_err(r.inv, e.hf, q, (float)(r.tn0 - ts), u0f, uf, (float)(fabs(ts) + r.tn0)) > kRefTol * (uf - u0f))
        atomicAdd(&g_diag[2], 1ull);
    }
#endif
    if (kExact || (SALF_BWD_REFINE && uf - u0f < e.hf * r.refine &&
                   chord_err(r.inv, e.hf, q, (float)(r.tn0 - ts), u0f, uf, (float)(fabs(ts) + r.tn0)) > kRefTol * (uf - u0f))) {
      double u0, u1;
      if (!chord64(r, e, ts, u0, u1)) return false;
      delta = (float)(u1 - u0);
      um = (float)(0.5 * (u0 + u1));
      return true;
    }
    delta = uf - u0f;
    um = 0.5f * (u0f + uf);
    return true;
  }
  double ti = 0.0, to = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    q[k] = (float)fma(ts, r.d[k], e.o[k]);
    const double lo = -e.half - e.o[k], hi = e.half - e.o[k];
    double nk, fk;
    if (r.d[k] == 0.0) {
      const bool inside = (e.o[k] >= -e.half) && (e.o[k] <= e.half);
      nk = inside ? -INFINITY : INFINITY;
      fk = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = 1.0 / r.d[k];
      const double ta = lo * inv, tb = hi * inv;
      nk = npmin(ta, tb);
      fk = npmax(ta, tb);
    }
    if (k == 0) { ti = nk; to = fk; }
    else { ti = npmax(ti, nk); to = npmin(to, fk); }
  }
  const double t0 = npmax(ti, r.tn0);
  if (!(to > t0 + 1e-12)) return false;
  delta = (float)(to - t0);
  um = (float)(0.5 * (t0 + to) - ts);
  return true;
}

// Per-pixel backward state.  The default backward walks each pixel's list
// BACK TO FRONT, from its last included hit (the forward's stop index) to the
// first entry, so the reference's suffix sum S_i = sum_{j>i} A_j w_j
// (backward.py:26-32, :62-64) is accumulated directly -- no "total - prefix"
// cancellation -- and the transmittance before each hit is recovered in log
// space, T_i = exp(-(Y_final - sum_{j>=i} y_j)) with the subtraction
// compensated (Neumaier), so its error stays ~1e-7 relative however many hits
// the pixel has.  (A running product of (1 - alpha) front to back loses
// ~n 2^-22 relative; exp(-Y) does not.)
struct BwdPix {
  RayF r;
  float dC[3], dws, tail;
  float Yh, Yc;  // Y after the current hit (compensated fp32), starts at Y_final
  float S;       // suffix sum of A w over the hits behind the current one
  double D;
  int n_stop;
};

__device__ __forceinline__ void bwd_pixel_init(const PinholeDev &c, const salf_raster_opts_t &opt, int px, int py,
                                               const double *__restrict__ saved, const double *__restrict__ d_rgb,
                                               const double *__restrict__ d_depth, BwdPix &q) {
  PixelRay pr;
  pixel_ray(c, px, py, pr);
  rayf_from_dir(pr.d, pr.t_near, q.r);
  const int64_t pix = (int64_t)py * c.width + px;
  const double *s = saved + pix * SALF_SAVED_STRIDE;
  double dCd[3];
  for (int k = 0; k < 3; ++k) dCd[k] = d_rgb[pix * 3 + k];
  const double acc_w = s[3], acc_wt = s[4];
  const bool ok = acc_w > kDepthWeightMin;  // depth_valid (backward.py:46-49)
  const double dd = (ok && d_depth) ? d_depth[pix] : 0.0;
  q.D = ok ? acc_wt / acc_w : 0.0;
  const double ws = ok ? acc_w : 1.0;
  // tail = (dC . background) * T_final (backward.py:62)
  q.tail = (float)((dCd[0] * opt.background[0] + dCd[1] * opt.background[1] + dCd[2] * opt.background[2]) * s[5]);
  q.dws = (float)(dd / ws);
  for (int k = 0; k < 3; ++k) q.dC[k] = (float)dCd[k];
  q.n_stop = (int)s[6];
  const double Yf = -log(s[5]);  // T_final = exp(-Y_final) of the included hits
  q.Yh = (float)Yf;
  q.Yc = (float)(Yf - (double)q.Yh);
  q.S = 0.f;
  if (!(dCd[0] != 0.0 || dCd[1] != 0.0 || dCd[2] != 0.0 || dd != 0.0)) q.n_stop = 0;  // zero seeds: no work
}

// The pair part of one hit (pixel q vs staged entry e): slab test, fp64
// chord for short chords, local coordinates.  Both pixels' pair parts run
// before the 27 gradient accumulators are live (register pressure).
struct PairHit {
  float x[3], delta, dq;
  float gam[4];  // SH basis of the (possibly rotated) ray direction
};

template <bool kRot, bool kDepth = true, bool kExact = false>
__device__ __forceinline__ bool bwd_pair(const salf_scene_t &sc, const EntryF &e, const BwdPix &q, PairHit &h) {
  float qv[3];
  double ts;
  const RayF *ray = &q.r;
  RayF rr;
  if (kRot && e.rot) {  // the pixel ray in the voxel's frame: d' = R^T d (render_raster.py:191-196)
    const double *R = sc.rot + 9 * (int64_t)e.vid;
    double d2[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) d2[i] = R[i] * q.r.d[0] + R[3 + i] * q.r.d[1] + R[6 + i] * q.r.d[2];
    rayf_from_dir(d2, q.r.tn0, rr);
    ray = &rr;
  }
  float um;
  if (!pair_hit_bwd<kExact>(*ray, e, qv, h.delta, um, ts)) return false;
  h.dq = kDepth ? (float)(ts - q.D) + um : 0.f;  // t_mid - D (no depth seeds: unused)
  // (fp32 below: explicit FMAs -- this file is compiled with --fmad=false)
#pragma unroll
  for (int k = 0; k < 3; ++k) h.x[k] = __fmaf_rn(um, ray->df[k], qv[k]) * e.inv_hf;
  if (kRot) {
#pragma unroll
    for (int k = 0; k < 4; ++k) h.gam[k] = ray->gam[k];
  }
  return true;
}

// The pair part of a KNOWN hit (hit words from the forward): the chord in
// fp64 -- the reference's slab test with reciprocal multiply (octree.py:184-194)
// in closest-approach coordinates u = t - t*, 1/d precomputed per pixel
// (iv, IEEE division) -- so delta and t_mid carry ~1e-16 h |1/d| absolute error
// however short the chord, with no per-pair refinement branch.  Kept iff
// t1 > t0 + 1e-12 (render_raster.py:241).  Rotated voxels and rays with a zero
// direction component take the general fp64 path.
template <bool kRot, bool kDepth>
__device__ __forceinline__ bool bwd_pair64(const salf_scene_t &sc, const EntryF &e, const BwdPix &q,
                                           const double *__restrict__ iv, PairHit &h) {
  if ((kRot && e.rot) || !q.r.fast) return bwd_pair<kRot, kDepth, true>(sc, e, q, h);
  const RayF &r = q.r;
  const double ts = -fma(e.o[2], r.d[2], fma(e.o[1], r.d[1], e.o[0] * r.d[0]));
  double u0 = r.tn0 - ts, u1 = INFINITY;
  float qf[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double qk = fma(ts, r.d[k], e.o[k]);
    const double ik = iv[k];
    const double hk = e.half * fabs(ik);
    u0 = fmax(u0, fma(-qk, ik, -hk));
    u1 = fmin(u1, fma(-qk, ik, hk));
    qf[k] = (float)qk;
  }
  if (!(u1 > u0 + 1e-12)) return false;
  h.delta = (float)(u1 - u0);
  const float um = (float)(0.5 * (u0 + u1));
  h.dq = kDepth ? (float)(ts - q.D) + um : 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) h.x[k] = __fmaf_rn(um, r.df[k], qf[k]) * e.inv_hf;
  if (kRot) {
#pragma unroll
    for (int k = 0; k < 4; ++k) h.gam[k] = r.gam[k];
  }
  return true;
}

// One included hit of pixel q against staged entry e, visited back to front
// (its pair part h from bwd_pair): adds its 27 gradient components to g.
template <bool kRot, bool sdf, bool kDepth = true>
__device__ __forceinline__ void bwd_segment(const EntryF &e, BwdPix &q, const PairHit &h, float g[32]) {
  const float delta = h.delta, dq = h.dq;
  const float *x = h.x;
  const float *gam = kRot ? h.gam : q.r.gam;

  // fp32 fields (scene.py:229-284)
  const VoxPrm &p = e.p;
  const float s = __fmaf_rn(p.ws[2], x[2], __fmaf_rn(p.ws[1], x[1], __fmaf_rn(p.ws[0], x[0], p.ws[3])));
  const float a = e.a, inv_b = e.inv_b;
  const float ha = 0.5f * a;
  float ee = 0.f, sigma;
  if (sdf) {
    // a/2 (1 + sign(s)(1 - e)): a - a/2 e for s > 0, a/2 e otherwise (e = 1 at s = 0)
    ee = fast_exp(-fabsf(s) * inv_b);
    const float he = ha * ee;
    sigma = s > 0.f ? a - he : he;
  } else {
    sigma = fast_exp(s);
  }
  constexpr float kYClamp = 27.631021115928547f;  // alpha >= 1 - 1e-12 (scene.py:32)
  const float yr = sigma * delta;
  const float om = fast_exp(-yr);                 // exp(-sigma delta), unclamped (backward.py:66)
  const bool clamped = yr > kYClamp;
  const float y = clamped ? kYClamp : yr;         // -log1p(-clip(alpha))
  const float alpha = clamped ? 1.f : -expm1_neg(-yr);
  const float omc = clamped ? 1e-12f : om;       // 1 - alpha as the reference clamps it
  // Y before this hit = Y after it - y (compensated)
  {
    const float Yt = q.Yh - y;
    q.Yc += fabsf(q.Yh) >= y ? (q.Yh - Yt) - y : (-y - Yt) + q.Yh;
    q.Yh = Yt;
  }
  const float T = fast_exp(-(q.Yh + q.Yc));
  // colour and its complement without cancellation: c = 1 / (1 + E), 1 - c = E c (E = e^-z)
  float col[3], omcol[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float z = __fmaf_rn(p.wc[3 * i + 2], x[2], __fmaf_rn(p.wc[3 * i + 1], x[1], p.wc[3 * i] * x[0]));
    z = __fmaf_rn(p.wsh[4 * i + 0], gam[0], z);
    z = __fmaf_rn(p.wsh[4 * i + 1], gam[1], z);
    z = __fmaf_rn(p.wsh[4 * i + 2], gam[2], z);
    z = __fmaf_rn(p.wsh[4 * i + 3], gam[3], z);
    const float E = fast_exp(-z);
    col[i] = fast_rcp(1.0f + E);
    omcol[i] = E * col[i];
  }
  const float w = T * alpha;
  // A = dC . c + dD (t_mid - D) / ws (backward.py:52-59)
  const float A = __fmaf_rn(q.dC[2], col[2], __fmaf_rn(q.dC[1], col[1], kDepth ? __fmaf_rn(q.dC[0], col[0], q.dws * dq)
                                                                             : q.dC[0] * col[0]));
  const float g_alpha = __fmaf_rn(A, T, -(q.S + q.tail) * fast_rcp(omc));  // backward.py:62-64
  q.S = __fmaf_rn(A, w, q.S);
  const float g_sigma = g_alpha * delta * om;                               // :66
  float ds, ga, gb;
  if (sdf) {
    const float k2e = ha * inv_b * ee;
    ds = (s == 0.f) ? 0.f : g_sigma * k2e;  // :92
    ga = g_sigma * sigma;                    // :94
    gb = -g_sigma * k2e * s;                 // :95
  } else {
    ds = g_sigma * sigma;
    ga = 0.f;
    gb = 0.f;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = __fmaf_rn(ds, x[k], g[k]);
  g[3] += ds;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float gz = q.dC[i] * (w * col[i]) * omcol[i];  // dC w c (1 - c)  :69-70
#pragma unroll
    for (int k = 0; k < 3; ++k) g[4 + 3 * i + k] = __fmaf_rn(gz, x[k], g[4 + 3 * i + k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) g[13 + 4 * i + k] = __fmaf_rn(gz, gam[k], g[13 + 4 * i + k]);
  }
  g[25] += ga;
  g[26] += gb;
}

// ---------------------------------------------------------------------------
// Certified mixed-precision forward (default, fast mode).
//
// Same pair test and fields as the mixed-precision backward (closest-approach
// fp32 geometry, fp32 fields).  The reference's transmittance is
// T = exp(cumsum(log1p(-alpha))) = exp(-Y), Y = sum of y = min(sigma delta,
// ln 1e12) (render_raster.py:258-266, scene.py:32); the kernel accumulates
// Y in fp64 from fp32 y together with a bound EY on |Y - Y_exact|, so every
// discrete decision of the reference is either certified or the pixel is
// flagged:
//   * hit / miss, t1 > t0 + 1e-12 (render_raster.py:241): a pair within its
//     fp32 error of grazing contributes y <= sigma 4 dd either way, which is
//     added to EY (SDF density, sigma <= a) or flags the pixel (raw density);
//   * inclusion, T_before > 1 - stop_threshold (:267), i.e.
//     Y < ln(1 / keep): certified outside +-(2 EY + 1e-9);
//   * depth validity, sum w > 0.5 (:299); sum w = 1 - T_final (the weights
//     telescope), i.e. Y_final > ln 2: certified outside the same band.
// Flagged pixels are marked with opacity = NaN and recomputed by
// k_composite_redo in fp64 reference order, so every pixel's hit set, stop
// index and NaN-depth mask equal the fp64 path's; values differ by fp32
// rounding (T = exp(-Y) to ~5e-7 relative).
//
// Error model (2^-24 = u): the u-parameters (+-h |1/d| - q / d) of a pair
// carry |du| <= u (h + 2|q_k| + 3 |u_k|) |1/d_k| <= dd = 8 u h max|1/d|
// (|q_k|, |u_k| <= sqrt(3) h wherever a hit is possible), so
// |d delta| <= 2 dd and |dx| <= dd / h + 6 u; the SDF then carries
// |ds| <= |w_s|_1 (|dx| + 4 u), sigma a relative error
// rel <= |ds| / b + 3e-7 (1 + |s| / b) + 2.4e-7 (MUFU ex2 and roundings),
// and |dy| <= y (rel + 2 u) + sigma 2 dd.
#ifndef SALF_PREFETCH
#define SALF_PREFETCH 1
#endif
// Prefetch the voxel records of the next chunk's entries into L2 while the
// current chunk is processed (thread j < cn of the CTA takes entry j).
__device__ __forceinline__ void prefetch_next(const salf_scene_t &sc, const int32_t *__restrict__ entries,
                                              int64_t next, int64_t end, int chunk) {
#if SALF_PREFETCH
  if (threadIdx.x < chunk && next + threadIdx.x < end) {
    const int64_t v = __ldg(entries + next + threadIdx.x);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.geo + 4 * v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.aux + 4 * v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.prm + v * SALF_PRM_STRIDE));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.prm + v * SALF_PRM_STRIDE + 24));
  }
#else
  (void)sc; (void)entries; (void)next; (void)end; (void)chunk;
#endif
}

// Split form: the entry index is loaded before the current chunk is staged
// (its latency hides behind the staging) and the prefetches issued after.
__device__ __forceinline__ int32_t prefetch_index(const int32_t *__restrict__ entries, int64_t first, int64_t lo,
                                                  int64_t hi, int chunk) {
#if SALF_PREFETCH
  const int64_t j = first + threadIdx.x;
  return (threadIdx.x < chunk && j >= lo && j < hi) ? __ldg(entries + j) : -1;
#else
  (void)entries; (void)first; (void)lo; (void)hi; (void)chunk;
  return -1;
#endif
}
__device__ __forceinline__ void prefetch_voxel(const salf_scene_t &sc, int32_t v) {
#if SALF_PREFETCH
  if (v >= 0) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.geo + 4 * (int64_t)v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.aux + 4 * (int64_t)v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.prm + (int64_t)v * SALF_PRM_STRIDE));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.prm + (int64_t)v * SALF_PRM_STRIDE + 24));
  }
#else
  (void)sc; (void)v;
#endif
}

// Same for the backward's back-to-front walk: the chunk before `prev` + chunk.
__device__ __forceinline__ void prefetch_prev(const salf_scene_t &sc, const int32_t *__restrict__ entries,
                                              int64_t prev, int64_t beg, int chunk) {
#if SALF_PREFETCH
  const int64_t j = prev + threadIdx.x;
  if (threadIdx.x < chunk && j >= beg) {
    const int64_t v = __ldg(entries + j);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.geo + 4 * v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.aux + 4 * v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.prm + v * SALF_PRM_STRIDE));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(sc.prm + v * SALF_PRM_STRIDE + 24));
  }
#else
  (void)sc; (void)entries; (void)prev; (void)beg; (void)chunk;
#endif
}

#ifndef SALF_FLAGMASK
#define SALF_FLAGMASK 7  // diagnostics: bit 0 hit, bit 1 inclusion, bit 2 depth certification
#endif
constexpr float kU24 = 5.9604645e-8f;  // 2^-24

// The reference's pair test in fp64 and in its own order (ray_box_range,
// octree.py:184-194, on o = camera - centre; t0 = max(t_in, t_near, 0); hit iff
// t1 > t0 + 1e-12, render_raster.py:239-241) for a pixel ray without zero
// components: what the certified forward falls back to for a chord its fp32
// bound cannot place on either side of zero.
__device__ __forceinline__ bool pair_hit_ref64(const RayF &r, const EntryF &e, double &t0, double &t1) {
  double ti = 0.0, to = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double inv = 1.0 / r.d[k];
    const double ta = __dmul_rn(__dsub_rn(-e.half, e.o[k]), inv), tb = __dmul_rn(__dsub_rn(e.half, e.o[k]), inv);
    const double nk = npmin(ta, tb), fk = npmax(ta, tb);
    ti = k ? npmax(ti, nk) : nk;
    to = k ? npmin(to, fk) : fk;
  }
  t0 = npmax(ti, r.tn0);  // max(max(t_in, t_near), 0) with r.tn0 = max(t_near, 0)
  t1 = to;
  return t1 > __dadd_rn(t0, 1e-12);
}

#ifndef SALF_FWDF_MINB
#define SALF_FWDF_MINB 3
#endif
#ifndef SALF_FWD_PARTS
#define SALF_FWD_PARTS 2  // 16 x 16 tiles: CTAs per tile (1: one 8-warp CTA, 2: 16 x 8 halves, 4: 16 x 4)
#endif
template <bool kRot, bool sdf>
__global__ void __launch_bounds__(256, SALF_FWDF_MINB) k_composite_fast(salf_scene_t sc, PinholeDev c, salf_raster_opts_t opt,
                                                        const int64_t *__restrict__ offsets,
                                                        const int32_t *__restrict__ entries,
                                                        float *__restrict__ out_rgb, float *__restrict__ out_op,
                                                        float *__restrict__ out_depth, double *__restrict__ saved,
                                                        const int32_t *__restrict__ vrange,
                                                        const int32_t *__restrict__ tile_order,
                                                        uint32_t *__restrict__ hitbits, int parts) {
  static_assert(kChunk == 64, "hit words: two 32-entry words per staged chunk");
  __shared__ EntryF sm[kChunk];
  // heaviest tiles first (tile_order: tiles by list length, descending) -> no ragged last wave
  // parts == 2 (16 x 16 tiles): two 4-warp CTAs per tile, one per 16 x 8 half (fewer warps meet
  // at each chunk barrier); parts == 1: one CTA per tile
  const int tslot = (int)blockIdx.x / parts, part = (int)blockIdx.x % parts;
  const int tile_id = tile_order ? __ldg(tile_order + tslot) : tslot;
  const int tx = tile_id % c.tiles_x, ty = tile_id / c.tiles_x;
  // 16 x 16 tiles: warp w shades the 8 x 4 pixel block (w & 1, w >> 1) of the tile, so the
  // per-entry footprint test below culls on columns as well as rows; other tile sizes: rows
  const int lane = threadIdx.x & 31, wid = part * ((int)blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool blocks = c.tile == 16;
  const int lx = blocks ? (wid & 1) * 8 + (lane & 7) : threadIdx.x % c.tile;
  const int ly = blocks ? (wid >> 1) * 4 + (lane >> 3) : threadIdx.x / c.tile;
  const int pslot = ly * c.tile + lx;  // pixel slot of the hit words (the backward's slot order)
  const int px = tx * c.tile + lx, py = ty * c.tile + ly;
  const bool inside = px < c.width && py < c.height && threadIdx.x < c.tile * c.tile;
  const int64_t beg = offsets[tile_id], end = offsets[tile_id + 1];
  const double y_stop_d = -log(1.0 - opt.stop_threshold);  // included iff Y_before < y_stop
  const float y_stop = (float)y_stop_d, y_stop_err = (float)fabs(y_stop_d - (double)y_stop);
  constexpr double kLn2 = 0.6931471805599453;             // sum w > 0.5 iff Y_final > ln 2
  constexpr float kYClamp = 27.631021115928547f;           // -ln(1 - kAlphaMax)

  RayF r;
  float pdd = 0.f, pdd0 = 0.f;  // dd = pdd h + pdd0 for this pixel
  if (inside) {
    PixelRay pr;
    pixel_ray(c, px, py, pr);
    rayf_from_dir(pr.d, pr.t_near, r);
    const float im = fmaxf(fabsf(r.inv[0]), fmaxf(fabsf(r.inv[1]), fabsf(r.inv[2])));
    pdd = 12.f * kU24 * im;
    pdd0 = 2e-12f * im;
  }
  // Y = Yh + Yc: compensated (Neumaier) fp32 sum, |error| <= 2^-23 Y + n 2^-46 Y
  float T = 1.f, acc_c[3] = {0.f, 0.f, 0.f}, acc_w = 0.f, acc_wt = 0.f, EY = 0.f, Yh = 0.f, Yc = 0.f;
  bool alive = inside, flag = false;
  int n_stop = (int)(end - beg), n_inc = 0;
  const int nthreads = blockDim.x;
  // pixel rows / columns this warp covers (for the per-entry footprint test)
  int wr0, wr1, wc0, wc1;
  if (blocks) {
    wr0 = ty * 16 + (wid >> 1) * 4;
    wr1 = wr0 + 3;
    wc0 = tx * 16 + (wid & 1) * 8;
    wc1 = wc0 + 7;
  } else {
    const int wfirst = threadIdx.x & ~31, wlast = min(wfirst + 31, c.tile * c.tile - 1);
    wr0 = ty * c.tile + wfirst / c.tile;
    wr1 = ty * c.tile + wlast / c.tile;
    wc0 = tx * c.tile;
    wc1 = wc0 + c.tile - 1;
  }

  const int64_t hb_base = hit_word_base(beg, tile_id);
  for (int64_t base = beg; base < end; base += kChunk) {
    const int cn = (int)min((int64_t)kChunk, end - base);
    const int32_t pf = prefetch_index(entries, base + kChunk, beg, end, kChunk);
    __syncthreads();
    for (int j = threadIdx.x; j < cn; j += nthreads) stage_entry_f<kRot>(sc, c, entries[base + j], sm[j], vrange);
    __syncthreads();
    prefetch_voxel(sc, pf);
    // entries whose footprint meets this warp's pixel rows and columns: one test per entry per
    // warp (lane l tests entries l and l + 32), the loop below visits only those
    uint64_t wmask;
    {
      bool f0 = false, f1 = false;
      if (lane < cn) {
        const EntryF &e = sm[lane];
        f0 = !(e.vhi < wr0 || e.vlo > wr1 || e.uhi < wc0 || e.ulo > wc1);
      }
      if (lane + 32 < cn) {
        const EntryF &e = sm[lane + 32];
        f1 = !(e.vhi < wr0 || e.vlo > wr1 || e.uhi < wc0 || e.ulo > wc1);
      }
      wmask = ((uint64_t)__ballot_sync(0xffffffffu, f1) << 32) | __ballot_sync(0xffffffffu, f0);
    }
    if (alive) {
      // the chunk's two 32-entry halves (32-bit bit scans and masks), each ending with its hit
      // word (bit jj: list position base - beg + 32 half + jj is an included hit).  A pixel that
      // stops in the first half never has its second word read (the backward reads words below
      // its stop index only).
      for (int half = 0; half < 2 && alive && (half == 0 || cn > 32); ++half) {
      uint32_t hb = 0u;
      for (uint32_t m = half ? (uint32_t)(wmask >> 32) : (uint32_t)wmask; m; m &= m - 1) {
        const int jj = __ffs(m) - 1, j = jj + 32 * half;
        const EntryF &e = sm[j];
        const RayF *ray = &r;
        RayF rr;
        if (kRot && e.rot) {  // the pixel ray in the voxel's frame (render_raster.py:191-196)
          const double *R = sc.rot + 9 * (int64_t)e.vid;
          double d2[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) d2[i] = R[i] * r.d[0] + R[3 + i] * r.d[1] + R[6 + i] * r.d[2];
          rayf_from_dir(d2, r.tn0, rr);
          ray = &rr;
        }
        float qv[3], u0, u1, ts;
        const bool hit = pair_hit_f(*ray, e, qv, u0, u1, ts);
        const float dd = __fmaf_rn(pdd, e.hf, pdd0);
        if (!hit) {
          // A near-grazing miss may be an fp64 hit with y <= sigma 4 dd <= a 4 dd (SDF: sigma <= a):
          // widen the band instead of flagging; raw density has no such bound.  (Near-grazing hits
          // are covered by the 2 sigma dd term of |dy|.)
          if ((SALF_FLAGMASK & 1) && ray->fast && u1 - u0 > -2.f * dd) {
            if (sdf) EY = __fmaf_rn(4.f * e.a, dd, EY);
            else flag = true;
          }
          continue;
        }
        float delta = u1 - u0, um = 0.5f * (u0 + u1);
        // a chord within its fp32 error of zero may be an fp64 miss: this pair is decided in fp64
        // in the reference's order (render_raster.py:239-241) -- rare, so no pixel-wide redo
        if ((SALF_FLAGMASK & 1) && u1 - u0 <= 2.f * dd && ray->fast &&
            u1 - u0 <= chord_err(ray->inv, e.hf, qv, ray->tn0f - ts, u0, u1, fabsf(ts) + ray->tn0f)) {
          double t0d, t1d;
          if (!pair_hit_ref64(*ray, e, t0d, t1d)) continue;
          delta = (float)(t1d - t0d);
          um = (float)(0.5 * (t0d + t1d) - (double)ts);
        }
        // inclusion of this hit: Y_before < y_stop (certified outside the band)
        const float Ys = Yh + Yc;
        const float gap = y_stop - Ys;
        if ((SALF_FLAGMASK & 2) && fabsf(gap) <= __fmaf_rn(2.f, EY, __fmaf_rn(4.f * kU24, Ys, y_stop_err + 1e-9f)))
          flag = true;
        if (!(gap > 0.f)) {  // stop: every later segment is excluded
          alive = false;
          n_stop = (int)(base - beg) + j;
          break;
        }
        hb |= 1u << jj;
        float x[3];
#if SALF_PAIR_PACK
        {
          const float2 x01 = __fmul2_rn(__ffma2_rn(make_float2(um, um), make_float2(ray->df[0], ray->df[1]),
                                                   make_float2(qv[0], qv[1])),
                                        make_float2(e.inv_hf, e.inv_hf));
          x[0] = x01.x;
          x[1] = x01.y;
          x[2] = __fmaf_rn(um, ray->df[2], qv[2]) * e.inv_hf;
        }
#else
#pragma unroll
        for (int k = 0; k < 3; ++k) x[k] = __fmaf_rn(um, ray->df[k], qv[k]) * e.inv_hf;
#endif
        const VoxPrm &p = e.p;
        const float s = __fmaf_rn(p.ws[2], x[2], __fmaf_rn(p.ws[1], x[1], __fmaf_rn(p.ws[0], x[0], p.ws[3])));
        const float ds_abs = e.wn * (__fmaf_rn(pdd0, e.inv_hf, pdd) + 10.f * kU24);
        float sigma, rel;
        if (sdf) {
          const float sb = fabsf(s) * e.inv_b;
          const float he = 0.5f * e.a * fast_exp(-sb);
          sigma = s > 0.f ? e.a - he : he;
          rel = __fmaf_rn(ds_abs, e.inv_b, __fmaf_rn(3e-7f, sb, 5.4e-7f));
        } else {
          sigma = fast_exp(s);
          rel = ds_abs + __fmaf_rn(3e-7f, fabsf(s), 5.4e-7f);
        }
        const float y = fminf(sigma * delta, kYClamp);  // -log1p(-clip(alpha))
        const float alpha = y >= kYClamp ? 1.f : -expm1_neg(-y);
        float col[3];
        eval_color32g(p, x, ray->gam, col);
        const float w = T * alpha;
#if SALF_PAIR_PACK
        {
          const float2 a01 = __ffma2_rn(make_float2(w, w), make_float2(col[0], col[1]), make_float2(acc_c[0], acc_c[1]));
          acc_c[0] = a01.x;
          acc_c[1] = a01.y;
          acc_c[2] = __fmaf_rn(w, col[2], acc_c[2]);
        }
#else
#pragma unroll
        for (int k = 0; k < 3; ++k) acc_c[k] = __fmaf_rn(w, col[k], acc_c[k]);
#endif
        acc_w += w;
        acc_wt = __fmaf_rn(w, ts + um, acc_wt);
        EY += __fmaf_rn(y, rel + 2.f * kU24, 2.f * sigma * dd);
        const float Yt = Yh + y;  // Neumaier: Yc collects the rounding of every addition
        Yc += fabsf(Yh) >= y ? (Yh - Yt) + y : (y - Yt) + Yh;
        Yh = Yt;
        T = fast_exp(-(Yh + Yc));
        ++n_inc;
      }
      if (hitbits) hitbits[hb_base + (int64_t)(((base - beg) >> 5) + half) * kHitSlots + pslot] = hb;
      }
    }
    if (!__syncthreads_or(alive)) break;
  }
  if (!inside) return;
  const double Y = (double)Yh + (double)Yc;
  if ((SALF_FLAGMASK & 4) && fabs(Y - kLn2) <= (double)__fmaf_rn(2.f, EY, __fmaf_rn(4.f * kU24, (float)Y, 1e-9f)))
    flag = true;
  const bool valid = Y > kLn2;  // sum w = 1 - T_final > 0.5
  const double wsum = -expm1(-Y);  // 1 - T_final, consistent with `valid`
  const int64_t pix = (int64_t)py * c.width + px;
#pragma unroll
  for (int k = 0; k < 3; ++k) out_rgb[pix * 3 + k] = __fmaf_rn(T, (float)opt.background[k], acc_c[k]);
  out_op[pix] = flag ? NAN : (float)(-expm1(-Y));  // 1 - T without cancellation near T = 1
  out_depth[pix] = valid ? (float)(acc_wt / (double)acc_w) : NAN;
  if (saved) {
    double *sv = saved + pix * SALF_SAVED_STRIDE;
    sv[0] = acc_c[0]; sv[1] = acc_c[1]; sv[2] = acc_c[2];
    sv[3] = valid ? fmax(wsum, 0.5000000001) : fmin(wsum, 0.5);
    sv[4] = (double)acc_wt * (sv[3] / (double)acc_w);  // keeps D = acc_wt / acc_w
    sv[5] = T; sv[6] = (double)n_stop; sv[7] = (double)n_inc;
  }
}

// fp64 reference-order recomputation of the pixels k_composite_fast flagged
// (opacity NaN).  One warp per 32 pixels of the image; for each flagged
// pixel of its slice the whole warp cooperates: lane k stages and shades
// entry base + k (fp64, the exact kernel's code), then the hits are
// composited in list order from lane-broadcast values, so the arithmetic is
// the sequential fp64 kernel's (same operations, same order).
template <bool kRot>
__global__ void __launch_bounds__(128) k_composite_redo(salf_scene_t sc, PinholeDev c, salf_raster_opts_t opt,
                                                       const int64_t *__restrict__ offsets,
                                                       const int32_t *__restrict__ entries,
                                                       float *__restrict__ out_rgb, float *__restrict__ out_op,
                                                       float *__restrict__ out_depth, double *__restrict__ saved,
                                                       uint32_t *__restrict__ hitbits) {
  const int64_t npx = (int64_t)c.width * c.height;
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(int64_t)31;
  const int lane = threadIdx.x & 31;
  if (p0 >= npx) return;
  const int64_t mine = p0 + lane;
  const float op = mine < npx ? out_op[mine] : 0.f;
  unsigned todo = __ballot_sync(0xffffffffu, op != op);
  const double keep = 1.0 - opt.stop_threshold;
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int64_t pix = p0 + src;
    const int px = (int)(pix % c.width), py = (int)(pix / c.width);
    const int tile_id = (py / c.tile) * c.tiles_x + px / c.tile;
    const int64_t beg = offsets[tile_id], end = offsets[tile_id + 1];
    PixelRay r;
    pixel_ray(c, px, py, r);
    double acc_w = 0.0, acc_wt = 0.0, T = 1.0;
    float acc_c[3] = {0.f, 0.f, 0.f};
    int64_t n_stop = end - beg;
    int n_inc = 0;
    bool alive = true;
    for (int64_t base = beg; base < end && alive; base += 32) {
      const int64_t j = base + lane;
      SegVals sv;
      bool hit = false;
      if (j < end) {
        Entry e;
        stage_entry<kRot>(sc, c, entries[j], e);
        hit = hit_and_shade<false, kRot>(sc, r, e, sv);
      }
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      const unsigned all_hits = hits;
      while (hits) {
        const int k = __ffs(hits) - 1;
        hits &= hits - 1;
        const double alpha = __shfl_sync(0xffffffffu, sv.alpha, k);
        const double om = __shfl_sync(0xffffffffu, sv.om, k);
        const double tm = __shfl_sync(0xffffffffu, sv.tm, k);
        float cf[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) cf[q] = __shfl_sync(0xffffffffu, sv.cf[q], k);
        if (!(T > keep)) {  // included iff T_before > keep (render_raster.py:267)
          n_stop = base - beg + k;
          alive = false;
          break;
        }
        const double w = __dmul_rn(T, alpha);
        const float wf = (float)w;
#pragma unroll
        for (int q = 0; q < 3; ++q) acc_c[q] = __fmaf_rn(wf, cf[q], acc_c[q]);
        acc_w = __dadd_rn(acc_w, w);
        acc_wt = __dadd_rn(acc_wt, __dmul_rn(w, tm));
        T = __dmul_rn(T, om);
        ++n_inc;
      }
      if (hitbits && lane == 0) {  // included hits of this 32-entry word (positions before the stop)
        const int ks = alive ? 32 : (int)(n_stop - (base - beg));
        const unsigned inc = ks >= 32 ? all_hits : (all_hits & ((1u << ks) - 1u));
        const int pslot = (py % c.tile) * c.tile + px % c.tile;
        hitbits[hit_word_base(beg, tile_id) + (int64_t)((base - beg) >> 5) * kHitSlots + pslot] = inc;
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 3; ++q) out_rgb[pix * 3 + q] = (float)__dadd_rn(acc_c[q], __dmul_rn(T, opt.background[q]));
      out_op[pix] = (float)__dsub_rn(1.0, T);
      out_depth[pix] = acc_w > kDepthWeightMin ? (float)__ddiv_rn(acc_wt, acc_w) : NAN;
      if (saved) {
        double *s = saved + pix * SALF_SAVED_STRIDE;
        s[0] = acc_c[0]; s[1] = acc_c[1]; s[2] = acc_c[2];
        s[3] = acc_w; s[4] = acc_wt; s[5] = T; s[6] = (double)n_stop; s[7] = (double)n_inc;
      }
    }
  }
}

#ifndef SALF_BWD_ROWCULL
#define SALF_BWD_ROWCULL 0  // per-warp footprint-row culling in the backward: measured slower (5.57 vs 5.42 ms)
#endif
#ifndef SALF_BWD_SMEMRED
#define SALF_BWD_SMEMRED 1  // warp reduction by a shared-memory transpose (0: shuffles; measured slower)
#endif
#ifndef SALF_BWD_ALL64
#define SALF_BWD_ALL64 false  // A/B: every fp32 hit's chord re-derived in fp64 (no refinement branch)
#endif
#ifndef SALF_BWD_NP
#define SALF_BWD_NP 2  // pixels per thread
#endif
#ifndef SALF_BWDF_MINB
#define SALF_BWDF_MINB 5  // resident 4-warp CTAs per SM the register budget is sized for (2-warp CTAs: twice as many)
#endif

template <bool kRot, int NP, bool sdf, bool kDepth = true>
__global__ void __launch_bounds__(256 / NP, SALF_BWDF_MINB) k_backward_fast(
    salf_scene_t sc, PinholeDev c, salf_raster_opts_t opt, const int64_t *__restrict__ offsets,
    const int32_t *__restrict__ entries, const double *__restrict__ saved, const double *__restrict__ d_rgb,
    const double *__restrict__ d_depth, double *__restrict__ grad, float *__restrict__ partial,
    const int32_t *__restrict__ vrange, const int32_t *__restrict__ tile_order) {
  __shared__ EntryF sm[kChunkB];
  __shared__ float red[kChunkB][8 / NP][kGradStride];
#if SALF_BWD_SMEMRED
  __shared__ __align__(16) float xp[8 / NP][32][28];
#endif
  __shared__ int s_max;
  const int tile_id = tile_order ? __ldg(tile_order + blockIdx.x) : (int)blockIdx.x;
  const int tx = tile_id % c.tiles_x, ty = tile_id / c.tiles_x;
  const int nthreads = blockDim.x;
  const int npix = c.tile * c.tile;
  const int64_t beg = offsets[tile_id], end = offsets[tile_id + 1];
  (void)end;

  BwdPix q[NP];
  bool in[NP];
  if (threadIdx.x == 0) s_max = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int li = threadIdx.x + k * nthreads;  // pixel slot in the tile
    const int px = tx * c.tile + li % c.tile, py = ty * c.tile + li / c.tile;
    in[k] = li < npix && px < c.width && py < c.height;
    q[k].n_stop = 0;
    if (in[k]) bwd_pixel_init(c, opt, px, py, saved, d_rgb, d_depth, q[k]);
  }
  __syncthreads();
  int my_max = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) my_max = max(my_max, q[k].n_stop);
  if (my_max > 0) atomicMax(&s_max, my_max);
  __syncthreads();
  const int64_t lim = beg + (int64_t)s_max;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = nthreads >> 5;
  int wr0[NP], wr1[NP];  // pixel rows of this warp's slot-k pixels (footprint test)
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int f = (threadIdx.x & ~31) + k * nthreads, l = min(f + 31, npix - 1);
    wr0[k] = ty * c.tile + f / c.tile;
    wr1[k] = f < npix ? ty * c.tile + l / c.tile : -1;
  }
  // back to front: chunks from the last one any pixel of the tile includes down to the first
  for (int64_t base = beg + ((lim - beg - 1) / kChunkB) * kChunkB; base >= beg && lim > beg; base -= kChunkB) {
    const int cn = (int)min((int64_t)kChunkB, lim - base);
    __syncthreads();
    for (int j = threadIdx.x; j < cn; j += nthreads) stage_entry_f<kRot>(sc, c, entries[base + j], sm[j], vrange);
    __syncthreads();
    prefetch_prev(sc, entries, base - kChunkB, beg, kChunkB);
    const int jb = (int)(base - beg);
    for (int j = cn - 1; j >= 0; --j) {
      const EntryF &e = sm[j];
      bool rows_hit[NP];
      bool any_rows = false;
#pragma unroll
      for (int k = 0; k < NP; ++k) {  // footprint vs this warp's pixel rows of slot k (warp-uniform)
        rows_hit[k] = !SALF_BWD_ROWCULL || !(e.vhi < wr0[k] || e.vlo > wr1[k]);
        any_rows |= rows_hit[k];
      }
      if (SALF_BWD_ROWCULL && !any_rows) {
        if (lane < kGradStride) red[j][warp][lane] = 0.f;
        continue;
      }
      PairHit ph[NP];
      bool hit[NP];
      bool act = false;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        hit[k] = rows_hit[k] && jb + j < q[k].n_stop && bwd_pair<kRot, kDepth, SALF_BWD_ALL64>(sc, e, q[k], ph[k]);
        act |= hit[k];
      }
      float g[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) g[k] = 0.f;
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (hit[k]) bwd_segment<kRot, sdf, kDepth>(e, q[k], ph[k], g);
      float tot = 0.0f;
#if SALF_BWD_SMEMRED
      // transpose through shared memory: 7 x STS.128 per lane, lane k sums column k
      if (__ballot_sync(0xffffffffu, act)) {
        float4 *row = reinterpret_cast<float4 *>(&xp[warp][lane][0]);
#pragma unroll
        for (int m = 0; m < 7; ++m) row[m] = make_float4(g[4 * m], g[4 * m + 1], g[4 * m + 2], g[4 * m + 3]);
        __syncwarp();
        if (lane < kGradStride) {
          // four independent partial sums: a 32-long serial FADD chain would
          // leave the warp waiting on the add latency
          float t0 = xp[warp][0][lane], t1 = xp[warp][1][lane], t2 = xp[warp][2][lane], t3 = xp[warp][3][lane];
#pragma unroll
          for (int rr = 4; rr < 32; rr += 4) {
            t0 += xp[warp][rr][lane];
            t1 += xp[warp][rr + 1][lane];
            t2 += xp[warp][rr + 2][lane];
            t3 += xp[warp][rr + 3][lane];
          }
          tot = (t0 + t1) + (t2 + t3);
        }
        __syncwarp();
      }
#else
      if (__ballot_sync(0xffffffffu, act)) tot = warp_transpose_reduce(g);
#endif
      if (lane < kGradStride) red[j][warp][lane] = tot;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < cn * kGradStride; t += nthreads) {
      const int j = t / kGradStride, k = t - j * kGradStride;
      float sum = 0.0f;
      for (int w = 0; w < nwarps; ++w) sum += red[j][w][k];
      if (partial) partial[(base + j) * kGradStride + k] = sum;  // deterministic mode: one row per instance
      else if (sum != 0.0f) atomicAdd(grad + sm[j].vid * kGradStride + k, (double)sum);
    }
  }
}

// ---------------------------------------------------------------------------
// Backward over the forward's hit words (default mode).  Two pixels per thread
// (rows ly and ly + 8 of the tile) processed TOGETHER in packed fp32x2
// arithmetic (FFMA2 / FMUL2 / FADD2, sm_100): lane .x is the first pixel,
// .y the second.  A pixel without a hit on the entry runs the same chain with
// delta = 0 and x = 0 (y = 0, alpha = 0, w = 0: it adds exact zeros and
// leaves its state unchanged), so one pass shades both pixels -- the scalar
// kernel ran one divergent pass per pixel.  Each packed op is two IEEE
// fp32 ops, so the per-pixel arithmetic is the scalar kernel's.

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 ex2_2(float2 t) {
  float2 y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(t.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(t.y));
  return y;
}
// fast_exp of both lanes (MUFU ex2 of x log2 e, as fast_exp)
__device__ __forceinline__ float2 exp2v(float2 x) { return ex2_2(mul2(x, f2(1.4426950408889634f))); }
__device__ __forceinline__ float2 rcp2(float2 x) {
  float2 y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(x.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(x.y));
  return y;
}
// expm1_neg of both lanes (same polynomial / branchless select)
__device__ __forceinline__ float2 expm1_neg2(float2 x) {
  float2 p = fma2(x, f2(1.0f / 5040.0f), f2(1.0f / 720.0f));
  p = fma2(x, p, f2(1.0f / 120.0f));
  p = fma2(x, p, f2(1.0f / 24.0f));
  p = fma2(x, p, f2(1.0f / 6.0f));
  p = fma2(x, p, f2(0.5f));
  const float2 small = fma2(mul2(x, x), p, x);
  const float2 big = add2(exp2v(x), f2(-1.0f));
  return make_float2(x.x > -0.25f ? small.x : big.x, x.y > -0.25f ? small.y : big.y);
}

#ifndef SALF_BWD_BLOCK
#define SALF_BWD_BLOCK 1  // 8 x 8 pixel block per warp in the hit-word backward (0: 16 x 2 strips)
#endif
#ifndef SALF_BWD_XPCOL
#define SALF_BWD_XPCOL 0  // 1: component-major warp reduction (A/B: 4.61 vs 4.59 ms, kept off)
#endif

constexpr int kXpRows = SALF_BWD_XPCOL ? 27 : 32, kXpCols = SALF_BWD_XPCOL ? 36 : 28;
constexpr size_t kXpBytes = sizeof(float) * 4 * kXpRows * kXpCols;  // 4 warps

#ifndef SALF_BWD_HALF
#define SALF_BWD_HALF 1  // atomic mode: two 2-warp CTAs per tile (0: one 4-warp CTA)
#endif

// per-entry field constants, one float each (the packed ops take them as a
// broadcast .F32 operand): w_s 0..3, w_c 4..12, w_sh 13..24, a 25, 1/b 26,
// a/2 27, (a/2)(1/b) 28
constexpr int kPP = 30;

struct Pix2 {
  RayF r[2];
  double D[2];
  int n_stop[2];
  float2 dC[3], dws, tail, Yh, Yc, S;
  float2 g1, g2, g3;  // SH basis C1 y, C1 z, C1 x per pixel (C0 is a constant)
};

struct Hit2 {
  float2 x[3], delta, dq;
  float2 gm[4];  // kRot: SH basis of the (possibly rotated) ray
};

template <bool kRot, bool sdf, bool kDepth>
__device__ __forceinline__ void bwd_segment2(const float *__restrict__ pp, Pix2 &q, const Hit2 &h, float g[32]) {
  const float2 X0 = h.x[0], X1 = h.x[1], X2 = h.x[2], dl = h.delta;
  const float2 G0 = f2((float)kShC0);
  const float2 G1 = kRot ? h.gm[1] : q.g1, G2 = kRot ? h.gm[2] : q.g2, G3 = kRot ? h.gm[3] : q.g3;
  // fields (scene.py:229-284)
  const float2 s = fma2(f2(pp[2]), X2, fma2(f2(pp[1]), X1, fma2(f2(pp[0]), X0, f2(pp[3]))));
  float2 ee = f2(0.f), sigma;
  if (sdf) {
    const float ib = pp[26];
    ee = exp2v(make_float2(-fabsf(s.x) * ib, -fabsf(s.y) * ib));
    const float2 he = mul2(f2(pp[27]), ee);
    const float2 ahe = add2(f2(pp[25]), neg2(he));
    sigma = make_float2(s.x > 0.f ? ahe.x : he.x, s.y > 0.f ? ahe.y : he.y);
  } else {
    sigma = exp2v(s);
    // an idle lane (delta = 0) must add exact zeros: raw density may overflow to inf
    sigma = make_float2(dl.x > 0.f ? sigma.x : 0.f, dl.y > 0.f ? sigma.y : 0.f);
  }
  constexpr float kYClamp = 27.631021115928547f;  // alpha >= 1 - 1e-12 (scene.py:32)
  const float2 yr = mul2(sigma, dl);
  const float2 nyr = neg2(yr);
  const float2 om = exp2v(nyr);      // exp(-sigma delta), unclamped (backward.py:66)
  const float2 em = expm1_neg2(nyr);
  const bool c0 = yr.x > kYClamp, c1 = yr.y > kYClamp;
  const float2 y = make_float2(c0 ? kYClamp : yr.x, c1 ? kYClamp : yr.y);
  const float2 alpha = make_float2(c0 ? 1.f : -em.x, c1 ? 1.f : -em.y);
  const float2 omc = make_float2(c0 ? 1e-12f : om.x, c1 ? 1e-12f : om.y);
  // Y before this hit = Y after it - y (compensated)
  {
    const float2 Yt = add2(q.Yh, neg2(y));
    const float2 u1 = add2(add2(q.Yh, neg2(Yt)), neg2(y));  // (Yh - Yt) - y
    const float2 u2 = add2(add2(neg2(y), neg2(Yt)), q.Yh);  // (-y - Yt) + Yh
    q.Yc = add2(q.Yc, make_float2(fabsf(q.Yh.x) >= y.x ? u1.x : u2.x, fabsf(q.Yh.y) >= y.y ? u1.y : u2.y));
    q.Yh = Yt;
  }
  const float2 T = exp2v(neg2(add2(q.Yh, q.Yc)));
  // colour and its complement: c = 1 / (1 + E), 1 - c = E c (E = e^-z)
  float2 col[3], omcol[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float2 z = fma2(f2(pp[4 + 3 * i + 2]), X2, fma2(f2(pp[4 + 3 * i + 1]), X1, mul2(f2(pp[4 + 3 * i]), X0)));
    z = fma2(f2(pp[13 + 4 * i + 0]), G0, z);
    z = fma2(f2(pp[13 + 4 * i + 1]), G1, z);
    z = fma2(f2(pp[13 + 4 * i + 2]), G2, z);
    z = fma2(f2(pp[13 + 4 * i + 3]), G3, z);
    const float2 E = exp2v(neg2(z));
    col[i] = rcp2(add2(f2(1.0f), E));
    omcol[i] = mul2(E, col[i]);
  }
  const float2 w = mul2(T, alpha);
  // A = dC . c + dD (t_mid - D) / ws (backward.py:52-59)
  const float2 A = fma2(q.dC[2], col[2], fma2(q.dC[1], col[1], kDepth ? fma2(q.dC[0], col[0], mul2(q.dws, h.dq))
                                                                       : mul2(q.dC[0], col[0])));
  const float2 ga = fma2(A, T, mul2(neg2(add2(q.S, q.tail)), rcp2(omc)));  // backward.py:62-64
  q.S = fma2(A, w, q.S);
  const float2 gs = mul2(mul2(ga, dl), om);  // :66
  float2 ds, gla, glb;
  if (sdf) {
    const float2 k2e = mul2(f2(pp[28]), ee);
    const float2 d = mul2(gs, k2e);
    ds = make_float2(s.x == 0.f ? 0.f : d.x, s.y == 0.f ? 0.f : d.y);  // :92
    gla = mul2(gs, sigma);                                               // :94
    glb = mul2(mul2(neg2(gs), k2e), s);                                  // :95
  } else {
    ds = mul2(gs, sigma);
    gla = f2(0.f);
    glb = f2(0.f);
  }
  const float2 X[3] = {X0, X1, X2};
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = __fmaf_rn(ds.y, X[k].y, __fmaf_rn(ds.x, X[k].x, g[k]));
  g[3] += ds.x + ds.y;
  const float2 Gs[4] = {G0, G1, G2, G3};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float2 gz = mul2(mul2(q.dC[i], mul2(w, col[i])), omcol[i]);  // dC w c (1 - c)  :69-70
#pragma unroll
    for (int k = 0; k < 3; ++k) g[4 + 3 * i + k] = __fmaf_rn(gz.y, X[k].y, __fmaf_rn(gz.x, X[k].x, g[4 + 3 * i + k]));
#pragma unroll
    for (int k = 0; k < 4; ++k)
      g[13 + 4 * i + k] = __fmaf_rn(gz.y, Gs[k].y, __fmaf_rn(gz.x, Gs[k].x, g[13 + 4 * i + k]));
  }
  g[25] += gla.x + gla.y;
  g[26] += glb.x + glb.y;
}

// The known hit's chord (bwd_pair64) written into lane `k` of the packed hit.
template <bool kRot, bool kDepth>
__device__ __forceinline__ bool pair64_into(const salf_scene_t &sc, const EntryF &e, const BwdPix &q,
                                            const double *__restrict__ iv, Hit2 &h, int k) {
  PairHit ph;
  if (!bwd_pair64<kRot, kDepth>(sc, e, q, iv, ph)) return false;
  float *hx0 = k ? &h.x[0].y : &h.x[0].x;
  float *hx1 = k ? &h.x[1].y : &h.x[1].x;
  float *hx2 = k ? &h.x[2].y : &h.x[2].x;
  *hx0 = ph.x[0];
  *hx1 = ph.x[1];
  *hx2 = ph.x[2];
  (k ? h.delta.y : h.delta.x) = ph.delta;
  (k ? h.dq.y : h.dq.x) = ph.dq;
  if (kRot) {
#pragma unroll
    for (int m = 0; m < 4; ++m) (k ? h.gm[m].y : h.gm[m].x) = ph.gam[m];
  }
  return true;
}

// Staged geometry of a hit-word backward entry (the field constants live in spp).
struct EntryG {
  double o[3], half;
  float hf, inv_hf;
  int vid, rot;
};
__device__ __forceinline__ EntryF entry_f(const EntryG &g) {
  EntryF e;  // the fields bwd_pair reads
#pragma unroll
  for (int m = 0; m < 3; ++m) e.o[m] = g.o[m];
  e.half = g.half;
  e.hf = g.hf;
  e.inv_hf = g.inv_hf;
  e.vid = g.vid;
  e.rot = g.rot;
  return e;
}

#ifndef SALF_BWD_RAYSMEM
#define SALF_BWD_RAYSMEM 1  // the pixels' fp64 direction and near plane in shared memory (not registers)
#endif
constexpr int kIvRow = SALF_BWD_RAYSMEM ? 7 : 3;  // doubles per pixel row of s_iv: 1/d (+ d, t_near0)

#ifndef SALF_BWD_PAIR2
#define SALF_BWD_PAIR2 1  // both pixels' fp64 chords as one straight-line block (0: one divergent pass per pixel)
#endif

// bwd_pair64 for BOTH pixels of a thread at once: the two fp64 chord chains
// are independent, so interleaving them halves the exposed DFMA latency of
// the per-pixel passes (which the warp runs back to back whenever any lane
// has each pixel hit -- nearly always).  Rotated voxels and rays with a zero
// component take bwd_pair per pixel.
template <bool kRot, bool kDepth>
__device__ __forceinline__ bool pair64_both(const salf_scene_t &sc, const EntryG &e, const BwdPix bp[2],
                                            const double *__restrict__ iv0, const double *__restrict__ iv1, bool h0,
                                            bool h1, Hit2 &h) {
  const bool gen0 = h0 && ((kRot && e.rot) || !bp[0].r.fast), gen1 = h1 && ((kRot && e.rot) || !bp[1].r.fast);
  const bool f0 = h0 && !gen0, f1 = h1 && !gen1;
  bool act = false;
  if (f0 || f1) {
    const double *ivp[2] = {iv0, iv1};
    double ts[2], u0[2], u1[2];
    float qf[2][3];
#pragma unroll
    for (int l = 0; l < 2; ++l) {
#if SALF_BWD_RAYSMEM
      const double *d = ivp[l] + 3;  // d[0..2], tn0 follow 1/d in the pixel's shared-memory row
      ts[l] = -fma(e.o[2], d[2], fma(e.o[1], d[1], e.o[0] * d[0]));
      u0[l] = d[3] - ts[l];
#else
      const RayF &r = bp[l].r;
      ts[l] = -fma(e.o[2], r.d[2], fma(e.o[1], r.d[1], e.o[0] * r.d[0]));
      u0[l] = r.tn0 - ts[l];
#endif
    }
    // plain compare-selects: every value here is finite (fast rays), so fmax / fmin's NaN
    // handling (several extra instructions per call on sm_100) is not needed
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
      for (int l = 0; l < 2; ++l) {
#if SALF_BWD_RAYSMEM
        const double qk = fma(ts[l], ivp[l][3 + k], e.o[k]);
#else
        const double qk = fma(ts[l], bp[l].r.d[k], e.o[k]);
#endif
        const double ik = ivp[l][k];
        const double hk = e.half * fabs(ik);
        const double n = fma(-qk, ik, -hk), f = fma(-qk, ik, hk);
        u0[l] = n > u0[l] ? n : u0[l];
        u1[l] = (k == 0 || f < u1[l]) ? f : u1[l];
        qf[l][k] = (float)qk;
      }
    }
    const bool ok0 = f0 && u1[0] > u0[0] + 1e-12, ok1 = f1 && u1[1] > u0[1] + 1e-12;
    float um[2], dl[2], dq[2];
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      dl[l] = (float)(u1[l] - u0[l]);
      um[l] = (float)(0.5 * (u0[l] + u1[l]));
      dq[l] = kDepth ? (float)(ts[l] - bp[l].D) + um[l] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float x0 = __fmaf_rn(um[0], bp[0].r.df[k], qf[0][k]) * e.inv_hf;
      const float x1 = __fmaf_rn(um[1], bp[1].r.df[k], qf[1][k]) * e.inv_hf;
      h.x[k] = make_float2(ok0 ? x0 : 0.f, ok1 ? x1 : 0.f);
    }
    h.delta = make_float2(ok0 ? dl[0] : 0.f, ok1 ? dl[1] : 0.f);
    h.dq = make_float2(ok0 ? dq[0] : 0.f, ok1 ? dq[1] : 0.f);
    if (kRot) {
#pragma unroll
      for (int m = 0; m < 4; ++m) h.gm[m] = make_float2(ok0 ? bp[0].r.gam[m] : 0.f, ok1 ? bp[1].r.gam[m] : 0.f);
    }
    act = ok0 || ok1;
  }
#if SALF_BWD_RAYSMEM
  // the general path reads the fp64 ray from its shared-memory row
  if (gen0 || gen1) {
    const double *ivq[2] = {iv0, iv1};
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      if (!(l ? gen1 : gen0)) continue;
      BwdPix b = bp[l];
#pragma unroll
      for (int k = 0; k < 3; ++k) b.r.d[k] = ivq[l][3 + k];
      b.r.tn0 = ivq[l][6];
      act |= pair64_into<kRot, kDepth>(sc, entry_f(e), b, ivq[l], h, l);
    }
  }
#else
  if (gen0) act |= pair64_into<kRot, kDepth>(sc, entry_f(e), bp[0], iv0, h, 0);
  if (gen1) act |= pair64_into<kRot, kDepth>(sc, entry_f(e), bp[1], iv1, h, 1);
#endif
  return act;
}

#ifndef SALF_BWD_WARPATOM
#define SALF_BWD_WARPATOM 1  // each warp adds its entry totals itself (0: block reduction, then one atomic per component)
#endif

// kW warps per CTA: 4 (a whole 16 x 16 tile; the deterministic mode, whose
// instance rows need one CTA per tile) or 2 (half a tile: two CTAs per tile,
// each staging the tile's list for its own 16 x 8 half).  With 2 the warps
// that meet at each chunk barrier are 2, not 4: less time lost to the
// slowest warp of the chunk, for twice the staging work.
template <bool kRot, bool sdf, bool kDepth, int kW>
__global__ void __launch_bounds__(32 * kW, (kRot ? 4 : SALF_BWDF_MINB) * 4 / kW) k_backward_hits(
    salf_scene_t sc, PinholeDev c, salf_raster_opts_t opt, const int64_t *__restrict__ offsets,
    const int32_t *__restrict__ entries, const double *__restrict__ saved, const double *__restrict__ d_rgb,
    const double *__restrict__ d_depth, double *__restrict__ grad, float *__restrict__ partial,
    const int32_t *__restrict__ vrange, const int32_t *__restrict__ tile_order,
    const uint32_t *__restrict__ hitbits) {
  static_assert(kChunkB == 32, "hit words: one 32-entry word per staged chunk");
  static_assert(kW == 2 || kW == 4, "a CTA covers a whole tile or half of one");
  constexpr int kParts = 4 / kW, kThreads = 32 * kW;
  __shared__ EntryG sm[kChunkB];
  __shared__ __align__(16) float spp[kChunkB][kPP];  // per-entry constants (broadcast operands of the packed ops)
  // per-warp entry totals for the CTA's fixed-order sum (deterministic mode: kW == 4 only)
  __shared__ float red[kW == 4 ? kChunkB : 1][kW][kGradStride];
  // warp-reduction scratch in dynamic shared memory (static + this exceed the 48 KB static limit)
  extern __shared__ __align__(16) float xp_dyn[];
  float(*xp)[kXpRows][kXpCols] = reinterpret_cast<float(*)[kXpRows][kXpCols]>(xp_dyn);
  __shared__ double s_iv[2 * kThreads * kIvRow];  // per pixel of this CTA: fp64 1/d (+ d, t_near0)
  __shared__ uint32_t s_wm[kW];     // per warp: entries of the chunk it includes
  __shared__ int s_max;
  const int tslot = (int)blockIdx.x / kParts, part = (int)blockIdx.x % kParts;
  const int tile_id = tile_order ? __ldg(tile_order + tslot) : tslot;
  const int tx = tile_id % c.tiles_x, ty = tile_id / c.tiles_x;
  const int npix = c.tile * c.tile;
  const int64_t beg = offsets[tile_id];
  const int64_t hb = hit_word_base(beg, tile_id);

  Pix2 q;
  BwdPix bp[2];
  bool in[2];
  if (threadIdx.x == 0) s_max = 0;
  // pixel slots of this thread's two pixels: 16 x 16 tiles with SALF_BWD_BLOCK give each warp an
  // 8 x 8 block (lane -> column, two vertically adjacent rows), so a warp's pixels see nearly the
  // same entries (more entries skipped by the whole warp, fewer idle lanes in the packed pass)
  int slot[2];
  const int lane0 = threadIdx.x & 31, wid0 = part * kW + (threadIdx.x >> 5);  // warp within the tile
  const int t0 = part * kThreads + threadIdx.x;                            // thread within the tile
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (SALF_BWD_BLOCK && c.tile == 16)
      slot[k] = ((wid0 >> 1) * 8 + (lane0 >> 3) * 2 + k) * 16 + (wid0 & 1) * 8 + (lane0 & 7);
    else
      slot[k] = t0 + k * 128;
  }
  // s_iv row of each pixel: this CTA's pixel k of thread t
  const int ivrow[2] = {(int)threadIdx.x, kThreads + (int)threadIdx.x};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int li = slot[k];
    const int px = tx * c.tile + li % c.tile, py = ty * c.tile + li / c.tile;
    in[k] = li < npix && px < c.width && py < c.height;
    bp[k].n_stop = 0;
    if (in[k]) {
      bwd_pixel_init(c, opt, px, py, saved, d_rgb, d_depth, bp[k]);
#pragma unroll
      for (int a = 0; a < 3; ++a) s_iv[ivrow[k] * kIvRow + a] = 1.0 / bp[k].r.d[a];
#if SALF_BWD_RAYSMEM
#pragma unroll
      for (int a = 0; a < 3; ++a) s_iv[ivrow[k] * kIvRow + 3 + a] = bp[k].r.d[a];
      s_iv[ivrow[k] * kIvRow + 6] = bp[k].r.tn0;
#endif
    } else {
      // idle slot (outside the image): finite state, never hit (n_stop 0); its lane of the
      // packed chain must stay finite (0 * NaN would poison the warp sums)
#pragma unroll
      for (int a = 0; a < 4; ++a) bp[k].r.gam[a] = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        bp[k].r.df[a] = 0.f;
        bp[k].r.d[a] = 0.0;
      }
      bp[k].dC[0] = bp[k].dC[1] = bp[k].dC[2] = 0.f;
      bp[k].dws = bp[k].tail = bp[k].Yh = bp[k].Yc = bp[k].S = 0.f;
      bp[k].D = 0.0;
    }
  }
  q.dC[0] = make_float2(bp[0].dC[0], bp[1].dC[0]);
  q.dC[1] = make_float2(bp[0].dC[1], bp[1].dC[1]);
  q.dC[2] = make_float2(bp[0].dC[2], bp[1].dC[2]);
  q.dws = make_float2(bp[0].dws, bp[1].dws);
  q.tail = make_float2(bp[0].tail, bp[1].tail);
  q.Yh = make_float2(bp[0].Yh, bp[1].Yh);
  q.Yc = make_float2(bp[0].Yc, bp[1].Yc);
  q.S = f2(0.f);
  q.g1 = make_float2(bp[0].r.gam[1], bp[1].r.gam[1]);
  q.g2 = make_float2(bp[0].r.gam[2], bp[1].r.gam[2]);
  q.g3 = make_float2(bp[0].r.gam[3], bp[1].r.gam[3]);
  __syncthreads();
  const int my_max = max(bp[0].n_stop, bp[1].n_stop);
  if (my_max > 0) atomicMax(&s_max, my_max);
  __syncthreads();
  const int64_t lim = beg + (int64_t)s_max;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // back to front: chunks from the last one any pixel of the tile includes down to the first
  for (int64_t base = beg + ((lim - beg - 1) / kChunkB) * kChunkB; base >= beg && lim > beg; base -= kChunkB) {
    const int cn = (int)min((int64_t)kChunkB, lim - base);
    __syncthreads();
    const int32_t pf = prefetch_index(entries, base - kChunkB, beg, lim, kChunkB);
    for (int j = threadIdx.x; j < cn; j += kThreads) {
      EntryF e;
      stage_entry_f<kRot>(sc, c, entries[base + j], e, nullptr);
      EntryG &eg = sm[j];
#pragma unroll
      for (int m = 0; m < 3; ++m) eg.o[m] = e.o[m];
      eg.half = e.half;
      eg.hf = e.hf;
      eg.inv_hf = e.inv_hf;
      eg.vid = e.vid;
      eg.rot = e.rot;
      float *pp = spp[j];
#pragma unroll
      for (int m = 0; m < 4; ++m) pp[m] = e.p.ws[m];
#pragma unroll
      for (int m = 0; m < 9; ++m) pp[4 + m] = e.p.wc[m];
#pragma unroll
      for (int m = 0; m < 12; ++m) pp[13 + m] = e.p.wsh[m];
      const float ha = 0.5f * e.a;
      pp[25] = e.a;
      pp[26] = e.inv_b;
      pp[27] = ha;
      pp[28] = ha * e.inv_b;
    }
    __syncthreads();
    prefetch_voxel(sc, pf);
    const int jb = (int)(base - beg);
    uint32_t wb0 = 0u, wb1 = 0u;  // hit words of this chunk
    if (in[0] && jb < bp[0].n_stop) wb0 = __ldg(hitbits + hb + (int64_t)(jb >> 5) * kHitSlots + slot[0]);
    if (in[1] && jb < bp[1].n_stop) wb1 = __ldg(hitbits + hb + (int64_t)(jb >> 5) * kHitSlots + slot[1]);
    // entries some pixel of this warp includes, back to front (the block reduction below reads
    // red[j][w] only where warp w's mask has bit j)
    const uint32_t wmask = __reduce_or_sync(0xffffffffu, wb0 | wb1);
    if (lane == 0) s_wm[warp] = wmask;
    for (uint32_t m = wmask; m; m &= ~(1u << (31 - __clz(m)))) {
      const int j = 31 - __clz(m);
      const bool h0 = (wb0 >> j) & 1u, h1 = (wb1 >> j) & 1u;
      const EntryG &e = sm[j];
      Hit2 hh;
      hh.x[0] = hh.x[1] = hh.x[2] = f2(0.f);
      hh.delta = hh.dq = f2(0.f);
      if (kRot) hh.gm[0] = hh.gm[1] = hh.gm[2] = hh.gm[3] = f2(0.f);
      bool act = false;
#if SALF_BWD_PAIR2
      act = pair64_both<kRot, kDepth>(sc, e, bp, s_iv + ivrow[0] * kIvRow, s_iv + ivrow[1] * kIvRow, h0, h1, hh);
#else
      if (h0) act |= pair64_into<kRot, kDepth>(sc, entry_f(e), bp[0], s_iv + ivrow[0] * kIvRow, hh, 0);
      if (h1) act |= pair64_into<kRot, kDepth>(sc, entry_f(e), bp[1], s_iv + ivrow[1] * kIvRow, hh, 1);
#endif
      float tot = 0.0f;
      if (__any_sync(0xffffffffu, act)) {
        float g[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) g[k] = 0.f;
        bwd_segment2<kRot, sdf, kDepth>(spp[j], q, hh, g);
        // warp reduction through shared memory, lane k sums component k over the 32 lanes
#if SALF_BWD_XPCOL
        // component-major: lane r stores its 27 values down column r (conflict-free STS), lane k
        // reads its component's 32 values as 8 LDS.128 (row pitch 36 floats: the 8 lanes of a
        // 128-bit phase hit distinct banks) and sums them with packed adds
        float *xc = &xp[warp][0][0];
#pragma unroll
        for (int m = 0; m < kGradStride; ++m) xc[m * 36 + lane] = g[m];
        __syncwarp();
        if (lane < kGradStride) {
          const float4 *rowk = reinterpret_cast<const float4 *>(xc + lane * 36);
          float2 a0 = f2(0.f), a1 = f2(0.f);
#pragma unroll
          for (int m = 0; m < 8; m += 2) {
            const float4 u = rowk[m], v = rowk[m + 1];
            a0 = add2(a0, add2(make_float2(u.x, u.y), make_float2(v.x, v.y)));
            a1 = add2(a1, add2(make_float2(u.z, u.w), make_float2(v.z, v.w)));
          }
          const float2 a = add2(a0, a1);
          tot = a.x + a.y;
        }
        __syncwarp();
#else
        float4 *row = reinterpret_cast<float4 *>(&xp[warp][lane][0]);
#pragma unroll
        for (int m = 0; m < 7; ++m) row[m] = make_float4(g[4 * m], g[4 * m + 1], g[4 * m + 2], g[4 * m + 3]);
        __syncwarp();
        if (lane < kGradStride) {
          float t0 = xp[warp][0][lane], t1 = xp[warp][1][lane], t2 = xp[warp][2][lane], t3 = xp[warp][3][lane];
#pragma unroll
          for (int rr = 4; rr < 32; rr += 4) {
            t0 += xp[warp][rr][lane];
            t1 += xp[warp][rr + 1][lane];
            t2 += xp[warp][rr + 2][lane];
            t3 += xp[warp][rr + 3][lane];
          }
          tot = (t0 + t1) + (t2 + t3);
        }
        __syncwarp();
#endif
      }
#if SALF_BWD_WARPATOM
      if (!partial) {  // each warp adds its own entry totals (no block reduction, no end-of-chunk barrier)
        if (lane < kGradStride && tot != 0.0f) atomicAdd(grad + sm[j].vid * kGradStride + lane, (double)tot);
        continue;
      }
#endif
      if constexpr (kW == 4) {
        if (lane < kGradStride) red[j][warp][lane] = tot;
      }
    }
#if SALF_BWD_WARPATOM
    if (!partial) continue;
#endif
    if constexpr (kW != 4) continue;  // (the deterministic mode launches whole-tile CTAs)
    __syncthreads();
    for (int t = threadIdx.x; t < cn * kGradStride; t += kThreads) {
      const int j = t / kGradStride, k = t - j * kGradStride;
      float r[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) r[w] = (w < kW && ((s_wm[w % kW] >> j) & 1u)) ? red[j][w % kW][k] : 0.f;
      const float sum = (r[0] + r[1]) + (r[2] + r[3]);
      if (partial) partial[(base + j) * kGradStride + k] = sum;  // deterministic mode: one row per instance
      else if (sum != 0.0f) atomicAdd(grad + sm[j].vid * kGradStride + k, (double)sum);
    }
  }
}

}  // namespace salf

// ---------------------------------------------------------------------------
// C ABI

using namespace salf;

extern "C" int salf_project_voxels(const salf_scene_t *scene, const salf_camera_t *cam, double near,
                                   int32_t tile, double *rect, double *z_center, uint8_t *culled,
                                   int32_t *span_ref, int32_t *span_fit, uint64_t *zkey, int32_t *vrange,
                                   void *stream) {
  SALF_TRY {
    if (cam->kind != SALF_PINHOLE) return set_error(SALF_EINVAL, "rasterizer supports pinhole cameras only, got %s",
                                                     camera_kind_repr(cam->kind));
    if (scene->n == 0) return SALF_OK;
    PinholeDev c = make_pinhole(cam, near, tile);
    const int bs = 128;
    k_project<<<(unsigned)((scene->n + bs - 1) / bs), bs, 0, (cudaStream_t)stream>>>(
        scene->n, reinterpret_cast<const double4 *>(scene->geo), scene->rot, c, reinterpret_cast<double4 *>(rect), z_center,
        culled, reinterpret_cast<int4 *>(span_ref), reinterpret_cast<int4 *>(span_fit), zkey, vrange);
    return check_cuda("salf_project_voxels");
  }
  SALF_CATCH
}

// workspace layout for salf_raster_bin
#ifndef SALF_DEPTH_BUCKET
#define SALF_DEPTH_BUCKET 1  // depth rank by splitter bucket sort (0: 8-pass radix sort)
#endif

struct BinWs {
  int64_t *cnt, *base_r;
  uint64_t *st_sel, *st_scan;  // look-back status of k_select_vis / k_scan_ranked
  uint32_t *tickets;           // [0] select, [1] scan
  size_t clear_bytes;          // st_sel .. tickets are contiguous (one memset)
  int32_t *vis_idx, *vis_sorted;
  uint64_t *zk_vis, *zk_sorted;
  uint32_t *keys_a, *keys_b;
  int32_t *vals_a;
  void *sort_tmp;
  size_t sort_bytes;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static BinWs carve(void *ws, int64_t n, int64_t cap, int n_tiles, size_t *total) {
  BinWs w;
  size_t off = 0;
  char *p = (char *)ws;
  auto take = [&](size_t bytes) { char *q = p ? p + off : nullptr; off += align_up(bytes); return q; };
  const int64_t scan_tiles = (n + sortk::kScanTile - 1) / sortk::kScanTile;
  const size_t st_b = sizeof(uint64_t) * scan_tiles;
  char *c = take(2 * st_b + 2 * sizeof(uint32_t));
  w.st_sel = (uint64_t *)c;
  w.st_scan = c ? (uint64_t *)(c + st_b) : nullptr;
  w.tickets = c ? (uint32_t *)(c + 2 * st_b) : nullptr;
  w.clear_bytes = 2 * st_b + 2 * sizeof(uint32_t);
  w.cnt = (int64_t *)take(sizeof(int64_t) * n);
  w.base_r = (int64_t *)take(sizeof(int64_t) * n);
  w.vis_idx = (int32_t *)take(sizeof(int32_t) * n);
  w.vis_sorted = (int32_t *)take(sizeof(int32_t) * n);
  w.zk_vis = (uint64_t *)take(sizeof(uint64_t) * n);
  w.zk_sorted = (uint64_t *)take(sizeof(uint64_t) * n);
  w.keys_a = (uint32_t *)take(sizeof(uint32_t) * cap);
  w.keys_b = (uint32_t *)take(sizeof(uint32_t) * cap);
  w.vals_a = (int32_t *)take(sizeof(int32_t) * cap);
  w.sort_bytes = std::max(std::max(radix_sort_workspace_bytes(n, 8, 0, 64), bucket_sort_workspace_bytes()),
                          radix_sort_workspace_bytes(cap, 4, 0, bits_for((uint64_t)std::max(n_tiles, 1))));
  w.sort_tmp = take(w.sort_bytes);
  *total = off;
  return w;
}

extern "C" size_t salf_raster_bin_workspace_bytes(int64_t n_voxels, int64_t capacity, int32_t n_tiles) {
  size_t total = 0;
  carve(nullptr, std::max<int64_t>(n_voxels, 1), std::max<int64_t>(capacity, 1), n_tiles, &total);
  return total;
}

extern "C" int salf_raster_bin(const salf_scene_t *scene, const salf_camera_t *cam, double near, int32_t tile,
                               int32_t mode, const uint64_t *zkey, const int32_t *span, const uint8_t *visible_hint,
                               void *workspace, size_t workspace_bytes, int64_t capacity, int64_t *offsets,
                               int32_t *entries, int64_t *counts, void *stream) {
  SALF_TRY {
    (void)visible_hint;
    (void)mode;
    cudaStream_t st = (cudaStream_t)stream;
    PinholeDev c = make_pinhole(cam, near, tile);
    const int n_tiles = c.tiles_x * c.tiles_y;
    const int64_t n = scene->n;
    cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st);
    if (n == 0) {
      cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (n_tiles + 1), st);
      return check_cuda("salf_raster_bin");
    }
    capacity = std::max<int64_t>(capacity, 1);
    size_t need = 0;
    BinWs w = carve(workspace, n, capacity, n_tiles, &need);
    if (need > workspace_bytes) return set_error(SALF_EWORKSPACE, "raster bin workspace too small: %zu < %zu",
                                                 workspace_bytes, need);
    cudaMemsetAsync(w.st_sel, 0, w.clear_bytes, st);
    // visible voxels (non-empty span, ascending index), their depth keys, instance counts and totals
    const unsigned gs = (unsigned)((n + sortk::kScanTile - 1) / sortk::kScanTile);
    k_select_vis<<<gs, sortk::kBlock, 0, st>>>(n, reinterpret_cast<const int4 *>(span), zkey, w.cnt, w.vis_idx,
                                               w.zk_vis, w.st_sel, w.tickets, counts);
    // global depth rank of the visible voxels: stable sort of (zkey, index) -> lexsort's (z, vox) order
#if SALF_DEPTH_BUCKET
    // vis_idx is ascending (stable compaction) and unique, so the (z, index)
    // bucket sort gives the stable radix sort's permutation
    int rc = bucket_sort_pairs_u64(w.zk_vis, w.vis_idx, w.zk_sorted, w.vis_sorted, counts, n, w.sort_tmp,
                                   w.sort_bytes, st);
#else
    int rc = radix_sort_pairs_u64(w.zk_vis, w.vis_idx, w.zk_sorted, w.vis_sorted, counts, n, 0, 64, w.sort_tmp,
                                  w.sort_bytes, st);
#endif
    if (rc != SALF_OK) return rc;
    // instance slots in rank order
    k_scan_ranked<<<gs, sortk::kBlock, 0, st>>>(counts, w.vis_sorted, w.cnt, w.base_r, w.st_scan, w.tickets + 1);
    const int bs = 256;
    const unsigned ge = (unsigned)std::min<int64_t>((n * kEmitLanes + bs - 1) / bs, 148 * 16);
    k_emit<<<ge, bs, 0, st>>>(counts, w.vis_sorted,
                                                                     reinterpret_cast<const int4 *>(span), w.base_r,
                                                                     c.tiles_x, capacity, w.keys_a, w.vals_a);
    // stable sort by tile: each tile's list stays in depth-rank order
    rc = radix_sort_pairs_u32(w.keys_a, w.vals_a, w.keys_b, entries, counts + 1, capacity, 0,
                              bits_for((uint64_t)n_tiles), w.sort_tmp, w.sort_bytes, st);
    if (rc != SALF_OK) return rc;
    k_offsets<<<(n_tiles + 1 + bs - 1) / bs, bs, 0, st>>>(n_tiles, counts, capacity, w.keys_b, offsets);
    return check_cuda("salf_raster_bin");
  }
  SALF_CATCH
}

extern "C" int salf_raster_composite(const salf_scene_t *scene, const salf_camera_t *cam,
                                     const salf_raster_opts_t *opts, const int64_t *offsets, const int32_t *entries,
                                     float *out_rgb, float *out_opacity, float *out_depth, double *saved,
                                     const int32_t *vrange, const int32_t *tile_order, uint32_t *hitbits,
                                     void *stream) {
  SALF_TRY {
    if (cam->kind != SALF_PINHOLE) return set_error(SALF_EINVAL, "rasterizer supports pinhole cameras only, got %s",
                                                     camera_kind_repr(cam->kind));
    if (opts->tile < 1 || opts->tile > 16) return set_error(SALF_EINVAL, "tile size must be in [1, 16]");
    PinholeDev c = make_pinhole(cam, opts->near, opts->tile);
    const int n_tiles = c.tiles_x * c.tiles_y;
    const int threads = std::max(32, opts->tile * opts->tile);
    cudaStream_t st = (cudaStream_t)stream;
    const bool rot = scene->rot != nullptr;
    if (opts->exact_color && rot)
      k_composite<true><<<n_tiles, threads, 0, st>>>(*scene, c, *opts, offsets, entries, out_rgb, out_opacity,
                                                           out_depth, saved);
    else if (opts->exact_color)
      k_composite<false><<<n_tiles, threads, 0, st>>>(*scene, c, *opts, offsets, entries, out_rgb, out_opacity,
                                                            out_depth, saved);
    else {
      // certified mixed-precision pass, then fp64 recomputation of the flagged pixels
      // (SALF_NO_REDO=1 skips the second pass: flagged pixels keep opacity NaN; diagnostics only)
      static const bool no_redo = getenv("SALF_NO_REDO") && getenv("SALF_NO_REDO")[0] == '1';
      const int64_t npx = (int64_t)c.width * c.height;
      const unsigned rb = (unsigned)((npx + 127) / 128);
      const bool sdf = scene->density_mode == SALF_DENSITY_SDF;
      // whole warps (the per-chunk footprint masks are warp ballots); slots past tile^2 idle.
      // 16 x 16 tiles: SALF_FWD_PARTS CTAs per tile
      const int fparts = opts->tile == 16 ? SALF_FWD_PARTS : 1;
      const int fthreads = ((threads + 31) & ~31) / fparts;
#define SALF_LAUNCH_FWD(ROT, SDF)                                                                             \
  k_composite_fast<ROT, SDF><<<n_tiles * fparts, fthreads, 0, st>>>(*scene, c, *opts, offsets, entries,       \
                                                                    out_rgb, out_opacity, out_depth, saved,  \
                                                                    vrange, tile_order, hitbits, fparts)
      if (rot) {
        if (sdf) SALF_LAUNCH_FWD(true, true); else SALF_LAUNCH_FWD(true, false);
        if (!no_redo)
          k_composite_redo<true><<<rb, 128, 0, st>>>(*scene, c, *opts, offsets, entries, out_rgb, out_opacity,
                                                     out_depth, saved, hitbits);
      } else {
        if (sdf) SALF_LAUNCH_FWD(false, true); else SALF_LAUNCH_FWD(false, false);
        if (!no_redo)
          k_composite_redo<false><<<rb, 128, 0, st>>>(*scene, c, *opts, offsets, entries, out_rgb, out_opacity,
                                                      out_depth, saved, hitbits);
      }
#undef SALF_LAUNCH_FWD
    }
    return check_cuda("salf_raster_composite");
  }
  SALF_CATCH
}

static int raster_backward_launch(const salf_scene_t *scene, const salf_camera_t *cam,
                                  const salf_raster_opts_t *opts, const int64_t *offsets, const int32_t *entries,
                                  const double *saved, const double *d_rgb, const double *d_depth, double *grad,
                                  float *partial, const int32_t *vrange, const int32_t *tile_order,
                                  const uint32_t *hitbits, cudaStream_t st) {
  if (cam->kind != SALF_PINHOLE) return set_error(SALF_EINVAL, "rasterizer supports pinhole cameras only, got %s",
                                                   camera_kind_repr(cam->kind));
  if (opts->tile < 1 || opts->tile > 16) return set_error(SALF_EINVAL, "tile size must be in [1, 16]");
  PinholeDev c = make_pinhole(cam, opts->near, opts->tile);
  const int n_tiles = c.tiles_x * c.tiles_y;
  const int threads = ((std::max(32, opts->tile * opts->tile) + 31) / 32) * 32;
  const int threads_np = ((std::max(32, (opts->tile * opts->tile + SALF_BWD_NP - 1) / SALF_BWD_NP) + 31) / 32) * 32;
  const bool rot = scene->rot != nullptr;
  if (opts->exact_color && rot)
    k_backward<true><<<n_tiles, threads, 0, st>>>(*scene, c, *opts, offsets, entries, saved, d_rgb, d_depth,
                                                        grad, partial);
  else if (opts->exact_color)
    k_backward<false><<<n_tiles, threads, 0, st>>>(*scene, c, *opts, offsets, entries, saved, d_rgb, d_depth,
                                                         grad, partial);
  else {
    const bool sdf = scene->density_mode == SALF_DENSITY_SDF;
    const bool depth = d_depth != nullptr;  // no depth seeds (colour-only loss): the depth term is dropped
#define SALF_LAUNCH_BWD(ROT, SDF, DEPTH)                                                                    \
  do {                                                                                                      \
    if (hitbits) {                                                                                          \
      static bool attr = false;                                                                             \
      if (!attr) {                                                                                          \
        cudaFuncSetAttribute(k_backward_hits<ROT, SDF, DEPTH, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)kXpBytes);                                                                \
        cudaFuncSetAttribute(k_backward_hits<ROT, SDF, DEPTH, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)(kXpBytes / 2));                                                          \
        attr = true;                                                                                        \
      }                                                                                                     \
      if (partial || !SALF_BWD_HALF)                                                                        \
        k_backward_hits<ROT, SDF, DEPTH, 4><<<n_tiles, 128, kXpBytes, st>>>(                                 \
            *scene, c, *opts, offsets, entries, saved, d_rgb, d_depth, grad, partial, vrange, tile_order, hitbits); \
      else                                                                                                  \
        k_backward_hits<ROT, SDF, DEPTH, 2><<<2 * n_tiles, 64, kXpBytes / 2, st>>>(                          \
            *scene, c, *opts, offsets, entries, saved, d_rgb, d_depth, grad, partial, vrange, tile_order, hitbits); \
    } else                                                                                                  \
      k_backward_fast<ROT, SALF_BWD_NP, SDF, DEPTH><<<n_tiles, threads_np, 0, st>>>(                        \
          *scene, c, *opts, offsets, entries, saved, d_rgb, d_depth, grad, partial, vrange, tile_order);    \
  } while (0)
    if (rot) {
      if (sdf) SALF_LAUNCH_BWD(true, true, true); else SALF_LAUNCH_BWD(true, false, true);
    } else if (depth) {
      if (sdf) SALF_LAUNCH_BWD(false, true, true); else SALF_LAUNCH_BWD(false, false, true);
    } else {
      if (sdf) SALF_LAUNCH_BWD(false, true, false); else SALF_LAUNCH_BWD(false, false, false);
    }
#undef SALF_LAUNCH_BWD
  }
  return check_cuda("salf_raster_backward");
}

extern "C" int salf_raster_backward(const salf_scene_t *scene, const salf_camera_t *cam,
                                    const salf_raster_opts_t *opts, const int64_t *offsets, const int32_t *entries,
                                    const double *saved, const double *d_rgb, const double *d_depth, double *grad,
                                    const int32_t *vrange, const int32_t *tile_order, const uint32_t *hitbits,
                                    void *stream) {
  SALF_TRY {
    return raster_backward_launch(scene, cam, opts, offsets, entries, saved, d_rgb, d_depth, grad, nullptr, vrange,
                                  tile_order, hitbits, (cudaStream_t)stream);
  }
  SALF_CATCH
}

// ---------------------------------------------------------------------------
// Deterministic raster backward (SPEC-mandated ordered reduction; SURVEY §7
// hard part 5): the kernel writes one 27-row per (tile, entry) instance --
// the CTA's fixed-order sum -- instead of atomics; instances are then
// stable-sorted by voxel (ties in instance, i.e. tile-major, order) and each
// voxel's rows are summed sequentially in fp64 by one warp (lane = component)
// and added to grad.  Bitwise identical across runs.

__global__ void k_iota32(int64_t n, int32_t *__restrict__ v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

// first row of each voxel's run in the vid-sorted rows
__global__ void k_run_first(int64_t n, const uint32_t *__restrict__ key, int32_t *__restrict__ first) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n && (p == 0 || key[p] != key[p - 1])) first[key[p]] = (int32_t)p;
}

// one warp per voxel; lane k sums component k over the voxel's rows in order
// (fp64) and adds it to grad (single writer per voxel)
__global__ void k_det_reduce(int64_t n, const int32_t *__restrict__ first, const uint32_t *__restrict__ vid,
                             const int32_t *__restrict__ row, const float *__restrict__ rows, int64_t n_vox,
                             double *__restrict__ grad) {
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= n_vox || lane >= kGradStride) return;
  const int64_t p0 = first[v];
  if (p0 < 0) return;
  double s = 0.0;
  for (int64_t p = p0; p < n && (int64_t)vid[p] == v; ++p) s += (double)rows[(int64_t)row[p] * kGradStride + lane];
  double *g = grad + v * kGradStride + lane;
  *g = *g + s;
}

struct DetWs {
  uint32_t *vid_sorted;
  int32_t *row, *row_sorted, *first;
  void *sort_tmp;
  size_t sort_bytes;
};

static DetWs carve_det(void *ws, int64_t ni, int64_t n_vox, size_t *total) {
  DetWs w;
  size_t off = 0;
  char *p = (char *)ws;
  auto take = [&](size_t bytes) { char *q = p ? p + off : nullptr; off += align_up(bytes); return q; };
  w.vid_sorted = (uint32_t *)take(sizeof(uint32_t) * ni);
  w.row = (int32_t *)take(sizeof(int32_t) * ni);
  w.row_sorted = (int32_t *)take(sizeof(int32_t) * ni);
  w.first = (int32_t *)take(sizeof(int32_t) * (n_vox + 1));
  w.sort_bytes = radix_sort_workspace_bytes(ni, 4, 0, 32);
  w.sort_tmp = take(w.sort_bytes);
  *total = off;
  return w;
}

size_t salf::det_reduce_workspace_bytes(int64_t n_rows, int64_t n_vox) {
  size_t total = 0;
  carve_det(nullptr, std::max<int64_t>(n_rows, 1), std::max<int64_t>(n_vox, 1), &total);
  return total;
}

// Ordered reduction of 27-rows into grad: rows stable-sorted by voxel id
// (row order within a voxel), summed sequentially per voxel.  row_vid[i] ==
// n_vox marks an unused row.
int salf::det_reduce_rows(int64_t n_rows, const uint32_t *row_vid, const float *rows, int64_t n_vox, double *grad,
                          void *workspace, size_t workspace_bytes, cudaStream_t st) {
  if (n_rows <= 0) return SALF_OK;
  size_t need = 0;
  DetWs w = carve_det(workspace, n_rows, std::max<int64_t>(n_vox, 1), &need);
  if (need > workspace_bytes)
    return set_error(SALF_EWORKSPACE, "deterministic reduction workspace too small: %zu < %zu", workspace_bytes, need);
  const int bs = 256;
  const unsigned g = (unsigned)((n_rows + bs - 1) / bs);
  k_iota32<<<g, bs, 0, st>>>(n_rows, w.row);
  const int rc = radix_sort_pairs_u32(row_vid, w.row, w.vid_sorted, w.row_sorted, nullptr, n_rows, 0,
                                      bits_for((uint64_t)std::max<int64_t>(n_vox, 1)), w.sort_tmp, w.sort_bytes, st);
  if (rc != SALF_OK) return rc;
  cudaMemsetAsync(w.first, 0xff, sizeof(int32_t) * (n_vox + 1), st);
  k_run_first<<<g, bs, 0, st>>>(n_rows, w.vid_sorted, w.first);
  k_det_reduce<<<(unsigned)((n_vox * 32 + bs - 1) / bs), bs, 0, st>>>(n_rows, w.first, w.vid_sorted, w.row_sorted,
                                                                     rows, n_vox, grad);
  return check_cuda("det_reduce_rows");
}

// tile launch order: 16-bit descending-length keys, stable radix sort (ties in tile order)
__global__ void k_tile_len_keys(int32_t n, const int64_t *__restrict__ offsets, uint32_t *__restrict__ keys,
                                int32_t *__restrict__ ids) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t len = offsets[t + 1] - offsets[t];
  keys[t] = 0xffffu - (uint32_t)(len < 0xffff ? len : 0xffff);
  ids[t] = t;
}

extern "C" size_t salf_raster_tile_order_workspace_bytes(int32_t n_tiles) {
  const size_t n = (size_t)std::max(n_tiles, 1);
  return align_up(2 * n * sizeof(uint32_t)) + align_up(n * sizeof(int32_t)) +
         radix_sort_workspace_bytes((int64_t)n, 4, 0, 16);
}

extern "C" int salf_raster_tile_order(const int64_t *offsets, int32_t n_tiles, int32_t *order, void *workspace,
                                      size_t workspace_bytes, void *stream) {
  SALF_TRY {
    if (n_tiles <= 0) return SALF_OK;
    if (workspace_bytes < salf_raster_tile_order_workspace_bytes(n_tiles))
      return set_error(SALF_EWORKSPACE, "tile order workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    char *p = (char *)workspace;
    uint32_t *ka = (uint32_t *)p, *kb = ka + n_tiles;
    p += align_up(2 * (size_t)n_tiles * sizeof(uint32_t));
    int32_t *ids = (int32_t *)p;
    p += align_up((size_t)n_tiles * sizeof(int32_t));
    k_tile_len_keys<<<(n_tiles + 255) / 256, 256, 0, st>>>(n_tiles, offsets, ka, ids);
    const int rc = radix_sort_pairs_u32(ka, ids, kb, order, nullptr, n_tiles, 0, 16, p,
                                        radix_sort_workspace_bytes(n_tiles, 4, 0, 16), st);
    if (rc != SALF_OK) return rc;
    return check_cuda("salf_raster_tile_order");
  }
  SALF_CATCH
}

extern "C" size_t salf_raster_backward_det_workspace_bytes(int64_t n_instances, int64_t n_voxels) {
  const int64_t ni = std::max<int64_t>(n_instances, 1);
  return align_up(sizeof(float) * kGradStride * ni) + det_reduce_workspace_bytes(ni, n_voxels);
}

extern "C" int salf_raster_backward_deterministic(const salf_scene_t *scene, const salf_camera_t *cam,
                                                  const salf_raster_opts_t *opts, const int64_t *offsets,
                                                  const int32_t *entries, int64_t n_instances, const double *saved,
                                                  const double *d_rgb, const double *d_depth, double *grad,
                                                  const int32_t *vrange, const int32_t *tile_order,
                                                  const uint32_t *hitbits, void *workspace, size_t workspace_bytes,
                                                  void *stream) {
  SALF_TRY {
    if (n_instances <= 0) return SALF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t part = align_up(sizeof(float) * kGradStride * n_instances);
    if (workspace_bytes < part) return set_error(SALF_EWORKSPACE, "deterministic backward workspace too small");
    float *partial = (float *)workspace;
    cudaMemsetAsync(partial, 0, sizeof(float) * kGradStride * n_instances, st);
    const int rc = raster_backward_launch(scene, cam, opts, offsets, entries, saved, d_rgb, d_depth, grad, partial,
                                          vrange, tile_order, hitbits, st);
    if (rc != SALF_OK) return rc;
    // instance rows keyed by their voxel (entries[i])
    return det_reduce_rows(n_instances, reinterpret_cast<const uint32_t *>(entries), partial, scene->n, grad,
                           (char *)workspace + part, workspace_bytes - part, st);
  }
  SALF_CATCH
}

#ifdef SALF_DIAG_CHORD
// diagnostics build only: backward hits / chords under the cheap bound / chords re-derived in fp64
extern "C" int salf_debug_counters(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, salf::g_diag, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(salf::g_diag, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" size_t salf_raster_hitbits_words(int64_t capacity, int32_t n_tiles) {
  return (size_t)salf::kHitSlots * (size_t)(std::max<int64_t>(capacity, 0) / 32 + std::max(n_tiles, 0) + 1);
}
