// salf_sort.cu -- stable LSD radix sort of (key, int32) pairs, hand-written for
// sm_100a (replaces the reference's np.lexsort in render_raster.py:177 and
// np.argsort in the deterministic reductions; see salf_sort.cuh).
//
// Per sort: one histogram kernel computes every pass's 256-bin digit histogram
// in one read of the keys; then one onesweep kernel per 8-bit digit:
//   * CTA tile = 4096 keys (256 threads x 16), tile id from an atomic ticket so
//     look-back only ever waits on CTAs that started earlier;
//   * warp w owns keys [w*512, (w+1)*512) of the tile, item k of lane l is key
//     w*512 + 32k + l: __match_any_sync ranks equal digits inside the warp in
//     key order and a per-warp shared histogram carries the count across items
//     -> stable;
//   * thread d of the CTA turns the per-warp counts of digit d into warp
//     prefixes, publishes the tile's count of d and looks back over earlier
//     tiles (flag + 30-bit count in one 32-bit word);
//   * scatter: global digit start + look-back prefix + warp prefix + rank.
// Element counts can be device-resident (n_dev): CTAs past the end exit.
#include "salf_internal.h"
#include "salf_sort.cuh"

namespace salf {
namespace sortk {

template <typename K>
__global__ void __launch_bounds__(kBlock) k_radix_hist(const K *__restrict__ keys, const int64_t *__restrict__ n_dev,
                                                       int64_t n_max, int begin_bit, int n_pass,
                                                       uint32_t *__restrict__ hist) {
  __shared__ uint32_t s[8][kRadix];
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) (&s[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = n_dev ? min(*n_dev, n_max) : n_max;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const K k = keys[i];
    for (int p = 0; p < n_pass; ++p) atomicAdd(&s[p][(uint32_t)(k >> (begin_bit + 8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_pass * kRadix; i += blockDim.x) {
    const uint32_t c = (&s[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// One 8-bit digit pass.  Keys are ranked per warp (match_any, stable), turned
// into block-local positions (digit-major), staged in shared memory in that
// order and written out from there: consecutive threads then write
// consecutive global slots of the same digit (coalesced runs).
template <typename K, int ITEMS>
__global__ void __launch_bounds__(kBlock) k_onesweep(const K *__restrict__ kin, const int32_t *__restrict__ vin,
                                                     K *__restrict__ kout, int32_t *__restrict__ vout,
                                                     const int64_t *__restrict__ n_dev, int64_t n_max, int shift,
                                                     const uint32_t *__restrict__ hist, uint32_t *__restrict__ status,
                                                     uint32_t *__restrict__ ticket) {
  constexpr int TILE = kBlock * ITEMS;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  K *s_key = reinterpret_cast<K *>(s_dyn);                    // TILE keys in block-local order
  int32_t *s_val = reinterpret_cast<int32_t *>(s_key + TILE);  // TILE values
  __shared__ uint32_t s_wh[kWarps][kRadix];
  __shared__ uint32_t s_glob[kRadix];  // global slot of the block's first key of digit d
  __shared__ uint32_t s_loc[kRadix];   // block-local start of digit d
  __shared__ uint32_t s_warp[kWarps], s_warp2[kWarps];
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kBlock) (&s_wh[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t n = n_dev ? min(*n_dev, n_max) : n_max;
  const int64_t start = (int64_t)tile * TILE;
  if (start >= n) return;  // uniform over the CTA
  const int cnt = (int)min((int64_t)TILE, n - start);

  K key[ITEMS];
  int32_t val[ITEMS];
  uint32_t loc[ITEMS];
  const int64_t wbase = start + (int64_t)w * (32 * ITEMS);
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t idx = wbase + 32 * k + lane;
    const bool ok = idx < n;
    key[k] = ok ? kin[idx] : (K)0;
    val[k] = ok ? vin[idx] : 0;
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const bool ok = wbase + 32 * k + lane < n;
    const uint32_t d = ok ? ((uint32_t)(key[k] >> shift) & 255u) : 256u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t b = 0;
    if (ok) b = s_wh[w][d];
    __syncwarp();
    if (ok) {
      loc[k] = b + __popc(peers & lt);
      if ((peers & lt) == 0) s_wh[w][d] = b + __popc(peers);  // lowest peer lane updates
    }
    __syncwarp();
  }
  __syncthreads();
  // digit tid: warp prefixes and the tile's count
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) {
    const uint32_t c = s_wh[i][tid];
    s_wh[i][tid] = run;
    run += c;
  }
  // block-local digit starts (exclusive scan of run) and global digit starts
  // (exclusive scan of the pass histogram), both over the 256 digits
  const uint32_t h = hist[tid];
  uint32_t x = run, y = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t xa = __shfl_up_sync(0xffffffffu, x, o), ya = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) {
      x += xa;
      y += ya;
    }
  }
  if (lane == 31) {
    s_warp[w] = x;
    s_warp2[w] = y;
  }
  // look-back for digit tid (overlaps the scan's barrier wait)
  uint32_t excl = 0;
  {
    uint32_t *me = status + (size_t)tile * kRadix + tid;
    if (tile == 0) {
      st_relaxed(me, kFlagP32 | run);
    } else {
      st_relaxed(me, kFlagA32 | run);
      for (int64_t p = (int64_t)tile - 1;; --p) {
        uint32_t v;
        do { v = ld_relaxed(status + (size_t)p * kRadix + tid); } while ((v & ~kVal32) == 0);
        excl += v & kVal32;
        if (v & kFlagP32) break;
      }
      st_relaxed(me, kFlagP32 | (excl + run));
    }
  }
  __syncthreads();
  uint32_t ox = 0, oy = 0;
  for (int i = 0; i < w; ++i) {
    ox += s_warp[i];
    oy += s_warp2[i];
  }
  const uint32_t lstart = ox + x - run;
  s_loc[tid] = lstart;
  s_glob[tid] = oy + y - h + excl;
  __syncthreads();
  // stage in block-local (digit-major, stable) order
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (wbase + 32 * k + lane < n) {
      const uint32_t d = (uint32_t)(key[k] >> shift) & 255u;
      const uint32_t lp = s_loc[d] + s_wh[w][d] + loc[k];
      s_key[lp] = key[k];
      s_val[lp] = val[k];
    }
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += kBlock) {
    const K kk = s_key[i];
    const uint32_t d = (uint32_t)(kk >> shift) & 255u;
    const uint32_t dst = s_glob[d] + (uint32_t)i - s_loc[d];
    kout[dst] = kk;
    vout[dst] = s_val[i];
  }
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct SortWs {
  uint32_t *hist, *ticket, *status;  // contiguous: cleared by one memset
  size_t clear_bytes;
  void *ktmp;
  int32_t *vtmp;
};

static SortWs carve_sort(void *ws, int64_t n_max, int key_bytes, int n_pass, size_t *total) {
  SortWs w;
  char *p = (char *)ws;
  size_t off = 0;
  auto take = [&](size_t bytes) { char *q = p ? p + off : nullptr; off += align_up(bytes); return q; };
  const int64_t tiles = std::max<int64_t>((n_max + (int64_t)kBlock * 4 - 1) / ((int64_t)kBlock * 4), 1);
  const size_t hist_b = sizeof(uint32_t) * kRadix * n_pass, tick_b = sizeof(uint32_t) * 8;
  const size_t stat_b = sizeof(uint32_t) * kRadix * (size_t)tiles * n_pass;
  char *c = take(hist_b + tick_b + stat_b);
  w.hist = (uint32_t *)c;
  w.ticket = c ? (uint32_t *)(c + hist_b) : nullptr;
  w.status = c ? (uint32_t *)(c + hist_b + tick_b) : nullptr;
  w.clear_bytes = hist_b + tick_b + stat_b;
  w.ktmp = take((size_t)key_bytes * std::max<int64_t>(n_max, 1));
  w.vtmp = (int32_t *)take(sizeof(int32_t) * std::max<int64_t>(n_max, 1));
  *total = off;
  return w;
}

// keys per thread: enough CTAs to cover the SMs twice, at most 16
static int items_for(int64_t n_max) {
  if (n_max <= (int64_t)kBlock * 4 * 148 * 2) return 4;
  if (n_max <= (int64_t)kBlock * 8 * 148 * 2) return 8;
  return 16;
}

static int n_passes(int begin_bit, int end_bit) { return std::max(1, (end_bit - begin_bit + 7) / 8); }

template <typename K>
static int radix_sort(const K *keys_in, const int32_t *vals_in, K *keys_out, int32_t *vals_out, const int64_t *n_dev,
                      int64_t n_max, int begin_bit, int end_bit, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (n_max <= 0) return SALF_OK;
  if (n_max >= (int64_t)kVal32) return set_error(SALF_EINVAL, "radix sort: %lld keys exceed 2^30", (long long)n_max);
  const int np = n_passes(begin_bit, end_bit);
  if (np > 8) return set_error(SALF_EINVAL, "radix sort: at most 64 key bits");
  size_t need = 0;
  SortWs w = carve_sort(ws, n_max, sizeof(K), np, &need);
  if (need > ws_bytes) return set_error(SALF_EWORKSPACE, "radix sort workspace too small: %zu < %zu", ws_bytes, need);
  cudaMemsetAsync(w.hist, 0, w.clear_bytes, st);
  const unsigned hb = (unsigned)std::min<int64_t>((n_max + kBlock * 8 - 1) / (kBlock * 8), 148 * 8);
  k_radix_hist<K><<<hb, kBlock, 0, st>>>(keys_in, n_dev, n_max, begin_bit, np, w.hist);
  // small sorts: short CTA tiles (more CTAs in flight); large: 16 keys per thread.  A
  // device-resident count is usually far below its bound (the visible voxels of a
  // frame vs the scene's voxels): size for a quarter of the bound.
  const int items = items_for(n_dev ? n_max / 4 : n_max);
  const int64_t tiles = (n_max + (int64_t)kBlock * items - 1) / ((int64_t)kBlock * items);
  const size_t smem = (size_t)kBlock * items * (sizeof(K) + sizeof(int32_t));
  static bool attr_set = false;  // dynamic shared memory above 48 KB needs the opt-in
  if (!attr_set) {
    cudaFuncSetAttribute(k_onesweep<K, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlock * 4 * 12);
    cudaFuncSetAttribute(k_onesweep<K, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlock * 8 * 12);
    cudaFuncSetAttribute(k_onesweep<K, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlock * 16 * 12);
    attr_set = true;
  }
  // ping-pong so that the last pass lands in keys_out / vals_out
  const K *ksrc = keys_in;
  const int32_t *vsrc = vals_in;
  for (int p = 0; p < np; ++p) {
    const bool to_out = ((np - 1 - p) % 2) == 0;
    K *kdst = to_out ? keys_out : (K *)w.ktmp;
    int32_t *vdst = to_out ? vals_out : w.vtmp;
    const int sh = begin_bit + 8 * p;
    uint32_t *stp = w.status + (size_t)p * kRadix * tiles;
    if (items == 4)
      k_onesweep<K, 4><<<(unsigned)tiles, kBlock, smem, st>>>(ksrc, vsrc, kdst, vdst, n_dev, n_max, sh,
                                                              w.hist + p * kRadix, stp, w.ticket + p);
    else if (items == 8)
      k_onesweep<K, 8><<<(unsigned)tiles, kBlock, smem, st>>>(ksrc, vsrc, kdst, vdst, n_dev, n_max, sh,
                                                              w.hist + p * kRadix, stp, w.ticket + p);
    else
      k_onesweep<K, 16><<<(unsigned)tiles, kBlock, smem, st>>>(ksrc, vsrc, kdst, vdst, n_dev, n_max, sh,
                                                               w.hist + p * kRadix, stp, w.ticket + p);
    ksrc = kdst;
    vsrc = vdst;
  }
  return check_cuda("radix_sort_pairs");
}

}  // namespace sortk

size_t radix_sort_workspace_bytes(int64_t n_max, int key_bytes, int begin_bit, int end_bit) {
  size_t total = 0;
  sortk::carve_sort(nullptr, std::max<int64_t>(n_max, 1), key_bytes, sortk::n_passes(begin_bit, end_bit), &total);
  return total;
}

int radix_sort_pairs_u32(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out, int32_t *vals_out,
                         const int64_t *n_dev, int64_t n_max, int begin_bit, int end_bit, void *ws, size_t ws_bytes,
                         cudaStream_t st) {
  return sortk::radix_sort<uint32_t>(keys_in, vals_in, keys_out, vals_out, n_dev, n_max, begin_bit, end_bit, ws,
                                     ws_bytes, st);
}

int radix_sort_pairs_u64(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out, int32_t *vals_out,
                         const int64_t *n_dev, int64_t n_max, int begin_bit, int end_bit, void *ws, size_t ws_bytes,
                         cudaStream_t st) {
  return sortk::radix_sort<uint64_t>(keys_in, vals_in, keys_out, vals_out, n_dev, n_max, begin_bit, end_bit, ws,
                                     ws_bytes, st);
}

}  // namespace salf

extern "C" size_t salf_sort_pairs_workspace_bytes(int64_t n_max, int32_t key_bytes, int32_t begin_bit,
                                                  int32_t end_bit) {
  return salf::radix_sort_workspace_bytes(n_max, key_bytes, begin_bit, end_bit);
}

extern "C" int salf_sort_pairs(const void *keys_in, const int32_t *vals_in, void *keys_out, int32_t *vals_out,
                               int32_t key_bytes, const int64_t *n_dev, int64_t n_max, int32_t begin_bit,
                               int32_t end_bit, void *workspace, size_t workspace_bytes, void *stream) {
  SALF_TRY {
    if (begin_bit < 0 || end_bit > 8 * key_bytes || begin_bit >= end_bit)
      return salf::set_error(SALF_EINVAL, "sort_pairs: bad bit range [%d, %d)", begin_bit, end_bit);
    cudaStream_t st = (cudaStream_t)stream;
    if (key_bytes == 4)
      return salf::radix_sort_pairs_u32((const uint32_t *)keys_in, vals_in, (uint32_t *)keys_out, vals_out, n_dev,
                                        n_max, begin_bit, end_bit, workspace, workspace_bytes, st);
    if (key_bytes == 8)
      return salf::radix_sort_pairs_u64((const uint64_t *)keys_in, vals_in, (uint64_t *)keys_out, vals_out, n_dev,
                                        n_max, begin_bit, end_bit, workspace, workspace_bytes, st);
    return salf::set_error(SALF_EINVAL, "sort_pairs: key_bytes must be 4 or 8, got %d", key_bytes);
  }
  SALF_CATCH
}
