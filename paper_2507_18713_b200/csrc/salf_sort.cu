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
#include <climits>

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


// ---------------------------------------------------------------------------
// Splitter bucket sort of (u64 key, int32 value) pairs that are unique as pairs
// (the binning's depth rank: values are voxel indices), ordered by (key, value)
// -- the same permutation as the stable LSD radix sort of keys over input in
// value order.  kBuckets - 1 splitters are taken at evenly spaced input
// positions and sorted; every element finds its bucket by binary search,
// buckets are filled through CTA-aggregated slot claims, and one CTA per bucket
// sorts it in shared memory (bitonic; global memory beyond the capacity).
// Five launches instead of the radix sort's nine, no per-digit look-back chain.
namespace sortk {

constexpr int kBuckets = 1024;
constexpr int kBktTile = 2048;  // elements per CTA of the count / scatter kernels
constexpr int kBktCap = 2048;   // bucket elements sorted in shared memory

__device__ __forceinline__ bool kv_less(uint64_t ka, int32_t va, uint64_t kb, int32_t vb) {
  return ka < kb || (ka == kb && va < vb);
}

// in-place direction-free bitonic network over P = next pow2 >= n elements
// (pairs past n skipped: the virtual pads are +inf)
template <typename KeyAt, typename ValAt>
__device__ __forceinline__ void bitonic_sort(int n, KeyAt key, ValAt val) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const bool mirror = j == (k >> 1);
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        int a, b;
        if (mirror) {
          const int h = k >> 1, blk = i >> (31 - __clz(h)), off = i & (h - 1);
          a = blk * k + off;
          b = blk * k + k - 1 - off;
        } else {
          a = 2 * i - (i & (j - 1));
          b = a + j;
        }
        if (b >= n) continue;
        const uint64_t ka = key(a), kb = key(b);
        const int32_t va = val(a), vb = val(b);
        if (kv_less(kb, vb, ka, va)) {
          key(a) = kb; key(b) = ka;
          val(a) = vb; val(b) = va;
        }
      }
      __syncthreads();
    }
  }
}

// splitters: kBktOver * kBuckets evenly spaced samples sorted in one CTA, every
// kBktOver-th kept (oversampling evens out the bucket sizes)
#ifndef SALF_BKT_OVER
#define SALF_BKT_OVER 2
#endif
constexpr int kBktOver = SALF_BKT_OVER;
__global__ void __launch_bounds__(1024) k_bkt_splitters(const uint64_t *__restrict__ kin,
                                                        const int32_t *__restrict__ vin,
                                                        const int64_t *__restrict__ n_dev, int64_t n_max,
                                                        uint64_t *__restrict__ sk, int32_t *__restrict__ sv) {
  constexpr int m = kBktOver * kBuckets;
  __shared__ uint64_t k_s[m];
  __shared__ int32_t v_s[m];
  const int64_t n = n_dev ? min(*n_dev, n_max) : n_max;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int64_t pos = (int64_t)(((double)i + 0.5) * (double)n / m);
    const bool ok = pos < n;
    k_s[i] = ok ? kin[pos] : ~0ull;
    v_s[i] = ok ? vin[pos] : INT_MAX;
  }
  __syncthreads();
  bitonic_sort(m, [&](int i) -> uint64_t & { return k_s[i]; }, [&](int i) -> int32_t & { return v_s[i]; });
  for (int i = threadIdx.x; i < kBuckets - 1; i += blockDim.x) {
    sk[i] = k_s[kBktOver * (i + 1)];
    sv[i] = v_s[kBktOver * (i + 1)];
  }
}

// bucket of (key, value): the number of splitters strictly below it
__device__ __forceinline__ int bkt_of(const uint64_t *sk, const int32_t *sv, uint64_t k, int32_t v) {
  int lo = 0, hi = kBuckets - 1;  // answer in [0, kBuckets - 1]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (kv_less(sk[mid], sv[mid], k, v)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// per-bucket counts (CTA-aggregated in shared memory)
__global__ void __launch_bounds__(256) k_bkt_count(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin,
                                                   const int64_t *__restrict__ n_dev, int64_t n_max,
                                                   const uint64_t *__restrict__ spk, const int32_t *__restrict__ spv,
                                                   uint32_t *__restrict__ bcnt) {
  __shared__ uint64_t sk[kBuckets - 1];
  __shared__ int32_t sv[kBuckets - 1];
  __shared__ uint32_t c[kBuckets];
  const int64_t n = n_dev ? min(*n_dev, n_max) : n_max;
  const int64_t start = (int64_t)blockIdx.x * kBktTile;
  if (start >= n) return;
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) {
    c[i] = 0;
    if (i < kBuckets - 1) { sk[i] = spk[i]; sv[i] = spv[i]; }
  }
  __syncthreads();
  const int64_t end = min(start + kBktTile, n);
  for (int64_t i = start + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&c[bkt_of(sk, sv, kin[i], vin[i])], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
    if (c[i]) atomicAdd(bcnt + i, c[i]);
}

// bucket offsets (exclusive scan, one CTA of kBuckets threads); cursors start there
__global__ void __launch_bounds__(kBuckets) k_bkt_scan(const uint32_t *__restrict__ bcnt, uint32_t *__restrict__ boff,
                                                       uint32_t *__restrict__ cursor) {
  __shared__ uint32_t s_w[kBuckets / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t v = bcnt[t];
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  uint32_t off = 0;
  for (int i = 0; i < w; ++i) off += s_w[i];
  const uint32_t ex = off + x - v;
  boff[t] = ex;
  cursor[t] = ex;
  if (t == kBuckets - 1) boff[kBuckets] = ex + v;
}

// scatter into the buckets (CTA-aggregated slot claims, any order inside a bucket)
__global__ void __launch_bounds__(256) k_bkt_scatter(const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin,
                                                     const int64_t *__restrict__ n_dev, int64_t n_max,
                                                     const uint64_t *__restrict__ spk, const int32_t *__restrict__ spv,
                                                     uint32_t *__restrict__ cursor, uint64_t *__restrict__ kout,
                                                     int32_t *__restrict__ vout) {
  __shared__ uint64_t sk[kBuckets - 1];
  __shared__ int32_t sv[kBuckets - 1];
  __shared__ uint32_t c[kBuckets];
  __shared__ uint16_t bk[kBktTile];
  const int64_t n = n_dev ? min(*n_dev, n_max) : n_max;
  const int64_t start = (int64_t)blockIdx.x * kBktTile;
  if (start >= n) return;
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) {
    c[i] = 0;
    if (i < kBuckets - 1) { sk[i] = spk[i]; sv[i] = spv[i]; }
  }
  __syncthreads();
  const int64_t end = min(start + kBktTile, n);
  for (int64_t i = start + threadIdx.x; i < end; i += blockDim.x) {
    const int b = bkt_of(sk, sv, kin[i], vin[i]);
    bk[i - start] = (uint16_t)b;
    atomicAdd(&c[b], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
    if (c[i]) c[i] = atomicAdd(cursor + i, c[i]);
  __syncthreads();
  for (int64_t i = start + threadIdx.x; i < end; i += blockDim.x) {
    const uint32_t pos = atomicAdd(&c[bk[i - start]], 1u);
    kout[pos] = kin[i];
    vout[pos] = vin[i];
  }
}

// one CTA per bucket: sort it by (key, value)
__global__ void __launch_bounds__(256) k_bkt_sort(const uint32_t *__restrict__ boff, uint64_t *__restrict__ kio,
                                                  int32_t *__restrict__ vio) {
  __shared__ uint64_t k_s[kBktCap];
  __shared__ int32_t v_s[kBktCap];
  const int64_t beg = boff[blockIdx.x];
  const int n = (int)(boff[blockIdx.x + 1] - beg);
  if (n <= 1) return;
  if (n <= kBktCap) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      k_s[i] = kio[beg + i];
      v_s[i] = vio[beg + i];
    }
    __syncthreads();
    bitonic_sort(n, [&](int i) -> uint64_t & { return k_s[i]; }, [&](int i) -> int32_t & { return v_s[i]; });
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      kio[beg + i] = k_s[i];
      vio[beg + i] = v_s[i];
    }
    return;
  }
  bitonic_sort(n, [&](int i) -> uint64_t & { return kio[beg + i]; }, [&](int i) -> int32_t & { return vio[beg + i]; });
}

}  // namespace sortk

size_t bucket_sort_workspace_bytes() {
  return 256 * 4 + (sizeof(uint64_t) + sizeof(int32_t)) * sortk::kBuckets + sizeof(uint32_t) * (3 * sortk::kBuckets + 1);
}

int bucket_sort_pairs_u64(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out, int32_t *vals_out,
                          const int64_t *n_dev, int64_t n_max, void *ws, size_t ws_bytes, cudaStream_t st) {
  using namespace sortk;
  if (n_max <= 0) return SALF_OK;
  if (n_max >= (int64_t)UINT32_MAX) return set_error(SALF_EINVAL, "bucket sort: too many keys");
  if (ws_bytes < bucket_sort_workspace_bytes()) return set_error(SALF_EWORKSPACE, "bucket sort workspace too small");
  char *p = (char *)ws;
  uint64_t *spk = (uint64_t *)p;
  p += sizeof(uint64_t) * kBuckets;
  int32_t *spv = (int32_t *)p;
  p += sizeof(int32_t) * kBuckets;
  uint32_t *bcnt = (uint32_t *)p, *boff = bcnt + kBuckets, *cursor = boff + kBuckets + 1;
  cudaMemsetAsync(bcnt, 0, sizeof(uint32_t) * kBuckets, st);
  const unsigned grid = (unsigned)((n_max + kBktTile - 1) / kBktTile);
  k_bkt_splitters<<<1, 1024, 0, st>>>(keys_in, vals_in, n_dev, n_max, spk, spv);
  k_bkt_count<<<grid, 256, 0, st>>>(keys_in, vals_in, n_dev, n_max, spk, spv, bcnt);
  k_bkt_scan<<<1, kBuckets, 0, st>>>(bcnt, boff, cursor);
  k_bkt_scatter<<<grid, 256, 0, st>>>(keys_in, vals_in, n_dev, n_max, spk, spv, cursor, keys_out, vals_out);
  k_bkt_sort<<<kBuckets, 256, 0, st>>>(boff, keys_out, vals_out);
  return check_cuda("bucket_sort_pairs");
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

extern "C" size_t salf_sort_pairs_unique_workspace_bytes(void) { return salf::bucket_sort_workspace_bytes(); }

extern "C" int salf_sort_pairs_unique(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out,
                                      int32_t *vals_out, const int64_t *n_dev, int64_t n_max, void *workspace,
                                      size_t workspace_bytes, void *stream) {
  SALF_TRY {
    return salf::bucket_sort_pairs_u64(keys_in, vals_in, keys_out, vals_out, n_dev, n_max, workspace,
                                       workspace_bytes, (cudaStream_t)stream);
  }
  SALF_CATCH
}
