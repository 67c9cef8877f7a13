// salf_sort.cuh -- hand-written device sort / compaction / scan primitives for
// the tile binning (reference render_raster.py:163-181: the row-major
// expansion and `lexsort((vox, z[vox], tile))`).  No CUB, no host sync: every
// element count can live on the device (the producing kernel writes it), so a
// frame's binning is one stream of launches.
//
// * radix_sort_pairs: stable LSD radix sort of (key, int32 value), 8-bit
//   digits, one "onesweep" kernel per digit (decoupled look-back across CTAs
//   in ticket order, warp-level match_any ranking inside a CTA -> stable).
// * Look-back status words carry the flag in the top bits of the same word as
//   the value, so one relaxed 32/64-bit load sees both.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace salf {
namespace sortk {

constexpr int kBlock = 256;  // threads per sort CTA (== radix)
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 16;   // keys per thread
constexpr int kTile = kBlock * kItems;  // keys per CTA
constexpr int kRadix = 256;
constexpr int kScanItems = 8;  // scan / select CTA: 2048 elements
constexpr int kScanTile = kBlock * kScanItems;

constexpr uint32_t kFlagA32 = 1u << 30, kFlagP32 = 2u << 30, kVal32 = (1u << 30) - 1;
constexpr uint64_t kFlagA64 = 1ull << 62, kFlagP64 = 2ull << 62, kVal64 = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back for one 64-bit running sum (one thread): publishes this
// tile's aggregate, walks back to the first inclusive prefix, publishes its own
// inclusive prefix and returns the exclusive prefix.
__device__ __forceinline__ uint64_t lookback64(uint64_t *status, uint32_t tile, uint64_t agg) {
  if (tile == 0) {
    st_relaxed(status, kFlagP64 | agg);
    return 0;
  }
  st_relaxed(status + tile, kFlagA64 | agg);
  uint64_t excl = 0;
  for (int64_t p = (int64_t)tile - 1;; --p) {
    uint64_t v;
    do { v = ld_relaxed(status + p); } while ((v & ~kVal64) == 0);
    excl += v & kVal64;
    if (v & kFlagP64) break;
  }
  st_relaxed(status + tile, kFlagP64 | (excl + agg));
  return excl;
}

// block-wide exclusive scan of one int64 per thread (kBlock threads)
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *s_warp /* kWarps + 1 */, int64_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < kWarps; ++i) {
      const int64_t c = s_warp[i];
      s_warp[i] = run;
      run += c;
    }
    s_warp[kWarps] = run;
  }
  __syncthreads();
  total = s_warp[kWarps];
  return s_warp[w] + x - v;
}

}  // namespace sortk

// Workspace bytes of radix_sort_pairs for at most n_max keys over [begin_bit, end_bit).
size_t radix_sort_workspace_bytes(int64_t n_max, int key_bytes, int begin_bit, int end_bit);

// Stable sort of (keys_in, vals_in)[0, n) into (keys_out, vals_out) by bits
// [begin_bit, end_bit) of the key (higher bits must be zero).  n = min(*n_dev,
// n_max) read on the device (n_dev may be null: n = n_max).  The inputs are not
// modified.  n_max < 2^30.
int radix_sort_pairs_u32(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out, int32_t *vals_out,
                         const int64_t *n_dev, int64_t n_max, int begin_bit, int end_bit, void *ws, size_t ws_bytes,
                         cudaStream_t st);
int radix_sort_pairs_u64(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out, int32_t *vals_out,
                         const int64_t *n_dev, int64_t n_max, int begin_bit, int end_bit, void *ws, size_t ws_bytes,
                         cudaStream_t st);

// Splitter bucket sort of (u64 key, int32 value) pairs unique as pairs, ordered by
// (key, value) -- for value-ordered input the same permutation as the stable
// radix sort of the keys.  Workspace: bucket_sort_workspace_bytes() (independent of n).
size_t bucket_sort_workspace_bytes();
int bucket_sort_pairs_u64(const uint64_t *keys_in, const int32_t *vals_in, uint64_t *keys_out, int32_t *vals_out,
                          const int64_t *n_dev, int64_t n_max, void *ws, size_t ws_bytes, cudaStream_t st);

}  // namespace salf
