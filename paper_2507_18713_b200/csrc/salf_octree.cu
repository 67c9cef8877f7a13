// salf_octree.cu -- linear octree build on the device,
// producing the reference's exact DFS layout (octree.py:54-125).
//
// The reference pops its stack LIFO with children pushed 0..7, so internal
// nodes are expanded in preorder with children visited 7, 6, ..., 0, and the
// child block of the r-th expanded node sits at 1 + 8 r.  A node's preorder
// position is therefore the lexicographic order of its path digits (7 - c_i)
// (ancestors first).  Each voxel emits the packed key of every ancestor and of
// itself: key = (sum_i (7 - c_i) << 3 (19 - i)) << 5 | depth.  Sorting the
// unique ancestor keys gives every internal node's rank; parents are found by
// clearing the last digit.  Sorting / unique / searchsorted are library
// primitives (torch/CUB); emission and the node fill are here.
#include "salf_common.cuh"
#include "salf_internal.h"

namespace salf {

constexpr int kKeyDepth = 19;

__device__ __forceinline__ uint64_t path_key(int depth, int D, int ix, int iy, int iz) {
  // digits for levels 1..depth of a cell at depth D (bit D - i of the coords)
  uint64_t k = 0;
  for (int i = 1; i <= depth; ++i) {
    const int sh = D - i;
    const int c = ((ix >> sh) & 1) | (((iy >> sh) & 1) << 1) | (((iz >> sh) & 1) << 2);
    k |= (uint64_t)(7 - c) << (3 * (kKeyDepth - i));
  }
  return (k << 5) | (uint64_t)depth;
}

// ancestors (depth 0..D-1) of every voxel, at base[v] .. base[v] + D - 1
__global__ void k_ancestor_keys(int64_t n, const uint8_t *__restrict__ level, const int32_t *__restrict__ ijk,
                                int root_depth, const int64_t *__restrict__ base, uint64_t *__restrict__ keys,
                                uint64_t *__restrict__ self_key) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int D = root_depth + level[v];
  const int ix = ijk[3 * v], iy = ijk[3 * v + 1], iz = ijk[3 * v + 2];
  for (int k = 0; k < D; ++k) keys[base[v] + k] = path_key(k, D, ix, iy, iz);
  self_key[v] = path_key(D, D, ix, iy, iz);
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t *a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Place node `key` (internal rank r -> word 1 + 8 r, or leaf word) into the
// child slot of its parent.
__device__ __forceinline__ void place(const uint64_t *internal, int64_t n_int, uint64_t key, int32_t word,
                                      int32_t *nodes) {
  const int depth = (int)(key & 31);
  if (depth == 0) {
    nodes[0] = word;
    return;
  }
  const uint64_t path = key >> 5;
  const int shift = 3 * (kKeyDepth - depth);
  const int c = 7 - (int)((path >> shift) & 7);
  const uint64_t parent = ((path & ~((uint64_t)7 << shift)) << 5) | (uint64_t)(depth - 1);
  const int64_t pr = lower_bound_u64(internal, n_int, parent);
  nodes[1 + 8 * pr + c] = word;
}

__global__ void k_fill_internal(int64_t n_int, const uint64_t *__restrict__ internal, int32_t *__restrict__ nodes) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_int) return;
  place(internal, n_int, internal[r], (int32_t)(1 + 8 * r), nodes);
}

__global__ void k_fill_leaves(int64_t n, int64_t n_int, const uint64_t *__restrict__ internal,
                              const uint64_t *__restrict__ self_key, int32_t *__restrict__ nodes,
                              int32_t *__restrict__ contained) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const uint64_t key = self_key[v];
  const int64_t pos = lower_bound_u64(internal, n_int, key);
  if (pos < n_int && internal[pos] == key) {  // a voxel at an internal node's depth
    atomicOr(contained, 1);
    return;
  }
  place(internal, n_int, key, (int32_t)(-(v + 2)), nodes);
}

}  // namespace salf

using namespace salf;

extern "C" int salf_octree_ancestor_keys(int64_t n, const uint8_t *level, const int32_t *ijk, int32_t root_depth,
                                         const int64_t *base, uint64_t *keys, uint64_t *self_key, void *stream) {
  SALF_TRY {
    if (n == 0) return SALF_OK;
    k_ancestor_keys<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(n, level, ijk, root_depth, base,
                                                                                   keys, self_key);
    return check_cuda("salf_octree_ancestor_keys");
  }
  SALF_CATCH
}

extern "C" int salf_octree_fill(int64_t n, int64_t n_internal, const uint64_t *internal, const uint64_t *self_key,
                                int32_t *nodes, int32_t *contained, void *stream) {
  SALF_TRY {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_internal)
      k_fill_internal<<<(unsigned)((n_internal + 255) / 256), 256, 0, st>>>(n_internal, internal, nodes);
    if (n)
      k_fill_leaves<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, n_internal, internal, self_key, nodes, contained);
    return check_cuda("salf_octree_fill");
  }
  SALF_CATCH
}
