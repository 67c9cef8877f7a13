// salf_host.cpp -- host-side pieces of libsalf_b200: last-error buffer, device
// query and the linear-octree build (reference octree.py:54-125).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "salf_internal.h"

namespace salf {
char *error_buffer() {
  static thread_local char buf[1024] = {0};
  return buf;
}
}  // namespace salf

using namespace salf;

extern "C" const char *salf_last_error(void) { return error_buffer(); }

extern "C" int salf_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

// Depth-first build with the reference's LIFO order: a node is numbered when
// its parent's child block is allocated; blocks are allocated in pop order,
// children are pushed 0..7 so octant 7 of the newest block expands first.
// Each stack item owns a contiguous range of a permutation of voxel ids,
// split into 8 octant ranges by a stable counting sort.
extern "C" int salf_octree_build_host(int64_t n, const uint8_t *level, const int32_t *ijk, int32_t root_depth,
                                      int32_t *nodes, int64_t capacity, int64_t *n_nodes, int32_t *max_depth) {
  SALF_TRY {
    std::vector<int32_t> out;
    out.push_back(-1);
    if (n == 0) {
      *n_nodes = 1;
      *max_depth = root_depth;
      if (nodes && capacity >= 1) nodes[0] = -1;
      return SALF_OK;
    }
    if (n > INT32_MAX - 2) return set_error(SALF_EINVAL, "too many voxels for 32-bit octree words");
    std::vector<int32_t> perm(n), tmp(n);
    int maxlev = 0;
    for (int64_t i = 0; i < n; ++i) {
      perm[i] = (int32_t)i;
      if (level[i] > maxlev) maxlev = level[i];
    }
    struct Item { int64_t node; int32_t dep; int64_t b, e; };
    std::vector<Item> stack;
    stack.push_back({0, 0, 0, n});
    while (!stack.empty()) {
      Item it = stack.back();
      stack.pop_back();
      const int64_t cnt = it.e - it.b;
      if (cnt == 0) continue;  // empty (-1, -1)
      bool at = false;
      for (int64_t k = it.b; k < it.e; ++k)
        if (root_depth + (int)level[perm[k]] == it.dep) { at = true; break; }
      if (at) {
        if (cnt > 1) return set_error(SALF_EINVAL, "stored voxel contains another stored voxel");
        out[it.node] = -(perm[it.b] + 2);
        continue;
      }
      const int64_t off = (int64_t)out.size();
      if (off + 8 > INT32_MAX) return set_error(SALF_EINVAL, "octree too large for 32-bit node words");
      out[it.node] = (int32_t)off;
      out.insert(out.end(), 8, -1);
      int64_t bucket[9] = {0};
      auto child_of = [&](int32_t v) {
        const int sh = root_depth + (int)level[v] - it.dep - 1;
        const int bx = (ijk[3 * (int64_t)v] >> sh) & 1, by = (ijk[3 * (int64_t)v + 1] >> sh) & 1,
                  bz = (ijk[3 * (int64_t)v + 2] >> sh) & 1;
        return bx + 2 * by + 4 * bz;
      };
      for (int64_t k = it.b; k < it.e; ++k) ++bucket[child_of(perm[k]) + 1];
      for (int c = 0; c < 8; ++c) bucket[c + 1] += bucket[c];
      int64_t pos[8];
      for (int c = 0; c < 8; ++c) pos[c] = it.b + bucket[c];
      for (int64_t k = it.b; k < it.e; ++k) tmp[pos[child_of(perm[k])]++] = perm[k];
      memcpy(&perm[it.b], &tmp[it.b], sizeof(int32_t) * cnt);
      for (int c = 0; c < 8; ++c) stack.push_back({off + c, it.dep + 1, it.b + bucket[c], it.b + bucket[c + 1]});
    }
    *n_nodes = (int64_t)out.size();
    *max_depth = root_depth + maxlev;
    if (nodes) {
      if (capacity < (int64_t)out.size()) return set_error(SALF_EWORKSPACE, "node capacity too small");
      memcpy(nodes, out.data(), sizeof(int32_t) * out.size());
    }
    return SALF_OK;
  }
  SALF_CATCH
}
