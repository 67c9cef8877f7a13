"""Linear octree + epsilon-marching -- drop-in for reference octree.py.

`build_octree` (octree.py:54-125) runs natively on the host
(`salf_octree_build_host`) and reproduces the reference's depth-first node
numbering exactly; the node table is uploaded once as 32-bit words
(word >= 0: internal node, children at word..word+7; -1: empty;
<= -2: leaf holding voxel -word-2).  `query_batch` and `march_batch` run on
the GPU with the reference's fp64 operation order, so hit lists are
bit-identical.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .scene import SceneBounds, SparseVoxelSet

EPS_ADVANCE = 1e-4
MIN_EDGE_FACTOR = 64
_MAX_ROUNDS = 200_000


# depth of the descent jump table (csrc salf_octree_jump_build; 0 disables it)
JUMP_LEVELS = int(os.environ.get("SALF_OCT_JUMP", "7"))


@dataclass
class OctreeBuffer:
    nodes: torch.Tensor  # (n_nodes,) int32 words on the device
    root_min: np.ndarray
    root_edge: float
    max_depth: int
    jump: torch.Tensor | None = None  # descent jump table (built on first use)
    jump_levels: int = 0  # its depth; -1: disabled for this tree

    @property
    def n_nodes(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def nodes_id(self) -> np.ndarray:
        w = self.nodes.cpu().numpy().astype(np.int64)
        return np.where(w >= 0, w, np.where(w == -1, -1, -w - 2))

    @property
    def nodes_leaf(self) -> np.ndarray:
        w = self.nodes.cpu().numpy()
        return np.where(w >= 0, 0, np.where(w == -1, -1, 1)).astype(np.int8)

    def c_struct(self) -> _lib.OctreeT:
        t = self._base_struct()
        if self.jump is None and self.jump_levels == 0 and JUMP_LEVELS > 0 and self.nodes.is_cuda \
                and self.max_depth > 0:
            # no deeper than the tree, and no larger (8^K words) than ~8x its node table
            k = min(JUMP_LEVELS, int(self.max_depth), int(np.log2(max(self.n_nodes, 1)) // 3) + 1)
            self._build_jump(t, k)
        if self.jump is not None:
            t.jump_levels = self.jump_levels
            t.jump = self.jump.data_ptr()
        return t

    def with_jump(self, levels: int) -> "OctreeBuffer":
        """A view of this tree whose descents use a jump table of depth
        `levels` (0: none, every query walks from the root)."""
        t = replace(self, jump=None, jump_levels=-1 if levels <= 0 else 0)
        if levels > 0:
            t._build_jump(t._base_struct(), min(int(levels), max(int(self.max_depth), 1)))
        return t

    def _base_struct(self) -> _lib.OctreeT:
        t = _lib.OctreeT()
        t.n_nodes = self.n_nodes
        t.nodes = self.nodes.data_ptr()
        t.root_min[:] = [float(v) for v in self.root_min]
        t.root_edge = float(self.root_edge)
        t.max_depth = int(self.max_depth)
        return t

    def _build_jump(self, t: _lib.OctreeT, levels: int) -> None:
        """Device jump table: the descent starts at depth `levels` (same
        words, corners and edges as the level-by-level walk)."""
        lib = _lib.load()
        nbytes = lib.salf_octree_jump_bytes(levels)
        jump = torch.empty(nbytes, dtype=torch.uint8, device=self.nodes.device)
        _lib.check(lib.salf_octree_jump_build(_lib.ref(t), levels, jump.data_ptr(), _lib.stream_ptr()),
                   "octree jump table")
        self.jump, self.jump_levels = jump, levels


def compute_child_index(p_local) -> np.ndarray:
    """octree.py:47-51."""
    bits = (np.asarray(p_local, np.float64) >= 0.5).astype(np.int64)
    return bits[..., 0] + 2 * (bits[..., 1] + 2 * bits[..., 2])


def build_octree(voxels: SparseVoxelSet, bounds: SceneBounds | None = None, device=None) -> OctreeBuffer:
    """Depth-first linear octree (octree.py:54-125); same errors and messages."""
    lib = _lib.load(require_cuda=False)
    if bounds is None:
        bounds = voxels.bounds
    extent = bounds.aabb_max - bounds.aabb_min
    m = max(0, int(np.ceil(np.log2(max(extent.max(), 1e-300) / bounds.base_edge) - 1e-12)))
    root_edge = bounds.base_edge * 2.0 ** m
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = voxels.n
    if n:
        level = voxels.level.astype(np.int64)
        cells = voxels.ijk.astype(np.int64)
        edges = voxels.edges()
        if edges.min() < MIN_EDGE_FACTOR * EPS_ADVANCE:
            raise ValueError(f"voxel edge {edges.min():.3g} m below the marching floor "
                             f"{MIN_EDGE_FACTOR * EPS_ADVANCE:.3g} m")
        keys = (level << 54) ^ (cells[:, 0] << 36) ^ (cells[:, 1] << 18) ^ cells[:, 2]
        if len(np.unique(keys)) != n:
            raise ValueError("duplicate voxel cells in the set")
        centers = voxels.centers()
        if np.any(centers < bounds.aabb_min) or np.any(centers > bounds.aabb_max):
            raise ValueError("voxel outside scene bounds")
    lv = np.ascontiguousarray(voxels.level.astype(np.uint8)) if n else np.zeros(1, np.uint8)
    ijk = np.ascontiguousarray(voxels.ijk.astype(np.int32)) if n else np.zeros((1, 3), np.int32)
    n_nodes = _lib.C.c_int64(0)
    depth = _lib.C.c_int32(0)
    _lib.check(lib.salf_octree_build_host(n, lv.ctypes.data, ijk.ctypes.data, m, None, 0,
                                          _lib.ref(n_nodes), _lib.ref(depth)), "build_octree")
    nodes = np.empty(n_nodes.value, np.int32)
    _lib.check(lib.salf_octree_build_host(n, lv.ctypes.data, ijk.ctypes.data, m, nodes.ctypes.data,
                                          nodes.shape[0], _lib.ref(n_nodes), _lib.ref(depth)),
               "build_octree")
    return OctreeBuffer(torch.as_tensor(nodes, device=dev), bounds.aabb_min.copy(), root_edge,
                        int(depth.value))


def build_octree_device(voxels: SparseVoxelSet, bounds: SceneBounds | None = None, device=None) -> OctreeBuffer:
    """build_octree on the GPU: the reference's DFS layout
    from sorted preorder keys (csrc/salf_octree.cu); same validation as
    build_octree."""
    if bounds is None:
        bounds = voxels.bounds
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if voxels.n and int(voxels.level.astype(np.int64).max()) + _root_depth(bounds) > 19:
        return build_octree(voxels, bounds, device)  # deeper than the packed key: host build
    lv = torch.as_tensor(voxels.level.astype(np.uint8), device=dev)
    ijk = torch.as_tensor(np.ascontiguousarray(voxels.ijk.astype(np.int32)).reshape(-1, 3), device=dev)
    return build_octree_from_device(lv, ijk, bounds)


def _root_depth(bounds: SceneBounds) -> int:
    extent = bounds.aabb_max - bounds.aabb_min
    return max(0, int(np.ceil(np.log2(max(extent.max(), 1e-300) / bounds.base_edge) - 1e-12)))


def build_octree_from_device(level: torch.Tensor, ijk: torch.Tensor, bounds: SceneBounds) -> OctreeBuffer:
    """build_octree (octree.py:54-125) from device-resident (level u8, ijk i32)
    -- e.g. a scene decoded on the device or a densified set -- with the
    reference's validation (octree.py:66-90) done on the device."""
    lib = _lib.load()
    dev = level.device
    m = _root_depth(bounds)
    root_edge = bounds.base_edge * 2.0 ** m
    n = int(level.numel())
    if n == 0:
        return OctreeBuffer(torch.full((1,), -1, dtype=torch.int32, device=dev), bounds.aabb_min.copy(),
                            root_edge, m)
    lv64 = level.to(torch.int64)
    max_level = int(lv64.max().item())
    if m + max_level > 19:
        raise ValueError("octree deeper than the packed device key; use build_octree")
    edges = bounds.base_edge / torch.exp2(lv64.to(torch.float64))
    if float(edges.min().item()) < MIN_EDGE_FACTOR * EPS_ADVANCE:
        raise ValueError(f"voxel edge {float(edges.min().item()):.3g} m below the marching floor "
                         f"{MIN_EDGE_FACTOR * EPS_ADVANCE:.3g} m")
    cells = ijk.to(torch.int64)
    keys = (lv64 << 54) ^ (cells[:, 0] << 36) ^ (cells[:, 1] << 18) ^ cells[:, 2]
    if int(torch.unique(keys).numel()) != n:
        raise ValueError("duplicate voxel cells in the set")
    lo = torch.as_tensor(bounds.aabb_min, device=dev)
    hi = torch.as_tensor(bounds.aabb_max, device=dev)
    centers = lo + (cells.to(torch.float64) + 0.5) * edges[:, None]
    if bool(((centers < lo) | (centers > hi)).any()):
        raise ValueError("voxel outside scene bounds")
    lv = level.to(torch.uint8).contiguous()
    ijk32 = ijk.to(torch.int32).contiguous()
    depth = m + lv64
    base = torch.cumsum(depth, 0) - depth
    total = int(depth.sum().item())
    akeys = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    skeys = torch.empty(n, dtype=torch.int64, device=dev)
    s = _lib.stream_ptr()
    _lib.check(lib.salf_octree_ancestor_keys(n, lv.data_ptr(), ijk32.data_ptr(), m, base.data_ptr(),
                                             akeys.data_ptr(), skeys.data_ptr(), s), "build_octree")
    # keys < 2^62, so signed int64 order == unsigned order
    internal = torch.unique(akeys[:total]) if total else akeys[:0]
    n_int = int(internal.numel())
    nodes = torch.full((1 + 8 * n_int,), -1, dtype=torch.int32, device=dev)
    contained = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.salf_octree_fill(n, n_int, internal.data_ptr(), skeys.data_ptr(), nodes.data_ptr(),
                                    contained.data_ptr(), s), "build_octree")
    if int(contained.item()):
        raise ValueError("stored voxel contains another stored voxel")
    return OctreeBuffer(nodes, bounds.aabb_min.copy(), root_edge, m + max_level)


def dump_table(buffer: OctreeBuffer) -> str:
    """octree.py:128-133."""
    ids, leaf = buffer.nodes_id, buffer.nodes_leaf
    lines = ["index is_leaf id_or_offset"]
    lines += [f"{i} {int(leaf[i])} {int(ids[i])}" for i in range(buffer.n_nodes)]
    return "\n".join(lines) + "\n"


def query_batch(buffer: OctreeBuffer, p):
    """octree.py:136-166 -> (is_leaf i8, voxel_id i64, node_min (n,3), node_edge), NumPy."""
    lib = _lib.load()
    dev = buffer.nodes.device
    pts = _lib.as_f64(np.atleast_2d(np.asarray(p, np.float64)) if not isinstance(p, torch.Tensor) else p,
                      dev).reshape(-1, 3)
    n = pts.shape[0]
    flag = torch.empty(n, dtype=torch.int8, device=dev)
    vid = torch.empty(n, dtype=torch.int64, device=dev)
    corner = torch.empty((n, 3), dtype=torch.float64, device=dev)
    edge = torch.empty(n, dtype=torch.float64, device=dev)
    outside = torch.zeros(1, dtype=torch.int32, device=dev)
    t = buffer.c_struct()
    _lib.check(lib.salf_octree_query(_lib.ref(t), n, pts.data_ptr(), flag.data_ptr(), vid.data_ptr(),
                                     corner.data_ptr(), edge.data_ptr(), outside.data_ptr(),
                                     _lib.stream_ptr()), "query_batch")
    if int(outside.item()):
        raise ValueError("query point outside the octree root cube")
    return flag.cpu().numpy(), vid.cpu().numpy(), corner.cpu().numpy(), edge.cpu().numpy()


def query_device(buffer: OctreeBuffer, pts: torch.Tensor):
    """query_batch on device tensors -> (flag int8, vid int64) CUDA tensors (no raise)."""
    lib = _lib.load()
    pts = pts.to(torch.float64).contiguous().reshape(-1, 3)
    n = pts.shape[0]
    dev = pts.device
    flag = torch.empty(n, dtype=torch.int8, device=dev)
    vid = torch.empty(n, dtype=torch.int64, device=dev)
    corner = torch.empty((n, 3), dtype=torch.float64, device=dev)
    edge = torch.empty(n, dtype=torch.float64, device=dev)
    outside = torch.zeros(1, dtype=torch.int32, device=dev)
    if n:
        t = buffer.c_struct()
        _lib.check(lib.salf_octree_query(_lib.ref(t), n, pts.data_ptr(), flag.data_ptr(), vid.data_ptr(),
                                         corner.data_ptr(), edge.data_ptr(), outside.data_ptr(),
                                         _lib.stream_ptr()), "query")
    return flag, vid


def query(buffer: OctreeBuffer, p) -> int:
    return int(query_batch(buffer, np.asarray(p, np.float64)[None, :])[1][0])


def _check_unit(dirs: torch.Tensor) -> None:
    if dirs.shape[0] and bool((torch.linalg.norm(dirs, dim=1) - 1.0).abs().gt(1e-6).any()):
        raise ValueError("ray directions must be unit norm")


def march_segments(buffer: OctreeBuffer, origins, dirs, t_max=np.inf, scene=None,
                   stop_threshold: float = 0.99, early_stop: bool = False):
    """Hit list in per-ray march order as device tensors (ray, vid, t0, t1)."""
    lib = _lib.load()
    dev = buffer.nodes.device
    o = _lib.as_f64(origins, dev).reshape(-1, 3)
    d = _lib.as_f64(dirs, dev).reshape(-1, 3)
    _check_unit(d)
    n = o.shape[0]
    tm = _lib.as_f64(np.broadcast_to(np.asarray(t_max, np.float64), (n,)) if not isinstance(t_max, torch.Tensor)
                     else t_max, dev).reshape(n)
    t = buffer.c_struct()
    sc = scene.c_struct() if scene is not None else None
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    s = _lib.stream_ptr()
    scp = _lib.ref(sc) if sc is not None else None
    _lib.check(lib.salf_march(_lib.ref(t), n, o.data_ptr(), d.data_ptr(), tm.data_ptr(), scp,
                              float(stop_threshold), int(early_stop), counts.data_ptr(), None, None,
                              None, None, status.data_ptr(), s), "march_batch")
    if n and bool((status & 1).any()):
        raise RuntimeError("octree marching failed to terminate")
    if n and bool((status & 2).any()):
        raise ValueError("query point outside the octree root cube")
    starts = torch.cumsum(counts, 0) - counts
    total = int(counts.sum().item()) if n else 0
    vid = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    t0 = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    t1 = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    if total:
        _lib.check(lib.salf_march(_lib.ref(t), n, o.data_ptr(), d.data_ptr(), tm.data_ptr(), scp,
                                  float(stop_threshold), int(early_stop), counts.data_ptr(),
                                  starts.data_ptr(), vid.data_ptr(), t0.data_ptr(), t1.data_ptr(),
                                  None, s), "march_batch")
    ray = torch.repeat_interleave(torch.arange(n, device=dev), counts)
    return ray, vid[:total], t0[:total], t1[:total]


def march_batch(buffer: OctreeBuffer, origins, dirs, t_max=np.inf):
    """octree.py:276-295: (ray, vid, t0, t1) NumPy arrays sorted by (ray, t0), stable."""
    ray, vid, t0, t1 = (x.cpu().numpy() for x in march_segments(buffer, origins, dirs, t_max))
    order = np.lexsort((t0, ray))
    return ray[order], vid[order], t0[order], t1[order]


def march(buffer: OctreeBuffer, origin, direction, t_max=np.inf):
    """octree.py:298-302: single ray -> [(voxel_id, t_entry, t_exit)]."""
    ray, vid, t0, t1 = march_batch(buffer, np.asarray(origin, np.float64)[None, :],
                                   np.asarray(direction, np.float64)[None, :], t_max)
    return list(zip(vid.tolist(), t0.tolist(), t1.tolist()))
