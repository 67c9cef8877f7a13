"""Device training state: Adam (reference optim.py) and the parameter
regularisers (reference losses.py:49-249) on the GPU.

`TrainableScene` keeps the optimisable parameters as one (M, 27) f64 block
(w_s, w_c, w_sh, log_a, log_b -- the gradient buffer's layout) with Adam
moments beside it; after each update the render-side f32 fields and the
density constants of the `DeviceScene` are refreshed in place by a kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceScene
from .octree import OctreeBuffer
from .scene import Scene

EMPTY_QUANTILE = 0.2
LIDAR_OPACITY_DELTA = 0.2


@dataclass
class AdamConfig:
    """optim.py:12-19."""

    lr: float = 0.01
    lr_decay: float = 0.8
    lr_decay_every: int = 800
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def learning_rate(cfg: AdamConfig, step: int) -> float:
    """optim.py:43-45: lr * decay^(step // every)."""
    return cfg.lr * cfg.lr_decay ** (step // cfg.lr_decay_every)


def _block(v) -> np.ndarray:
    m = v.n
    b = np.empty((m, 27), np.float64)
    b[:, 0:4] = v.w_s
    b[:, 4:13] = v.w_c.reshape(m, 9)
    b[:, 13:25] = v.w_sh.reshape(m, 12)
    b[:, 25] = v.log_a
    b[:, 26] = v.log_b
    return b


class TrainableScene:
    """The static owner's parameters (trainer.py:132 lists the static set first;
    actor voxel sets are rendered but not optimised here).  `ds` holds exactly
    the static rows, so `params`, the Adam moments and the refresh kernel all
    cover the same M rows (actors never enter the block)."""

    def __init__(self, scene: Scene, device=None):
        self.scene = scene
        self.ds = DeviceScene.from_static(scene, device=device)
        dev = self.ds.device
        self.params = torch.as_tensor(_block(scene.static), device=dev).contiguous()
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.level = torch.as_tensor(scene.static.level.astype(np.int64), device=dev)
        self.level8 = torch.as_tensor(scene.static.level.astype(np.uint8), device=dev)
        self.ijk = torch.as_tensor(np.ascontiguousarray(scene.static.ijk.astype(np.int32)), device=dev)
        self.step = 0

    @property
    def n(self) -> int:
        return self.ds.n

    def zero_grad(self) -> torch.Tensor:
        return torch.zeros_like(self.params)

    def refresh(self) -> None:
        lib = _lib.load()
        if self.params.shape[0] != self.ds.n:
            raise ValueError(f"parameter block has {self.params.shape[0]} rows, device scene {self.ds.n}")
        _lib.check(lib.salf_scene_refresh(self.params.data_ptr(), self.ds.n, self.ds.prm.data_ptr(),
                                          self.ds.aux.data_ptr(), _lib.stream_ptr()), "refresh")

    def adam_step(self, grad: torch.Tensor, cfg: AdamConfig = AdamConfig()) -> float:
        """optim.py:48-62: one in-place update of every parameter; returns the lr used."""
        lib = _lib.load()
        lr = learning_rate(cfg, self.step)
        self.step += 1
        _lib.check(lib.salf_adam_step(self.params.numel(), self.params.data_ptr(), grad.data_ptr(),
                                      self.m.data_ptr(), self.v.data_ptr(), lr, cfg.beta1, cfg.beta2,
                                      cfg.eps, self.step, _lib.stream_ptr()), "adam_step")
        self.refresh()
        return lr

    def densify(self, grad_acc: torch.Tensor, cfg=None):
        """trainer.py:198-206 on the device: one densify/prune round
        (densify.py:53-94) over the live parameters, Adam moments remapped
        (optim.py:35-40), device scene arrays rebuilt from (level, ijk);
        returns (keep_idx, n_split).  The caller rebuilds the octree
        (`host_voxel_set()` + octree.build_octree_device) and resets grad_acc."""
        from .densify import DensifyConfig, densify_device
        lib = _lib.load()
        cfg = cfg or DensifyConfig()
        b = self.scene.bounds
        r = densify_device(self.params, self.ds.geo, self.level8, self.ijk, grad_acc, cfg, b.max_levels,
                           self.ds.density_mode, self.m, self.v)
        n = int(r["level"].numel())
        dev = self.params.device
        self.params, self.m, self.v = r["params"].contiguous(), r["m"].contiguous(), r["v"].contiguous()
        self.level8, self.ijk = r["level"].contiguous(), r["ijk"].contiguous()
        self.level = self.level8.to(torch.int64)
        geo = torch.empty((max(n, 1), 4), dtype=torch.float64, device=dev)
        aux = torch.empty((max(n, 1), 4), dtype=torch.float64, device=dev)
        prm = torch.zeros((max(n, 1), _lib.PRM_STRIDE), dtype=torch.float32, device=dev)
        lo = np.ascontiguousarray(b.aabb_min, np.float64)
        _lib.check(lib.salf_voxel_geometry(n, self.level8.data_ptr(), self.ijk.data_ptr(), lo.ctypes.data,
                                           float(b.base_edge), self.params.data_ptr(), geo.data_ptr(),
                                           aux.data_ptr(), prm.data_ptr(), _lib.stream_ptr()), "densify")
        self.ds = DeviceScene.from_arrays(geo, aux, prm, n, self.ds.density_mode)
        return r["keep_idx"], r["n_split"]

    def host_voxel_set(self):
        """The current static set on the host (for the octree rebuild / export)."""
        from .scene import SparseVoxelSet
        p = self.to_numpy()
        v = SparseVoxelSet(self.scene.bounds, budget=self.scene.static.budget)
        return v.set_arrays(self.level8.cpu().numpy(), self.ijk.cpu().numpy(), p["w_s"], p["w_c"], p["w_sh"],
                            p["log_a"], p["log_b"])

    def to_numpy(self) -> dict:
        b = self.params.cpu().numpy()
        m = b.shape[0]
        return {"w_s": b[:, 0:4], "w_c": b[:, 4:13].reshape(m, 3, 3),
                "w_sh": b[:, 13:25].reshape(m, 3, 4), "log_a": b[:, 25], "log_b": b[:, 26]}


def _idx(idx, dev) -> torch.Tensor:
    return torch.as_tensor(np.asarray(idx) if not isinstance(idx, torch.Tensor) else idx,
                           dtype=torch.int64, device=dev).contiguous()


def loss_eikonal(ts: TrainableScene, sample_idx, grad: torch.Tensor) -> float:
    """losses.py:49-60: mean | ||W_s[:3]|| - 1 |; gradient added into grad."""
    lib = _lib.load()
    idx = _idx(sample_idx, grad.device)
    if idx.numel() == 0:
        return 0.0
    acc = torch.zeros(1, dtype=torch.float64, device=grad.device)
    _lib.check(lib.salf_loss_eikonal(ts.params.data_ptr(), idx.numel(), idx.data_ptr(), grad.data_ptr(),
                                     acc.data_ptr(), _lib.stream_ptr()), "loss_eikonal")
    return float(acc.item()) / idx.numel()


def loss_empty(ts: TrainableScene, outer_idx, grad: torch.Tensor) -> float:
    """losses.py:210-249: mean opacity of the lowest 20% outer voxels (stable order)."""
    lib = _lib.load()
    idx = _idx(outer_idx, grad.device)
    n = idx.numel()
    if n == 0:
        return 0.0
    mode = _lib.DENSITY[ts.ds.density_mode]
    alpha = torch.empty(n, dtype=torch.float64, device=grad.device)
    _lib.check(lib.salf_center_alpha(ts.params.data_ptr(), ts.ds.geo.data_ptr(), mode, n, idx.data_ptr(),
                                     alpha.data_ptr(), _lib.stream_ptr()), "loss_empty")
    k = max(1, int(np.ceil(EMPTY_QUANTILE * n)))
    order = torch.sort(alpha, stable=True).indices[:k]
    sel = idx[order].contiguous()
    _lib.check(lib.salf_loss_empty_grad(ts.params.data_ptr(), ts.ds.geo.data_ptr(), mode, k, sel.data_ptr(),
                                        grad.data_ptr(), _lib.stream_ptr()), "loss_empty")
    return float(alpha[order].mean().item())


_FACES = [(0, 1), (0, -1), (1, 1), (1, -1), (2, 1), (2, -1)]


def face_pairs(ts: TrainableScene, octree: OctreeBuffer, sample_idx):
    """losses.py:66-92 on the device: (fine, coarse, axis, sign) of each
    adjacent pair with a same-or-coarser neighbour, first occurrence in the
    reference's (face, sample) iteration order."""
    from .octree import query_device
    dev = ts.params.device
    idx = _idx(sample_idx, dev)
    if idx.numel() == 0:
        return None
    level = ts.level
    centers, edges = ts.ds.geo[idx, :3], ts.ds.geo[idx, 3]
    rmin = torch.as_tensor(octree.root_min, device=dev)
    rmax = rmin + octree.root_edge
    cand = []
    n = idx.numel()
    for f, (axis, sign) in enumerate(_FACES):
        probe = centers.clone()
        probe[:, axis] += sign * (0.5 * edges + 1e-6 * edges)
        inside = torch.all((probe >= rmin) & (probe <= rmax), dim=1)
        rows = torch.nonzero(inside, as_tuple=True)[0]
        if rows.numel() == 0:
            continue
        _flag, nb = query_device(octree, probe[rows])
        fine = idx[rows]
        ok = (nb >= 0) & (nb != fine)
        ok &= level[nb.clamp_min(0)] <= level[fine]
        rows, fine, nb = rows[ok], fine[ok], nb[ok]
        same = level[nb] == level[fine]
        lo = torch.where(same, torch.minimum(fine, nb), fine)
        hi = torch.where(same, torch.maximum(fine, nb), nb)
        key = ((lo << 24) | hi) * 3 + axis
        cand.append((f * n + rows, key, fine, nb, torch.full_like(fine, axis),
                     torch.full(fine.shape, float(sign), dtype=torch.float64, device=dev)))
    if not cand:
        return None
    order, key, fine, nb, ax, sg = (torch.cat([c[i] for c in cand]) for i in range(6))
    pos = torch.argsort(order)  # reference iteration order
    key, fine, nb, ax, sg = key[pos], fine[pos], nb[pos], ax[pos], sg[pos]
    # first occurrence of each key (stable sort keeps iteration order within a key)
    ks, perm = torch.sort(key, stable=True)
    first = torch.ones_like(ks, dtype=torch.bool)
    first[1:] = ks[1:] != ks[:-1]
    keep = torch.sort(perm[first]).values
    return fine[keep], nb[keep], ax[keep].to(torch.int32), sg[keep]


def loss_smooth(ts: TrainableScene, octree: OctreeBuffer, sample_idx, grad: torch.Tensor) -> float:
    """losses.py:95-185: mean |SDF difference| + mean |colour difference| at the
    four corners of each shared face (colour viewed along the face normal)."""
    lib = _lib.load()
    pairs = face_pairs(ts, octree, sample_idx)
    if pairs is None or pairs[0].numel() == 0:
        return 0.0
    fine, nb, ax, sg = (x.contiguous() for x in pairs)
    n = fine.numel()
    sums = torch.zeros(2, dtype=torch.float64, device=grad.device)
    _lib.check(lib.salf_loss_smooth(ts.params.data_ptr(), ts.ds.geo.data_ptr(), n, fine.data_ptr(),
                                    nb.data_ptr(), ax.data_ptr(), sg.data_ptr(), grad.data_ptr(),
                                    sums.data_ptr(), _lib.stream_ptr()), "loss_smooth")
    s = sums.cpu().numpy()
    return float(s[0] / (4 * n) + s[1] / (12 * n))


def loss_opacity_lidar(ts: TrainableScene, octree: OctreeBuffer, points, grad: torch.Tensor) -> float:
    """losses.py:188-226: drive opacity at LiDAR points towards 1 over 20 cm."""
    from .octree import query_batch
    lib = _lib.load()
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    if pts.shape[0] == 0:
        return 0.0
    rmax = octree.root_min + octree.root_edge
    pts = pts[np.all((pts >= octree.root_min) & (pts <= rmax), axis=1)]
    if pts.shape[0] == 0:
        return 0.0
    _f, vid, _c, _e = query_batch(octree, pts)
    sel = vid >= 0
    if not np.any(sel):
        return 0.0
    dev = grad.device
    p = torch.as_tensor(pts[sel], device=dev).contiguous()
    v = torch.as_tensor(vid[sel], dtype=torch.int64, device=dev).contiguous()
    acc = torch.zeros(1, dtype=torch.float64, device=dev)
    _lib.check(lib.salf_loss_opacity_lidar(ts.params.data_ptr(), ts.ds.geo.data_ptr(),
                                           _lib.DENSITY[ts.ds.density_mode], v.numel(), p.data_ptr(),
                                           v.data_ptr(), grad.data_ptr(), acc.data_ptr(),
                                           _lib.stream_ptr()), "loss_opacity_lidar")
    return float(acc.item()) / v.numel()
