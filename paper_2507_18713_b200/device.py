"""Device-resident scene: the HBM layout the kernels read.

Per voxel (SoA of AoS blocks, all 16-byte aligned):
  geo  double4  (cx, cy, cz, edge)           32 B  projection, slab tests, local coords
  aux  double4  (a = exp(log_a), 1/b, 2/edge, 0)  32 B  density transfer, local coords
  prm  float[28] w_s[4] w_c[9] w_sh[12] pad[3] 112 B  field parameters (7 x 16-B loads)
Centres, edges and exp(log a|b) are computed on the host with NumPy exactly as
the reference does (scene.py:186-194, :249), so the kernels start from the
reference's own fp64 values.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .scene import FlatVoxels, Scene, flatten_scene


class DeviceScene:
    def __init__(self, flat: FlatVoxels, device=None):
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.n = flat.n
        self.density_mode = flat.density_mode
        geo = np.empty((flat.n, 4), np.float64)
        geo[:, :3] = flat.centers
        geo[:, 3] = flat.edges
        aux = np.zeros((flat.n, 4), np.float64)
        if flat.n:
            aux[:, 0] = np.exp(flat.log_a)
            aux[:, 1] = 1.0 / np.exp(flat.log_b)
            aux[:, 2] = 2.0 / flat.edges  # world_to_local scale (scene.py:209)
        prm = np.zeros((flat.n, _lib.PRM_STRIDE), np.float32)
        prm[:, 0:4] = flat.w_s.reshape(-1, 4)
        prm[:, 4:13] = flat.w_c.reshape(-1, 9)
        prm[:, 13:25] = flat.w_sh.reshape(-1, 12)
        # keep at least one element so data pointers are valid for empty scenes
        pad = lambda a: a if a.shape[0] else np.zeros((1,) + a.shape[1:], a.dtype)
        self.geo = torch.as_tensor(pad(geo), device=self.device).contiguous()
        self.aux = torch.as_tensor(pad(aux), device=self.device).contiguous()
        self.prm = torch.as_tensor(pad(prm), device=self.device).contiguous()
        # voxel rotations (flattened actors): the reference rotates only when
        # not np.allclose(rotations, identity) (render_raster.py:107, :192)
        self.rot = None
        if flat.n and not np.allclose(flat.rotations, np.array([1.0, 0.0, 0.0, 0.0])):
            from .scene import quat_to_matrix
            self.rot = torch.as_tensor(np.ascontiguousarray(quat_to_matrix(flat.rotations).reshape(-1, 9)),
                                       device=self.device)
        self.flat = flat

    @classmethod
    def from_arrays(cls, geo: torch.Tensor, aux: torch.Tensor, prm: torch.Tensor, n: int,
                    density_mode: str) -> "DeviceScene":
        """A static device scene from device arrays already in the HBM layout
        (e.g. rebuilt on the device after densification)."""
        self = cls.__new__(cls)
        self.device = geo.device
        self.n = int(n)
        self.density_mode = density_mode
        self.geo, self.aux, self.prm = geo, aux, prm
        self.rot = None
        self.flat = None
        return self

    @classmethod
    def from_scene(cls, scene: Scene, t_stamp: float = 0.0, device=None) -> "DeviceScene":
        return cls(flatten_scene(scene, t_stamp), device)

    def c_struct(self) -> _lib.SceneT:
        s = _lib.SceneT()
        s.n = self.n
        s.geo, s.aux, s.prm = self.geo.data_ptr(), self.aux.data_ptr(), self.prm.data_ptr()
        s.rot = self.rot.data_ptr() if self.rot is not None else None
        s.density_mode = _lib.DENSITY[self.density_mode]
        return s

    @property
    def nbytes(self) -> int:
        return int(self.geo.nbytes + self.aux.nbytes + self.prm.nbytes)


def as_device_scene(obj, device=None) -> DeviceScene:
    if isinstance(obj, DeviceScene):
        return obj
    if isinstance(obj, FlatVoxels):
        return DeviceScene(obj, device)
    if isinstance(obj, Scene):
        return DeviceScene.from_scene(obj, device=device)
    raise TypeError(f"expected Scene, FlatVoxels or DeviceScene, got {type(obj).__name__}")


def grads_to_dict(grad: torch.Tensor) -> dict:
    """(M, 27) gradient buffer -> the reference's {param: array} layout (backward.py:24)."""
    g = grad.detach().cpu().numpy()
    m = g.shape[0]
    return {"w_s": g[:, 0:4].copy(), "w_c": g[:, 4:13].reshape(m, 3, 3).copy(),
            "w_sh": g[:, 13:25].reshape(m, 3, 4).copy(), "log_a": g[:, 25].copy(),
            "log_b": g[:, 26].copy()}
