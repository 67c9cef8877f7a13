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

    def set_params(self, w_s, w_c, w_sh, log_a, log_b) -> "DeviceScene":
        """Refresh the field parameters in place (geometry, rotations and the
        octree stay): the host-side counterpart of salf_scene_refresh, for callers
        that update NumPy parameter arrays between renders (reference optim.py)."""
        n = self.n
        if n == 0:
            return self
        aux = np.empty((n, 2), np.float64)
        aux[:, 0] = np.exp(np.asarray(log_a, np.float64).reshape(n))
        aux[:, 1] = 1.0 / np.exp(np.asarray(log_b, np.float64).reshape(n))
        prm = np.zeros((n, _lib.PRM_STRIDE), np.float32)
        prm[:, 0:4] = np.asarray(w_s).reshape(-1, 4)
        prm[:, 4:13] = np.asarray(w_c).reshape(-1, 9)
        prm[:, 13:25] = np.asarray(w_sh).reshape(-1, 12)
        self.aux[:n, :2].copy_(torch.from_numpy(aux), non_blocking=False)
        self.prm[:n].copy_(torch.from_numpy(prm), non_blocking=False)
        return self

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
        """The composed scene at t (static + posed actor voxels, render_raster.py:63-89)."""
        return cls(flatten_scene(scene, t_stamp), device)

    @classmethod
    def from_static(cls, scene: Scene, device=None) -> "DeviceScene":
        """The static voxel set only (the ray path marches actors in their own
        frames; the trainable parameter block covers the static owner)."""
        from .scene import FlatVoxels
        v = scene.static
        return cls(FlatVoxels(v.centers(), v.edges(), v.rotation, v.w_s, v.w_c, v.w_sh, v.log_a, v.log_b,
                              scene.density_mode), device)

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


_FIELDS = ("w_s", "w_c", "w_sh", "log_a", "log_b")


def load_device_scene(path, device=None) -> DeviceScene:
    """salf.v1 static voxel set straight into HBM (container.py:91-100,
    :130-158): voxels.bin is read once into pinned host
    memory, copied to the device as raw 121-byte records and decoded there
    (`salf_decode_records`) into the render layout plus the (M, 27) f64
    parameter block, level and ijk (attributes `params`, `level`, `ijk`,
    `bounds`, `meta`).  Validation and messages follow the reference loader:
    size mismatch, non-finite fields (first offending field in record
    order), duplicate cells.  Actors, if any, are left to `scene.load_scene`."""
    import json
    from pathlib import Path

    from .scene import FORMAT_VERSION, VOXEL_DTYPE, ContainerError, SceneBounds
    path = Path(path)
    meta = json.loads((path / "meta.json").read_text(encoding="utf-8"))
    if meta.get("format") != FORMAT_VERSION:
        raise ContainerError(f"meta.json: unsupported format {meta.get('format')!r}")
    bounds = SceneBounds.from_dict(meta["bounds"])
    count = int(meta["voxel_count"])
    vb = path / "voxels.bin"
    size = vb.stat().st_size
    rec_size = VOXEL_DTYPE.itemsize
    if size != count * rec_size:
        raise ContainerError(f"voxels.bin: size mismatch, expected {count * rec_size} bytes for {count} voxels, "
                             f"got {size}")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load()
    m = max(count, 1)
    host = torch.empty(((count * rec_size + 15) // 16) * 16 or 16, dtype=torch.uint8).pin_memory()
    with open(vb, "rb") as f:
        f.readinto(host.numpy()[: count * rec_size].data)
    raw = host.to(dev, non_blocking=True)
    level = torch.empty(m, dtype=torch.uint8, device=dev)
    ijk = torch.empty((m, 3), dtype=torch.int32, device=dev)
    params = torch.empty((m, 27), dtype=torch.float64, device=dev)
    geo = torch.empty((m, 4), dtype=torch.float64, device=dev)
    aux = torch.empty((m, 4), dtype=torch.float64, device=dev)
    prm = torch.zeros((m, _lib.PRM_STRIDE), dtype=torch.float32, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    lo = np.ascontiguousarray(bounds.aabb_min, np.float64)
    _lib.check(lib.salf_decode_records(count, raw.data_ptr(), lo.ctypes.data, float(bounds.base_edge),
                                       level.data_ptr(), ijk.data_ptr(), params.data_ptr(), geo.data_ptr(),
                                       aux.data_ptr(), prm.data_ptr(), bad.data_ptr(), _lib.stream_ptr()),
               "load_device_scene")
    flags = int(bad.item())
    for k, name in enumerate(_FIELDS):
        if flags >> k & 1:
            raise ContainerError(f"voxels.bin: non-finite values in field {name!r}")
    if count and int(torch.unique(torch.cat([level[:, None].to(torch.int32), ijk], 1), dim=0).shape[0]) != count:
        raise ContainerError("voxels.bin: duplicate voxel cells")
    ds = DeviceScene.from_arrays(geo, aux, prm, count, meta.get("density_mode", "sdf"))
    ds.params, ds.level, ds.ijk, ds.bounds, ds.meta = params[:count], level[:count], ijk[:count], bounds, meta
    return ds


_IDENTITY_ROT: dict = {}


def _identity_rot(n: int, device) -> torch.Tensor:
    """(n, 9) identity rotations (static rows of a composed scene), grown and cached per device."""
    t = _IDENTITY_ROT.get(str(device))
    if t is None or t.shape[0] < n:
        t = torch.eye(3, dtype=torch.float64, device=device).reshape(1, 9).repeat(max(n, 1), 1)
        _IDENTITY_ROT[str(device)] = t
    return t[:n]


def static_device_scene(scene: Scene, device=None) -> DeviceScene:
    """The static set of `scene` on the device, uploaded once per set: cached on
    the Scene object and keyed by the identity of its arrays (densification
    builds new arrays).  Parameters updated IN PLACE on the host are not seen --
    call `scene.__dict__.pop("_b200_static", None)` (the reference drop-in,
    dropin.py, refreshes them on every call instead)."""
    v = scene.static
    key = tuple(id(a) for a in (v.level, v.ijk, v.rotation, v.w_s, v.w_c, v.w_sh, v.log_a, v.log_b))
    cached = scene.__dict__.get("_b200_static")
    if cached is not None and scene.__dict__.get("_b200_static_key", key) == key:
        return cached
    ds = DeviceScene.from_static(scene, device)
    scene.__dict__["_b200_static"] = ds
    scene.__dict__["_b200_static_key"] = key
    return ds


def composed_device_scene(scene: Scene, t_stamp: float = 0.0, device=None) -> DeviceScene:
    """flatten_scene (render_raster.py:63-89) with the static set resident: only
    the actor voxels posed at t (host NumPy, the reference's own expressions)
    are uploaded and appended behind the static rows; static rows get identity
    rotations so the kernels' per-entry rotation test sees them as axis-aligned."""
    st = static_device_scene(scene, device)
    live = [a for a in scene.actors if a.voxels.n]
    if not live:
        return st
    from .scene import quat_multiply, quat_to_matrix
    centers, edges, rots, ws, wc, wsh, la, lb = [], [], [], [], [], [], [], []
    for actor in live:
        pos, quat = actor.pose_at(np.asarray(t_stamp))
        rmat = quat_to_matrix(quat)
        centers.append(actor.voxels.centers() @ rmat.T + pos)
        edges.append(actor.voxels.edges())
        rots.append(quat_multiply(quat, actor.voxels.rotation))
        ws.append(actor.voxels.w_s)
        wc.append(actor.voxels.w_c)
        wsh.append(actor.voxels.w_sh)
        la.append(actor.voxels.log_a)
        lb.append(actor.voxels.log_b)
    cat = np.concatenate
    da = DeviceScene(FlatVoxels(cat(centers), cat(edges), cat(rots), cat(ws), cat(wc), cat(wsh), cat(la), cat(lb),
                                scene.density_mode), st.device)
    n_s = st.n
    out = DeviceScene.from_arrays(torch.cat([st.geo[:n_s], da.geo[: da.n]]), torch.cat([st.aux[:n_s], da.aux[: da.n]]),
                                  torch.cat([st.prm[:n_s], da.prm[: da.n]]), n_s + da.n, scene.density_mode)
    rot_a = da.rot if da.rot is not None else _identity_rot(da.n, st.device)
    out.rot = torch.cat([_identity_rot(n_s, st.device), rot_a[: da.n]]).contiguous()
    return out
