"""Sensor models and GPU ray generation (reference sensors.py, rotations.py).

`CameraModel` / `LidarModel` / `RayBatch` keep the reference's fields and
validation messages (sensors.py:29-98); ray generation runs on the GPU
(`salf_camera_rays` / `salf_lidar_rays`) and returns a `RayBatch` whose arrays
are CUDA float64 tensors.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib

PINHOLE = "pinhole"
FISHEYE = "fisheye_equidistant"
EQUIRECT = "equirect"
IDENTITY_QUAT = np.array([1.0, 0.0, 0.0, 0.0])


def quat_to_matrix(q) -> np.ndarray:
    """rotations.py:19-33 (host; the same expression the reference evaluates)."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    m = np.empty(q.shape[:-1] + (3, 3))
    m[..., 0, 0] = 1 - 2 * (y * y + z * z)
    m[..., 0, 1] = 2 * (x * y - w * z)
    m[..., 0, 2] = 2 * (x * z + w * y)
    m[..., 1, 0] = 2 * (x * y + w * z)
    m[..., 1, 1] = 1 - 2 * (x * x + z * z)
    m[..., 1, 2] = 2 * (y * z - w * x)
    m[..., 2, 0] = 2 * (x * z - w * y)
    m[..., 2, 1] = 2 * (y * z + w * x)
    m[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return m


def look_at_quaternion(position, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """Camera-to-world quaternion, +z toward target, +y down (synthetic.py:164-197)."""
    position = np.asarray(position, np.float64)
    fwd = np.asarray(target, np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    nr = np.linalg.norm(right)
    right = np.array([1.0, 0.0, 0.0]) if nr < 1e-9 else right / nr
    down = np.cross(fwd, right)
    m = np.stack([right, down, fwd], axis=1)
    t = np.trace(m)
    if t > 0:
        s = np.sqrt(t + 1.0) * 2
        return np.array([0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s,
                         (m[1, 0] - m[0, 1]) / s])
    i = int(np.argmax(np.diag(m)))
    j, k = (i + 1) % 3, (i + 2) % 3
    s = np.sqrt(max(m[i, i] - m[j, j] - m[k, k] + 1.0, 1e-12)) * 2
    q = np.zeros(4)
    q[0] = (m[k, j] - m[j, k]) / s
    q[1 + i] = 0.25 * s
    q[1 + j] = (m[j, i] + m[i, j]) / s
    q[1 + k] = (m[k, i] + m[i, k]) / s
    return q / np.linalg.norm(q)


@dataclass
class RayBatch:
    origins: torch.Tensor  # (N, 3) f64
    dirs: torch.Tensor  # (N, 3) f64, unit
    t_stamps: torch.Tensor  # (N,)
    keys: torch.Tensor  # (N, 2) int64
    valid: torch.Tensor  # (N,) bool
    shape: tuple
    # directions generated here (cos/sin / normalised), i.e. unit by
    # construction: the renderers skip their host-synchronising norm check
    generated: bool = False

    @property
    def n(self) -> int:
        return int(self.origins.shape[0])


@dataclass
class CameraModel:
    kind: str
    width: int
    height: int
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    distortion: tuple = (0.0, 0.0, 0.0, 0.0)
    position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    quaternion: np.ndarray = field(default_factory=lambda: IDENTITY_QUAT.copy())
    readout_duration: float = 0.0
    linear_velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    angular_velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if self.kind not in (PINHOLE, FISHEYE, EQUIRECT):
            raise ValueError(f"unknown camera kind {self.kind!r}")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be at least 1")
        if self.readout_duration < 0:
            raise ValueError("readout_duration must be non-negative")
        self.position = np.asarray(self.position, np.float64)
        self.quaternion = np.asarray(self.quaternion, np.float64)
        self.linear_velocity = np.asarray(self.linear_velocity, np.float64)
        self.angular_velocity = np.asarray(self.angular_velocity, np.float64)

    def rotation_matrix(self) -> np.ndarray:
        return quat_to_matrix(self.quaternion)

    def c_struct(self, t0: float = 0.0, rolling: bool = True) -> _lib.CameraT:
        c = _lib.CameraT()
        c.kind = _lib.KINDS[self.kind]
        c.width, c.height = int(self.width), int(self.height)
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.k[:] = [float(v) for v in self.distortion]
        c.position[:] = self.position.tolist()
        c.rot[:] = self.rotation_matrix().ravel().tolist()
        c.readout_duration = float(self.readout_duration) if rolling else 0.0
        c.linear_velocity[:] = self.linear_velocity.tolist()
        c.angular_velocity[:] = self.angular_velocity.tolist()
        c.t0 = float(t0)
        return c

    @classmethod
    def from_dict(cls, d: dict) -> "CameraModel":
        """container.py sensor_from_dict for cameras."""
        return cls(kind=d["kind"], width=int(d["width"]), height=int(d["height"]),
                   fx=float(d.get("fx", 0.0)), fy=float(d.get("fy", 0.0)),
                   cx=float(d.get("cx", 0.0)), cy=float(d.get("cy", 0.0)),
                   distortion=tuple(d.get("distortion", (0.0, 0.0, 0.0, 0.0))),
                   position=np.array(d.get("position", [0, 0, 0]), np.float64),
                   quaternion=np.array(d.get("quaternion", [1, 0, 0, 0]), np.float64),
                   readout_duration=float(d.get("readout_duration", 0.0)),
                   linear_velocity=np.array(d.get("linear_velocity", [0, 0, 0]), np.float64),
                   angular_velocity=np.array(d.get("angular_velocity", [0, 0, 0]), np.float64))


@dataclass
class LidarModel:
    beam_elevations: np.ndarray
    azimuth_start: float = 0.0
    azimuth_end: float = 2.0 * np.pi
    steps: int = 360
    scan_period: float = 0.1
    position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    quaternion: np.ndarray = field(default_factory=lambda: IDENTITY_QUAT.copy())
    linear_velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    angular_velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if self.steps < 1:
            raise ValueError("steps must be at least 1")
        if self.scan_period <= 0:
            raise ValueError("scan_period must be positive")
        self.beam_elevations = np.atleast_1d(np.asarray(self.beam_elevations, np.float64))
        self.position = np.asarray(self.position, np.float64)
        self.quaternion = np.asarray(self.quaternion, np.float64)
        self.linear_velocity = np.asarray(self.linear_velocity, np.float64)
        self.angular_velocity = np.asarray(self.angular_velocity, np.float64)

    def c_struct(self, t0: float = 0.0) -> _lib.LidarT:
        s = _lib.LidarT()
        s.n_beams, s.steps = int(self.beam_elevations.shape[0]), int(self.steps)
        s.azimuth_start, s.azimuth_end = float(self.azimuth_start), float(self.azimuth_end)
        s.scan_period = float(self.scan_period)
        s.position[:] = self.position.tolist()
        s.rot[:] = quat_to_matrix(self.quaternion).ravel().tolist()
        s.linear_velocity[:] = self.linear_velocity.tolist()
        s.angular_velocity[:] = self.angular_velocity.tolist()
        s.t0 = float(t0)
        return s


def _device(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _camera_batch(cam: CameraModel, t0: float, rolling: bool, device=None, stream=None) -> RayBatch:
    lib = _lib.load()
    dev = _device(device)
    h, w = cam.height, cam.width
    n = h * w
    o = torch.empty((n, 3), dtype=torch.float64, device=dev)
    d = torch.empty((n, 3), dtype=torch.float64, device=dev)
    ts = torch.empty(n, dtype=torch.float64, device=dev)
    valid = torch.empty(n, dtype=torch.bool, device=dev)  # the kernel writes 0 / 1 bytes
    keys = torch.empty((n, 2), dtype=torch.int64, device=dev)
    cs = cam.c_struct(t0, rolling)
    with torch.cuda.device(dev):  # one launch: rays, time stamps, valid mask and keys
        _lib.check(lib.salf_camera_batch(_lib.ref(cs), o.data_ptr(), d.data_ptr(), ts.data_ptr(),
                                         valid.data_ptr(), keys.data_ptr(), _lib.stream_ptr(stream)), "camera_rays")
    return RayBatch(o, d, ts, keys, valid, (h, w), generated=True)


def gen_camera_rays(cam: CameraModel, t0: float = 0.0, device=None) -> RayBatch:
    """Global-shutter batch, one ray per pixel, row-major (sensors.py:129-161)."""
    return _camera_batch(cam, t0, rolling=False, device=device)


def camera_rays(cam: CameraModel, t0: float = 0.0, device=None) -> RayBatch:
    """Generation plus the configured rolling shutter (sensors.py:185-190), fused."""
    return _camera_batch(cam, t0, rolling=cam.readout_duration > 0.0, device=device)


def apply_rolling_shutter(batch: RayBatch, cam: CameraModel) -> RayBatch:
    """sensors.py:164-182 for a batch produced by gen_camera_rays of the same camera."""
    if cam.readout_duration == 0.0:
        return batch
    t0 = float(batch.t_stamps[0].item())
    out = camera_rays(cam, t0, device=batch.origins.device)
    return replace(batch, origins=out.origins, dirs=out.dirs, t_stamps=out.t_stamps)


def gen_lidar_rays(lidar: LidarModel, t0: float = 0.0, device=None) -> RayBatch:
    """Spinning LiDAR batch, beam-major (sensors.py:193-232)."""
    lib = _lib.load()
    dev = _device(device)
    nb, steps = lidar.beam_elevations.shape[0], lidar.steps
    n = nb * steps
    o = torch.empty((n, 3), dtype=torch.float64, device=dev)
    d = torch.empty((n, 3), dtype=torch.float64, device=dev)
    ts = torch.empty(n, dtype=torch.float64, device=dev)
    keys = torch.empty((n, 2), dtype=torch.int64, device=dev)
    valid = torch.empty(n, dtype=torch.bool, device=dev)
    el = _elevations_on(lidar.beam_elevations, dev)
    ls = lidar.c_struct(t0)
    with torch.cuda.device(dev):  # one launch: rays, time stamps, keys and the valid mask
        _lib.check(lib.salf_lidar_batch(_lib.ref(ls), el.data_ptr(), o.data_ptr(), d.data_ptr(), ts.data_ptr(),
                                        keys.data_ptr(), valid.data_ptr(), _lib.stream_ptr()), "lidar_rays")
    return RayBatch(o, d, ts, keys, valid, (nb, steps), generated=True)


_ELEV_CACHE: dict = {}


def _elevations_on(elev, dev) -> torch.Tensor:
    """Device copy of a LiDAR's beam elevations, cached by value: a sweep per
    frame does not pay a synchronous host-to-device copy each time."""
    a = np.ascontiguousarray(np.asarray(elev, np.float64))
    key = (str(dev), a.tobytes())
    t = _ELEV_CACHE.get(key)
    if t is None:
        if len(_ELEV_CACHE) > 64:
            _ELEV_CACHE.clear()
        t = torch.as_tensor(a, device=dev)
        _ELEV_CACHE[key] = t
    return t


def sensor_from_dict(d: dict):
    if d.get("type") == "lidar":
        return LidarModel(beam_elevations=np.array(d["beam_elevations"], np.float64),
                          azimuth_start=float(d.get("azimuth_start", 0.0)),
                          azimuth_end=float(d.get("azimuth_end", 2 * np.pi)),
                          steps=int(d["steps"]), scan_period=float(d.get("scan_period", 0.1)),
                          position=np.array(d.get("position", [0, 0, 0]), np.float64),
                          quaternion=np.array(d.get("quaternion", [1, 0, 0, 0]), np.float64),
                          linear_velocity=np.array(d.get("linear_velocity", [0, 0, 0]), np.float64),
                          angular_velocity=np.array(d.get("angular_velocity", [0, 0, 0]), np.float64))
    return CameraModel.from_dict(d)
