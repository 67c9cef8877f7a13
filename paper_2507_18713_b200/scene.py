"""Scene data model and the `salf.v1` container (host side).

Mirrors the reference types the render path consumes -- `SceneBounds`,
`SparseVoxelSet`, `Scene`, `FlatVoxels` (reference scene.py:38-223,
render_raster.py:44-89) and the container loader (container.py:27-175) --
so a scene saved by the reference loads here byte-for-byte.  Field
evaluation lives on the GPU (`csrc/`); this module only holds arrays.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

DENSITY_SDF = "sdf"
DENSITY_RAW = "raw"
FORMAT_VERSION = "salf.v1"
IDENTITY_QUAT = np.array([1.0, 0.0, 0.0, 0.0])

# 121-byte voxel record (reference container.py:27-35)
VOXEL_DTYPE = np.dtype([
    ("level", "u1"), ("ijk", "<i4", (3,)), ("w_s", "<f4", (4,)), ("w_c", "<f4", (3, 3)),
    ("w_sh", "<f4", (3, 4)), ("log_a", "<f4"), ("log_b", "<f4"),
])


class ContainerError(ValueError):
    pass


@dataclass(frozen=True)
class SceneBounds:
    aabb_min: np.ndarray
    aabb_max: np.ndarray
    base_edge: float
    max_levels: int

    def __post_init__(self):
        object.__setattr__(self, "aabb_min", np.asarray(self.aabb_min, dtype=np.float64))
        object.__setattr__(self, "aabb_max", np.asarray(self.aabb_max, dtype=np.float64))
        if not np.all(self.aabb_min < self.aabb_max):
            raise ValueError("aabb_min must be strictly below aabb_max componentwise")
        if self.base_edge <= 0:
            raise ValueError("base_edge must be positive")
        if self.max_levels < 1:
            raise ValueError("max_levels must be at least 1")

    def level_edge(self, level) -> np.ndarray:
        return self.base_edge / np.exp2(np.asarray(level, dtype=np.float64))

    def to_dict(self) -> dict:
        return {"aabb_min": self.aabb_min.tolist(), "aabb_max": self.aabb_max.tolist(),
                "base_edge": self.base_edge, "max_levels": self.max_levels}

    @classmethod
    def from_dict(cls, d: dict) -> "SceneBounds":
        return cls(np.array(d["aabb_min"], np.float64), np.array(d["aabb_max"], np.float64),
                   float(d["base_edge"]), int(d["max_levels"]))


class SparseVoxelSet:
    """Structure-of-arrays voxel store (reference scene.py:82-223)."""

    def __init__(self, bounds: SceneBounds, budget: int = 2_500_000):
        self.bounds = bounds
        self.budget = int(budget)
        self.level = np.zeros(0, np.uint8)
        self.ijk = np.zeros((0, 3), np.int32)
        self.w_s = np.zeros((0, 4))
        self.w_c = np.zeros((0, 3, 3))
        self.w_sh = np.zeros((0, 3, 4))
        self.log_a = np.zeros(0)
        self.log_b = np.zeros(0)
        self.rotation = np.zeros((0, 4))

    @property
    def n(self) -> int:
        return int(self.level.shape[0])

    def __len__(self) -> int:
        return self.n

    def set_arrays(self, level, ijk, w_s, w_c, w_sh, log_a, log_b):
        self.level = np.asarray(level, np.uint8)
        self.ijk = np.asarray(ijk, np.int32).reshape(-1, 3)
        self.w_s = np.asarray(w_s, np.float64).reshape(-1, 4)
        self.w_c = np.asarray(w_c, np.float64).reshape(-1, 3, 3)
        self.w_sh = np.asarray(w_sh, np.float64).reshape(-1, 3, 4)
        self.log_a = np.asarray(log_a, np.float64).reshape(-1)
        self.log_b = np.asarray(log_b, np.float64).reshape(-1)
        self.rotation = np.broadcast_to(IDENTITY_QUAT, (self.n, 4)).copy()
        return self

    def edges(self, idx=None) -> np.ndarray:
        lv = self.level if idx is None else self.level[idx]
        return self.bounds.level_edge(lv)

    def centers(self, idx=None) -> np.ndarray:
        """aabb_min + (ijk + 0.5) * edge, exactly the reference's rounding."""
        lv = self.level if idx is None else self.level[idx]
        cells = self.ijk if idx is None else self.ijk[idx]
        edge = self.bounds.level_edge(lv)
        return self.bounds.aabb_min + (cells.astype(np.float64) + 0.5) * edge[..., None]

    def param_arrays(self) -> dict:
        return {"w_s": self.w_s, "w_c": self.w_c, "w_sh": self.w_sh,
                "log_a": self.log_a, "log_b": self.log_b}


def quat_to_matrix(q) -> np.ndarray:
    """rotations.py:19-33."""
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


def quat_slerp(q0, q1, t) -> np.ndarray:
    """rotations.py:36-50."""
    q0 = np.asarray(q0, dtype=np.float64)
    q1 = np.asarray(q1, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)[..., None]
    dot = np.sum(q0 * q1, axis=-1, keepdims=True)
    q1 = np.where(dot < 0.0, -q1, q1)
    dot = np.abs(dot)
    theta = np.arccos(np.clip(dot, -1.0, 1.0))
    sin_theta = np.sin(theta)
    small = sin_theta < 1e-9
    w0 = np.where(small, 1.0 - t, np.sin((1.0 - t) * theta) / np.where(small, 1.0, sin_theta))
    w1 = np.where(small, t, np.sin(t * theta) / np.where(small, 1.0, sin_theta))
    q = w0 * q0 + w1 * q1
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def quat_multiply(q0, q1) -> np.ndarray:
    """rotations.py:74-88 (Hamilton product, q1 applied first)."""
    q0 = np.asarray(q0, dtype=np.float64)
    q1 = np.asarray(q1, dtype=np.float64)
    w0, x0, y0, z0 = q0[..., 0], q0[..., 1], q0[..., 2], q0[..., 3]
    w1, x1, y1, z1 = q1[..., 0], q1[..., 1], q1[..., 2], q1[..., 3]
    return np.stack([w0 * w1 - x0 * x1 - y0 * y1 - z0 * z1, w0 * x1 + x0 * w1 + y0 * z1 - z0 * y1,
                     w0 * y1 - x0 * z1 + y0 * w1 + z0 * x1, w0 * z1 + x0 * y1 - y0 * x1 + z0 * w1], axis=-1)


@dataclass
class Actor:
    """A rigid dynamic volume with its own voxel set and trajectory (scene.py:290-331)."""

    actor_id: str
    extents: np.ndarray
    voxels: SparseVoxelSet
    times: np.ndarray
    positions: np.ndarray
    quaternions: np.ndarray

    def __post_init__(self):
        self.extents = np.asarray(self.extents, dtype=np.float64)
        self.times = np.asarray(self.times, dtype=np.float64)
        self.positions = np.asarray(self.positions, dtype=np.float64)
        self.quaternions = np.asarray(self.quaternions, dtype=np.float64)
        if self.times.ndim != 1 or len(self.times) == 0:
            raise ValueError("trajectory must contain at least one pose")
        if np.any(np.diff(self.times) <= 0):
            raise ValueError("trajectory timestamps must be strictly increasing")

    def pose_at(self, t):
        """(translation, quaternion) at time(s) t; lerp + slerp (scene.py:316-331)."""
        t = np.asarray(t, dtype=np.float64)
        if np.any(t < self.times[0] - 1e-12) or np.any(t > self.times[-1] + 1e-12):
            raise ValueError("timestamp outside the actor trajectory")
        if len(self.times) == 1:
            shape = t.shape
            return (np.broadcast_to(self.positions[0], shape + (3,)).copy(),
                    np.broadcast_to(self.quaternions[0], shape + (4,)).copy())
        hi = np.clip(np.searchsorted(self.times, t, side="right"), 1, len(self.times) - 1)
        lo = hi - 1
        span = self.times[hi] - self.times[lo]
        frac = np.clip((t - self.times[lo]) / span, 0.0, 1.0)
        pos = self.positions[lo] + frac[..., None] * (self.positions[hi] - self.positions[lo])
        return pos, quat_slerp(self.quaternions[lo], self.quaternions[hi], frac)


def make_actor_bounds(extents, base_edge: float, max_levels: int = 6) -> SceneBounds:
    extents = np.asarray(extents, dtype=np.float64)
    return SceneBounds(-extents / 2.0, extents / 2.0, base_edge, max_levels)


@dataclass
class Scene:
    bounds: SceneBounds
    static: SparseVoxelSet
    actors: list = field(default_factory=list)
    density_mode: str = DENSITY_SDF
    inner_aabb: np.ndarray | None = None

    def __post_init__(self):
        if self.density_mode not in (DENSITY_SDF, DENSITY_RAW):
            raise ValueError(f"unknown density mode {self.density_mode!r}")


@dataclass
class FlatVoxels:
    """Scene voxels flattened into one global-frame list (render_raster.py:44-60)."""

    centers: np.ndarray
    edges: np.ndarray
    rotations: np.ndarray
    w_s: np.ndarray
    w_c: np.ndarray
    w_sh: np.ndarray
    log_a: np.ndarray
    log_b: np.ndarray
    density_mode: str

    @property
    def n(self) -> int:
        return int(self.centers.shape[0])


def flatten_scene(scene: Scene, t_stamp: float = 0.0) -> FlatVoxels:
    """Static voxels plus actor voxels rigidly posed at t_stamp (render_raster.py:63-89)."""
    s = scene.static
    centers, edges, rots = [s.centers()], [s.edges()], [s.rotation]
    w_s, w_c, w_sh, la, lb = [s.w_s], [s.w_c], [s.w_sh], [s.log_a], [s.log_b]
    for actor in scene.actors:
        if actor.voxels.n == 0:
            continue
        pos, quat = actor.pose_at(np.asarray(t_stamp))
        rmat = quat_to_matrix(quat)
        centers.append(actor.voxels.centers() @ rmat.T + pos)
        edges.append(actor.voxels.edges())
        rots.append(quat_multiply(quat, actor.voxels.rotation))
        w_s.append(actor.voxels.w_s)
        w_c.append(actor.voxels.w_c)
        w_sh.append(actor.voxels.w_sh)
        la.append(actor.voxels.log_a)
        lb.append(actor.voxels.log_b)
    return FlatVoxels(centers=np.concatenate(centers), edges=np.concatenate(edges),
                      rotations=np.concatenate(rots), w_s=np.concatenate(w_s),
                      w_c=np.concatenate(w_c), w_sh=np.concatenate(w_sh),
                      log_a=np.concatenate(la), log_b=np.concatenate(lb),
                      density_mode=scene.density_mode)


# -- salf.v1 container ---------------------------------------------------------

def records_from_set(vset: SparseVoxelSet) -> np.ndarray:
    rec = np.zeros(vset.n, dtype=VOXEL_DTYPE)
    rec["level"], rec["ijk"] = vset.level, vset.ijk
    rec["w_s"], rec["w_c"], rec["w_sh"] = vset.w_s, vset.w_c, vset.w_sh
    rec["log_a"], rec["log_b"] = vset.log_a, vset.log_b
    return rec


def set_from_records(rec: np.ndarray, bounds: SceneBounds, budget: int, name: str):
    for f in ("w_s", "w_c", "w_sh", "log_a", "log_b"):
        if not np.all(np.isfinite(rec[f].astype(np.float64))):
            raise ContainerError(f"{name}: non-finite values in field {f!r}")
    v = SparseVoxelSet(bounds, budget)
    if rec.size:
        v.set_arrays(rec["level"], rec["ijk"], rec["w_s"], rec["w_c"], rec["w_sh"],
                     rec["log_a"], rec["log_b"])
    return v


def load_scene(path) -> tuple[Scene, dict]:
    """Load a reference `salf.v1` directory; returns (scene, sensors dict)."""
    path = Path(path)
    meta = json.loads((path / "meta.json").read_text(encoding="utf-8"))
    if meta.get("format") != FORMAT_VERSION:
        raise ContainerError(f"meta.json: unsupported format {meta.get('format')!r}")
    bounds = SceneBounds.from_dict(meta["bounds"])
    count = int(meta["voxel_count"])
    data = (path / "voxels.bin").read_bytes()
    if len(data) != count * VOXEL_DTYPE.itemsize:
        raise ContainerError(f"voxels.bin: size mismatch, expected "
                             f"{count * VOXEL_DTYPE.itemsize} bytes for {count} voxels, "
                             f"got {len(data)}")
    budget = int(meta.get("budget", 2_500_000))
    static = set_from_records(np.frombuffer(data, VOXEL_DTYPE), bounds, budget, "voxels.bin")
    actors = []
    ap = path / "actors.json"
    actors_meta = json.loads(ap.read_text(encoding="utf-8"))["actors"] if ap.exists() else []
    if len(actors_meta) != int(meta.get("actor_count", 0)):
        raise ContainerError("actor_count in meta.json disagrees with actors.json")
    for am in actors_meta:  # container.py:161-175
        a_bounds = make_actor_bounds(np.array(am["extents"]), float(am["base_edge"]), int(am["max_levels"]))
        cnt = int(am["voxel_count"])
        raw = (path / f"actor_{am['id']}.bin").read_bytes()
        if len(raw) != cnt * VOXEL_DTYPE.itemsize:
            raise ContainerError(f"actor_{am['id']}.bin: size mismatch, expected "
                                 f"{cnt * VOXEL_DTYPE.itemsize} bytes for {cnt} voxels, got {len(raw)}")
        vset = set_from_records(np.frombuffer(raw, VOXEL_DTYPE), a_bounds, budget,
                                f"actor_{am['id']}.bin")
        traj = am["trajectory"]
        actors.append(Actor(actor_id=str(am["id"]), extents=np.array(am["extents"], np.float64),
                            voxels=vset, times=np.array([q["t"] for q in traj]),
                            positions=np.array([q["position"] for q in traj]),
                            quaternions=np.array([q["quaternion"] for q in traj])))
    inner = meta.get("inner_aabb")
    scene = Scene(bounds=bounds, static=static, actors=actors,
                  density_mode=meta.get("density_mode", "sdf"),
                  inner_aabb=None if inner is None else np.array(inner, np.float64))
    sensors = {}
    sp = path / "sensors.json"
    if sp.exists():
        sensors = json.loads(sp.read_text(encoding="utf-8")).get("sensors", {})
    return scene, sensors


def save_scene(scene: Scene, path, sensors: dict | None = None) -> None:
    """Byte-compatible with the reference's save_scene (container.py:103-136)."""
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    meta = {
        "format": FORMAT_VERSION, "bounds": scene.bounds.to_dict(),
        "density_mode": scene.density_mode, "voxel_count": scene.static.n,
        "actor_count": len(scene.actors), "budget": scene.static.budget,
        "inner_aabb": None if scene.inner_aabb is None
        else [scene.inner_aabb[0].tolist(), scene.inner_aabb[1].tolist()],
    }
    dump = lambda p, d: p.write_text(json.dumps(d, indent=2, sort_keys=True) + "\n",
                                     encoding="utf-8")
    dump(path / "meta.json", meta)
    (path / "voxels.bin").write_bytes(records_from_set(scene.static).tobytes())
    actors_meta = []
    for a in scene.actors:  # container.py:120-133
        actors_meta.append({
            "id": a.actor_id, "extents": a.extents.tolist(),
            "base_edge": a.voxels.bounds.base_edge, "max_levels": a.voxels.bounds.max_levels,
            "voxel_count": a.voxels.n,
            "trajectory": [{"t": float(t), "position": p.tolist(), "quaternion": q.tolist()}
                           for t, p, q in zip(a.times, a.positions, a.quaternions)],
        })
        (path / f"actor_{a.actor_id}.bin").write_bytes(records_from_set(a.voxels).tobytes())
    dump(path / "actors.json", {"actors": actors_meta})
    if sensors is not None:
        dump(path / "sensors.json", {"sensors": sensors})
