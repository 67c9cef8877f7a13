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
    """Static voxels as a flat list (render_raster.py:63-89).

    Dynamic actors are a later §8(f) row; a scene carrying live actors is
    rejected rather than silently rendered without them."""
    if any(getattr(a, "voxels", None) is not None and a.voxels.n for a in scene.actors):
        raise NotImplementedError("dynamic actors are not supported by the B200 path yet")
    s = scene.static
    return FlatVoxels(centers=s.centers(), edges=s.edges(), rotations=s.rotation,
                      w_s=s.w_s, w_c=s.w_c, w_sh=s.w_sh, log_a=s.log_a, log_b=s.log_b,
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
    static = set_from_records(np.frombuffer(data, VOXEL_DTYPE), bounds,
                              int(meta.get("budget", 2_500_000)), "voxels.bin")
    if int(meta.get("actor_count", 0)):
        raise NotImplementedError("dynamic actors are not supported by the B200 path yet")
    inner = meta.get("inner_aabb")
    scene = Scene(bounds=bounds, static=static, density_mode=meta.get("density_mode", "sdf"),
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
    dump(path / "actors.json", {"actors": []})
    if sensors is not None:
        dump(path / "sensors.json", {"sensors": sensors})
