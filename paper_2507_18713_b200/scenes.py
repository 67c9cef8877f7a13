"""Benchmark scene construction (synthetic inputs, host side).

The benchmark scenes are the reference's own pipeline output:
`salf make-synthetic --spec standard` followed by
`salf init --margin-up 1 --margin-down 1 --margin-lateral 1 --max-levels 10
--base-edge B`.  The point cloud and trajectory of the first
step are committed under `tests/golden/`; this module re-runs the second step
(reference densify.py:121-229, `init_multiscale`) vectorised, drawing the
random field initialisation in exactly the reference's RNG order, so the
resulting `salf.v1` bytes are identical to the reference CLI's (pinned by the
SHA-256 digests in `tests/golden/scene_digests.json`).

It also builds the two regimes the survey asks to report:
  * "init"    -- the scene as initialised (nearly transparent outer shells);
  * "surface" -- fields baked from the analytic primitives of the standard
    synthetic spec (a = 50, b = 0.02, DC colour = logit(albedo)/C0), then
    pruned by the reference rule (centre opacity < 0.005, densify.py:39-46).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .scene import (DENSITY_SDF, Scene, SceneBounds, SparseVoxelSet, load_scene, records_from_set,
                    save_scene, set_from_records)

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
DATA = REPO / "data"

INIT_A_OCCUPIED = 2.0
INIT_A_EMPTY = 0.1
INIT_B = 0.2
_INNER_LEVEL = 4
BASE_EDGES = {"S20k": 0.3, "S1M": 0.07, "S2M": 0.055}


def read_ply(path) -> np.ndarray:
    """ASCII PLY points, parsed with Python float() like the reference (imaging.py:87-100)."""
    lines = Path(path).read_text(encoding="ascii").splitlines()
    n, body = 0, 0
    for i, line in enumerate(lines):
        if line.startswith("element vertex"):
            n = int(line.split()[-1])
        if line.strip() == "end_header":
            body = i + 1
            break
    pts = [tuple(float(v) for v in row.split()[:3]) for row in lines[body:body + n]]
    return np.array(pts, dtype=np.float64).reshape(n, 3)


def _cell_keys(cells: np.ndarray) -> np.ndarray:
    c = cells.astype(np.int64) + (1 << 20)
    return (c[:, 0] << 42) | (c[:, 1] << 21) | c[:, 2]


def _occupied(points, origin, edge) -> np.ndarray:
    if points.shape[0] == 0:
        return np.zeros(0, np.int64)
    return np.unique(_cell_keys(np.floor((points - origin) / edge).astype(np.int64)))


def init_multiscale(points, traj_positions, box_extents, base_edge=1.0, margin_up=10.0,
                    margin_down=5.0, margin_lateral=40.0, max_levels=10, budget=2_500_000,
                    seed=0) -> Scene:
    """Vectorised restatement of densify.init_multiscale (reference densify.py:121-229)."""
    points = np.atleast_2d(np.asarray(points, np.float64)).reshape(-1, 3)
    traj = np.atleast_2d(np.asarray(traj_positions, np.float64))
    half = np.asarray(box_extents, np.float64) / 2.0
    lo = traj.min(axis=0) - half
    hi = traj.max(axis=0) + half
    lo -= np.array([margin_lateral, margin_lateral, margin_down])
    hi += np.array([margin_lateral, margin_lateral, margin_up])
    quant = 4.0 * base_edge
    dims = hi - lo
    snapped = np.ceil(dims / quant - 1e-9) * quant
    pad = (snapped - dims) / 2.0
    inner_lo = lo - pad
    inner_hi = inner_lo + snapped
    d = snapped
    aabb_min = inner_lo - 7.5 * d
    aabb_max = aabb_min + 16.0 * d
    bounds = SceneBounds(aabb_min, aabb_max, base_edge=16.0 * base_edge, max_levels=max_levels)
    boxes = [(inner_lo, inner_hi)]
    for l in range(1, 5):
        c = (inner_lo + inner_hi) / 2.0
        boxes.append((c - 2.0 ** (l - 1) * d, c + 2.0 ** (l - 1) * d))
    rng = np.random.default_rng(seed)
    parts = []

    def add(level, cells, occ_keys):
        m = cells.shape[0]
        if m == 0:
            return
        occ = np.isin(_cell_keys(cells), occ_keys) if occ_keys.size else np.zeros(m, bool)
        a = np.where(occ, INIT_A_OCCUPIED, INIT_A_EMPTY)
        # draw order = SparseVoxelSet.add_voxels (reference scene.py:145-149)
        w_s = rng.uniform(-1.0 / np.sqrt(3.0), 1.0 / np.sqrt(3.0), size=(m, 4))
        w_c = rng.uniform(-1.0 / np.sqrt(3.0), 1.0 / np.sqrt(3.0), size=(m, 3, 3))
        w_sh = rng.uniform(-0.5, 0.5, size=(m, 3, 4))
        parts.append((np.full(m, level, np.uint8), cells.astype(np.int32), w_s, w_c, w_sh,
                      np.log(a), np.log(np.full(m, INIT_B))))

    def grid(i0, i1):
        g = np.meshgrid(*[np.arange(i0[k], i1[k]) for k in range(3)], indexing="ij")
        return np.stack([x.ravel() for x in g], axis=1)

    for l in range(1, 5):
        level = _INNER_LEVEL - l
        edge = bounds.level_edge(level)
        (blo, bhi), (plo, phi) = boxes[l], boxes[l - 1]
        cells = grid(np.round((blo - aabb_min) / edge).astype(np.int64),
                     np.round((bhi - aabb_min) / edge).astype(np.int64))
        centers = aabb_min + (cells + 0.5) * edge
        cells = cells[~np.all((centers > plo) & (centers < phi), axis=1)]
        add(level, cells, _occupied(points, aabb_min, edge))
    edge_in = bounds.level_edge(_INNER_LEVEL)
    inner = grid(np.round((inner_lo - aabb_min) / edge_in).astype(np.int64),
                 np.round((inner_hi - aabb_min) / edge_in).astype(np.int64))
    in_box = np.all((points >= inner_lo) & (points <= inner_hi), axis=1) \
        if points.shape[0] else np.zeros(0, bool)
    pin = points[in_box]
    if pin.shape[0] == 0:
        add(_INNER_LEVEL, inner, np.zeros(0, np.int64))
    else:
        kept = inner[np.isin(_cell_keys(inner), _occupied(pin, aabb_min, edge_in))]
        offs = np.array([[x, y, z] for z in (0, 1) for y in (0, 1) for x in (0, 1)])
        child = (kept[:, None, :] * 2 + offs[None]).reshape(-1, 3)
        add(_INNER_LEVEL + 1, child, _occupied(pin, aabb_min, bounds.level_edge(_INNER_LEVEL + 1)))
    vset = SparseVoxelSet(bounds, budget)
    cat = [np.concatenate([p[i] for p in parts]) for i in range(7)]
    if cat[0].shape[0] > budget:
        raise ValueError(f"voxel budget exceeded: {cat[0].shape[0]} > {budget}")
    vset.set_arrays(*cat)
    return Scene(bounds=bounds, static=vset, density_mode=DENSITY_SDF,
                 inner_aabb=np.stack([inner_lo, inner_hi]))


def standard_inputs():
    points = read_ply(GOLDEN / "standard_points.ply")
    traj = json.loads((GOLDEN / "standard_trajectory.json").read_text(encoding="utf-8"))
    pos = np.array([p["position"] for p in traj["poses"]], np.float64)
    ext = np.array(traj.get("box_extents", [1.0, 1.0, 1.0]), np.float64)
    return points, pos, ext


def f32_roundtrip(scene: Scene) -> Scene:
    """Params as a salf.v1 load sees them (f32 on disk, f64 in memory)."""
    v = scene.static
    rec = records_from_set(v)
    out = set_from_records(rec, scene.bounds, v.budget, "memory")
    return Scene(bounds=scene.bounds, static=out, density_mode=scene.density_mode,
                 inner_aabb=scene.inner_aabb)


def make_init_scene(name: str) -> Scene:
    """S20k / S1M / S2M exactly as `salf init` writes them and `load_scene` reads
    them back."""
    points, pos, ext = standard_inputs()
    return f32_roundtrip(init_multiscale(points, pos, ext, base_edge=BASE_EDGES[name],
                                         margin_up=1.0, margin_down=1.0, margin_lateral=1.0,
                                         max_levels=10))


# -- surface regime --------------------------------------------------------------

SH_C0 = 0.2820947918
_STANDARD_BOXES = [((-1.2, -1.4, 0.0), (-0.2, -0.4, 1.0), (0.85, 0.15, 0.1)),
                   ((0.3, -0.3, 0.0), (1.3, 0.9, 0.7), (0.1, 0.6, 0.85)),
                   ((-0.9, 0.5, 0.0), (-0.1, 1.3, 1.4), (0.9, 0.75, 0.1))]
_STANDARD_SPHERES = [((0.9, -1.0, 0.35), 0.35, (0.2, 0.8, 0.25))]
_GROUND = (0.0, (-2.5, 2.5), (-2.5, 2.5), (0.45, 0.42, 0.4))


def _primitive_sdf(p):
    """Signed distance (positive inside = occupied) and albedo of the nearest primitive
    of the standard synthetic spec (reference synthetic.py:76-95)."""
    best = np.full(p.shape[0], -np.inf)
    alb = np.zeros((p.shape[0], 3))
    cands = []
    for bmin, bmax, col in _STANDARD_BOXES:
        bmin, bmax = np.array(bmin), np.array(bmax)
        c, h = (bmin + bmax) / 2, (bmax - bmin) / 2
        q = np.abs(p - c) - h
        outside = np.linalg.norm(np.maximum(q, 0), axis=1) + np.minimum(q.max(axis=1), 0)
        cands.append((-outside, col))
    for c, r, col in _STANDARD_SPHERES:
        cands.append((r - np.linalg.norm(p - np.array(c), axis=1), col))
    z, xr, yr, col = _GROUND
    q = np.stack([np.maximum(xr[0] - p[:, 0], p[:, 0] - xr[1]),
                  np.maximum(yr[0] - p[:, 1], p[:, 1] - yr[1]), p[:, 2] - z], axis=1)
    cands.append((-(np.linalg.norm(np.maximum(q, 0), axis=1) + np.minimum(q.max(axis=1), 0)), col))
    for s, col in cands:
        better = s > best
        best = np.where(better, s, best)
        alb[better] = col
    return best, alb


def bake_surface(scene: Scene, a=50.0, b=0.02, prune=0.005) -> Scene:
    """'Surface' regime: analytic bake then the reference prune rule (densify.py:39-46)."""
    v = scene.static
    c = v.centers()
    e = v.edges()
    s, alb = _primitive_sdf(c)
    eps = 1e-3
    grad = np.stack([(_primitive_sdf(c + eps * np.eye(3)[k])[0] - _primitive_sdf(c - eps * np.eye(3)[k])[0])
                     / (2 * eps) for k in range(3)], axis=1)
    w_s = np.concatenate([grad * (e[:, None] / 2.0), s[:, None]], axis=1)
    w_sh = np.zeros((v.n, 3, 4))
    al = np.clip(alb, 1e-3, 1 - 1e-3)
    w_sh[:, :, 0] = np.log(al / (1 - al)) / SH_C0
    w_c = np.zeros((v.n, 3, 3))
    log_a = np.full(v.n, np.log(a))
    log_b = np.full(v.n, np.log(b))
    # centre opacity with delta = edge (densify.py:39-46: sigma at centre, x = 0 -> s = bias)
    sig = 0.5 * a * (1.0 + np.sign(s) * (1.0 - np.exp(-np.abs(s) / b)))
    op = -np.expm1(-sig * e)
    keep = op >= prune
    out = SparseVoxelSet(scene.bounds, v.budget).set_arrays(
        v.level[keep], v.ijk[keep], w_s[keep].astype(np.float32), w_c[keep].astype(np.float32),
        w_sh[keep].astype(np.float32), log_a[keep].astype(np.float32),
        log_b[keep].astype(np.float32))
    return Scene(bounds=scene.bounds, static=out, density_mode=DENSITY_SDF,
                 inner_aabb=scene.inner_aabb)


def _bake_fields(centers, edges, a, b):
    s, alb = _primitive_sdf(centers)
    eps = 1e-4
    grad = np.stack([(_primitive_sdf(centers + eps * np.eye(3)[k])[0]
                      - _primitive_sdf(centers - eps * np.eye(3)[k])[0]) / (2 * eps) for k in range(3)],
                    axis=1)
    n = centers.shape[0]
    w_s = np.concatenate([grad * (edges[:, None] / 2.0), s[:, None]], axis=1)
    w_sh = np.zeros((n, 3, 4))
    al = np.clip(alb, 1e-3, 1 - 1e-3)
    w_sh[:, :, 0] = np.log(al / (1 - al)) / SH_C0
    return w_s, np.zeros((n, 3, 3)), w_sh, np.full(n, np.log(a)), np.full(n, np.log(b))


def make_dense_surface_scene(name: str = "S1M", level: int = 7, a: float = 400.0,
                             b: float = 0.004, band: float = 1.15) -> Scene:
    """'surface-dense' regime: a trained-like scene of ~1M voxels.

    Starting from the inner region of the reference-pipeline scene `name` at
    its base level, cells whose cube can touch a primitive surface
    (|sdf(centre)| <= half-diagonal, widened to a `band` x half-diagonal shell
    at the finest level) are subdivided down to `level` (octree aligned, like
    the reference's densification, densify.py:53-94); the surviving cells get
    fields baked from the analytic primitives.  S1M -> ~1.0M voxels."""
    base = make_init_scene(name)
    bounds = base.bounds
    lo, hi = base.inner_aabb
    e0 = bounds.level_edge(_INNER_LEVEL)
    i0 = np.round((lo - bounds.aabb_min) / e0).astype(np.int64)
    i1 = np.round((hi - bounds.aabb_min) / e0).astype(np.int64)
    g = np.meshgrid(*[np.arange(i0[k], i1[k]) for k in range(3)], indexing="ij")
    cells = np.stack([x.ravel() for x in g], axis=1)
    offs = np.array([[x, y, z] for z in (0, 1) for y in (0, 1) for x in (0, 1)])
    lev = _INNER_LEVEL
    extra = (band - 1.0) * 0.8661 * bounds.level_edge(level)
    while True:
        e = bounds.level_edge(lev)
        c = bounds.aabb_min + (cells + 0.5) * e
        sd, _ = _primitive_sdf(c)
        cells = cells[np.abs(sd) <= 0.8661 * e + extra]
        if lev == level:
            break
        cells = (cells[:, None, :] * 2 + offs[None]).reshape(-1, 3)
        lev += 1
    e = bounds.level_edge(level)
    centers = bounds.aabb_min + (cells + 0.5) * e
    fields = _bake_fields(centers, np.full(cells.shape[0], e), a, b)
    vset = SparseVoxelSet(bounds, max(base.static.budget, cells.shape[0]))
    vset.set_arrays(np.full(cells.shape[0], level, np.uint8), cells.astype(np.int32), *fields)
    return f32_roundtrip(Scene(bounds=bounds, static=vset, density_mode=DENSITY_SDF,
                               inner_aabb=base.inner_aabb))


def get_scene(name: str, regime: str = "init", cache: bool = True) -> Scene:
    """Load (or build and cache under data/) a benchmark scene as salf.v1."""
    d = DATA / f"{name}_{regime}"
    if cache and (d / "meta.json").exists():
        return load_scene(d)[0]
    if regime == "surface-dense":
        scene = make_dense_surface_scene(name)
    else:
        scene = make_init_scene(name)
        if regime == "surface":
            scene = bake_surface(scene)
        elif regime != "init":
            raise ValueError(f"unknown regime {regime!r}")
    if cache:
        # atomic publish: concurrent builders (spawned CPU-baseline workers)
        # never observe a half-written container
        import os
        import shutil
        tmp = d.parent / f".{d.name}.tmp{os.getpid()}"
        save_scene(scene, tmp)
        try:
            os.rename(tmp, d)
        except OSError:
            shutil.rmtree(tmp, ignore_errors=True)  # another process published first
        return load_scene(d)[0]  # f32 round trip, identical to what the reference loads
    return scene


def with_moving_actors(scene: Scene, seed: int = 7, n_actors: int = 2, cell: float = 0.1) -> Scene:
    """The scene plus `n_actors` rigid car-sized actors (4.4 x 1.8 x 1.5 m box of
    `cell`-edge voxels, ~12k each, init-regime random fields) driving through the
    C3 LiDAR's view over t in [0, 1] s with a yaw change -- the dynamic-actor
    workload of the bench (reference scene.py:290-331 Actor, render_ray.py:161-239)."""
    from .scene import Actor, make_actor_bounds
    rng = np.random.default_rng(seed)
    extents = np.array([4.4, 1.8, 1.5])
    dims = np.round(extents / cell).astype(int)
    actors = []
    for k in range(n_actors):
        b = make_actor_bounds(extents, cell, 1)
        cells = np.stack(np.meshgrid(*[np.arange(m) for m in dims], indexing="ij"), -1).reshape(-1, 3)
        v = SparseVoxelSet(b, budget=cells.shape[0] + 10)
        n = cells.shape[0]
        v.set_arrays(np.zeros(n, np.uint8), cells.astype(np.int32),
                     rng.uniform(-1, 1, (n, 4)) / np.sqrt(3.0), rng.uniform(-1, 1, (n, 3, 3)) / np.sqrt(3.0),
                     rng.uniform(-0.5, 0.5, (n, 3, 4)), np.full(n, np.log(2.0)), np.full(n, np.log(0.2)))
        y = 3.0 if k % 2 == 0 else -3.5
        p0, p1 = np.array([6.0 + 4 * k, y, 0.8]), np.array([16.0 + 4 * k, y, 0.8])
        yaw0, yaw1 = 0.0, 0.3 * (1 if k % 2 == 0 else -1)
        q = lambda a: np.array([np.cos(a / 2), 0.0, 0.0, np.sin(a / 2)])
        actors.append(Actor(f"car{k}", extents, v, np.array([0.0, 1.0]), np.stack([p0, p1]),
                            np.stack([q(yaw0), q(yaw1)])))
    return Scene(bounds=scene.bounds, static=scene.static, actors=actors, density_mode=scene.density_mode,
                 inner_aabb=scene.inner_aabb)
