"""GPU: the reference's own hot-path pins for the rasterizer (
reference test_render_raster.py), restated on this package's API:
projection at the centre pixel (:36-45), behind-camera culling (:47-51), the
projected rect width f/9.5 (:53-59), a small voxel in a single tile (:70-78),
per-tile order equal to the global (z, index) sort (:80-91), separated voxels
raster == ray (:125-138), tile size as scheduling only (:140-150) and the
raster-vs-ray mean L1 bound on a random scene (:160-166); and for the ray
path (test_render_ray.py) time invariance of a static scene (:128-135) and
the early-stopped static march against the merged path (:137-154)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _identity_cam(width=128, height=128, f=100.0, cx=64.0, cy=64.0, position=(0, 0, 0)):
    from paper_2507_18713_b200.sensors import CameraModel
    return CameraModel(kind="pinhole", width=width, height=height, fx=f, fy=f, cx=cx, cy=cy,
                       position=np.asarray(position, np.float64), quaternion=np.array([1.0, 0, 0, 0]))


def _cam_at(position, target, width=64, height=64, f=80.0):
    from paper_2507_18713_b200.sensors import CameraModel, look_at_quaternion
    return CameraModel(kind="pinhole", width=width, height=height, fx=f, fy=f, cx=width / 2.0, cy=height / 2.0,
                       position=np.asarray(position, np.float64), quaternion=look_at_quaternion(position, target))


def _voxels(bounds, levels, cells, rng, a=2.0, b=0.2):
    """Voxels with the reference's init distribution (scene.py:143-149)."""
    from paper_2507_18713_b200.scene import SparseVoxelSet
    n = len(cells)
    v = SparseVoxelSet(bounds, budget=max(n, 1) * 4)
    v.set_arrays(levels, cells, rng.uniform(-1 / np.sqrt(3), 1 / np.sqrt(3), (n, 4)),
                 rng.uniform(-1 / np.sqrt(3), 1 / np.sqrt(3), (n, 3, 3)), rng.uniform(-0.5, 0.5, (n, 3, 4)),
                 np.full(n, np.log(a)), np.full(n, np.log(b)))
    return v


def _one_voxel_scene(center, edge=1.0):
    from paper_2507_18713_b200.scene import Scene, SceneBounds
    b = SceneBounds(np.asarray(center, float) - 8.5 * edge, np.asarray(center, float) + 7.5 * edge, edge, 2)
    v = _voxels(b, [0], [[8, 8, 8]], np.random.default_rng(0))
    np.testing.assert_allclose(v.centers()[0], center)
    return Scene(bounds=b, static=v)


def _random_scene(seed, n, levels=3, extent=8.0, a_range=(0.5, 4.0)):
    """Non-overlapping multi-level random scene: distinct cells of the finest
    grid, each kept at a random level whose parent cell is still free."""
    from paper_2507_18713_b200.scene import Scene, SceneBounds
    from paper_2507_18713_b200.scenes import f32_roundtrip
    rng = np.random.default_rng(seed)
    b = SceneBounds(np.zeros(3), np.full(3, extent), 1.0, levels)
    taken = set()
    lv, ijk = [], []
    while len(lv) < n:
        level = int(rng.integers(0, levels))
        res = int(extent) << level
        c = tuple(int(x) for x in rng.integers(0, res, 3))
        # the cell's footprint at the finest level must be free
        s = 1 << (levels - 1 - level)
        fine = [(c[0] * s + i, c[1] * s + j, c[2] * s + k) for i in range(s) for j in range(s) for k in range(s)]
        if any(f in taken for f in fine):
            continue
        taken.update(fine)
        lv.append(level)
        ijk.append(c)
    v = _voxels(b, lv, ijk, rng)
    v.log_a = np.log(rng.uniform(*a_range, n))
    return f32_roundtrip(Scene(bounds=b, static=v))


def test_center_projection_and_depth():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    flat = flatten_scene(_one_voxel_scene([0, 0, 10.0]))
    rmin, rmax, zc, culled = RR.project_voxels(flat, _identity_cam())
    assert zc[0] == pytest.approx(10.0)
    assert not culled[0]
    np.testing.assert_allclose(0.5 * (rmin[0] + rmax[0]), [64.0, 64.0])


def test_behind_camera_culled():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    _rmin, _rmax, _z, culled = RR.project_voxels(flatten_scene(_one_voxel_scene([0, 0, -10.0])), _identity_cam())
    assert culled[0]


def test_projected_rect_width():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    rmin, rmax, _z, _c = RR.project_voxels(flatten_scene(_one_voxel_scene([0, 0, 10.0])), _identity_cam())
    width = rmax[0, 0] - rmin[0, 0]
    assert width >= 100.0 / 10.5
    assert width == pytest.approx(100.0 / 9.5, rel=1e-6)


def test_small_voxel_single_tile():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import Scene, SceneBounds, flatten_scene
    b = SceneBounds([-8, -8, 0], [8, 8, 16], 1.0, 2)
    v = _voxels(b, [1], [[16, 16, 20]], np.random.default_rng(0))  # 0.5 m at z = 10
    bins = RR.cull_and_bin(flatten_scene(Scene(bounds=b, static=v)), _identity_cam(f=60.0))
    assert np.flatnonzero(np.diff(bins.offsets)).size == 1


def test_per_tile_order_matches_global_sort():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    flat = flatten_scene(_random_scene(61, 400))
    cam = _cam_at([12.0, 12.0, 6.0], [4.0, 4.0, 2.0])
    bins = RR.cull_and_bin(flat, cam)
    _rmin, _rmax, z, _c = RR.project_voxels(flat, cam)
    order = np.lexsort((np.arange(flat.n), z))
    rank = np.empty(flat.n, np.int64)
    rank[order] = np.arange(flat.n)
    assert bins.entries.size > 0
    for t in range(len(bins.offsets) - 1):
        e = bins.entries[bins.offsets[t]:bins.offsets[t + 1]]
        assert np.all(np.diff(rank[e]) > 0)


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_separated_voxels_raster_equals_ray(exact):
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.scene import Scene, SceneBounds, flatten_scene
    from paper_2507_18713_b200.scenes import f32_roundtrip
    from paper_2507_18713_b200.sensors import camera_rays
    b = SceneBounds([-8, -8, 0], [8, 8, 16], 1.0, 2)
    cells = [[7 + i % 3, 7 + (i // 3) % 3, 3 + 2 * i] for i in range(5)]
    scene = f32_roundtrip(Scene(bounds=b, static=_voxels(b, [0] * 5, cells, np.random.default_rng(62), a=3.0)))
    cam = _identity_cam(width=64, height=64, f=60.0, cx=32.0, cy=32.0, position=(0.0, 0.0, 0.2))
    fb = RR.rasterize(flatten_scene(scene), cam, exact_color=exact)
    color, _op, _d = RY.render_rays_image(scene, RY.build_scene_octrees(scene), camera_rays(cam),
                                          exact_color=exact)
    tol = 1e-6 if exact else 5e-6  # fp32 output planes; the fp32 field path adds a few ulps
    assert float(np.max(np.abs(fb.color.cpu().numpy() - np.asarray(color.cpu() if hasattr(color, "cpu")
                                                                      else color)))) < tol


def test_tile_size_is_scheduling_only():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    flat = flatten_scene(_random_scene(63, 200))
    cam = _cam_at([12.0, 10.0, 6.0], [4.0, 4.0, 2.0], width=48, height=48, f=50.0)
    for exact in (True, False):
        a = RR.rasterize(flat, cam, tile=16, exact_color=exact)
        b = RR.rasterize(flat, cam, tile=1, exact_color=exact)
        assert torch.equal(a.color, b.color) and torch.equal(a.opacity, b.opacity)
        na = torch.isnan(a.depth)
        assert torch.equal(na, torch.isnan(b.depth)) and torch.equal(a.depth[~na], b.depth[~na])


def test_raster_ray_mean_l1_small():
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.sensors import camera_rays
    scene = _random_scene(65, 300, a_range=(1.0, 6.0))
    cam = _cam_at([13.0, 11.0, 7.0], [4.0, 4.0, 2.0], width=96, height=96, f=90.0)
    fb = RR.rasterize(scene, cam)
    color, _op, _d = RY.render_rays_image(scene, RY.build_scene_octrees(scene), camera_rays(cam))
    color = color.cpu().numpy() if hasattr(color, "cpu") else np.asarray(color)
    assert float(np.mean(np.abs(fb.color.cpu().numpy() - color))) < 0.02


def _random_rays(rng, n, lo, hi):
    """Origins in the box (jittered off the grid planes), unit directions."""
    o = rng.uniform(lo, hi, (n, 3)) + 0.0137
    d = rng.normal(size=(n, 3))
    return o, d / np.linalg.norm(d, axis=1, keepdims=True)


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_time_invariance_static_scene(exact):
    """reference test_render_ray.py:128-135."""
    from paper_2507_18713_b200 import render_ray as RY
    scene = _random_scene(43, 100)
    oc = RY.build_scene_octrees(scene)
    o, d = _random_rays(np.random.default_rng(44), 50, [0, 0, 0], [8, 8, 8])
    a = RY.integrate_rays(scene, oc, o, d, np.zeros(50), exact_color=exact)
    b = RY.integrate_rays(scene, oc, o, d, np.full(50, 7.5), exact_color=exact)
    assert torch.equal(a.out_color, b.out_color) and torch.equal(a.opacity, b.opacity)


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_early_stopped_static_path_equals_merged_path(exact):
    """reference test_render_ray.py:137-154: the early-stopped static march
    equals the march-everything path taken when an (empty) actor exists."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.scene import Actor, Scene, SparseVoxelSet, make_actor_bounds
    scene = _random_scene(45, 300, a_range=(2.0, 8.0))
    o, d = _random_rays(np.random.default_rng(46), 100, [0, 0, 0], [8, 8, 8])
    fused = RY.integrate_rays(scene, RY.build_scene_octrees(scene), o, d, exact_color=exact)
    ghost = Actor("ghost", np.array([0.5, 0.5, 0.5]), SparseVoxelSet(make_actor_bounds([0.5, 0.5, 0.5], 0.25),
                                                                        budget=1),
                  times=np.array([0.0]), positions=np.zeros((1, 3)), quaternions=np.array([[1.0, 0, 0, 0]]))
    scene_a = Scene(bounds=scene.bounds, static=scene.static, actors=[ghost])
    merged = RY.integrate_rays(scene_a, RY.build_scene_octrees(scene_a), o, d, np.zeros(100), exact_color=exact)
    tol = 1e-12 if exact else 2e-6  # mixed: the certified fp32 static path against the fp64 merge
    np.testing.assert_allclose(fused.out_color.double().cpu().numpy(), merged.out_color.double().cpu().numpy(),
                               atol=tol, rtol=0)
    np.testing.assert_allclose(fused.opacity.double().cpu().numpy(), merged.opacity.double().cpu().numpy(),
                               atol=tol, rtol=0)


def test_colour_only_backward_equals_zero_depth_seeds():
    """rasterize_backward(d_depth=None) -- the colour-only instantiation --
    gives the gradients of zero depth seeds (bitwise, deterministic mode)."""
    from paper_2507_18713_b200 import render_raster as RR
    scene = _random_scene(66, 300)
    cam = _cam_at([13.0, 11.0, 7.0], [4.0, 4.0, 2.0], width=80, height=72, f=70.0)
    fb, st = RR.rasterize(scene, cam, return_state=True)
    rng = np.random.default_rng(7)
    dc = torch.as_tensor(np.sign(rng.normal(size=(72, 80, 3))) / 1e4, device="cuda")
    zd = torch.zeros((72, 80), dtype=torch.float64, device="cuda")
    for det in (True, False):
        a = RR.rasterize_backward(st, dc, zd, as_dict=False, deterministic=det).cpu().numpy()
        b = RR.rasterize_backward(st, dc, None, as_dict=False, deterministic=det).cpu().numpy()
        if det:
            np.testing.assert_array_equal(a, b)
        else:
            np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-18)
        assert np.count_nonzero(b) > 0
