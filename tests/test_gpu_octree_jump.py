"""GPU: the octree descent jump table (csrc salf_octree_jump_build) changes no
result.  Queries, hit lists, LiDAR ranges and ray-path gradients are compared
bitwise between descents that walk every level from the root (jump off) and
descents that start from the depth-K table, K = 1..8, on the golden scenes and
the S1M init scene."""

import dataclasses

import numpy as np
import pytest
import torch

from conftest import load_golden_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _probe_points(tree, n, seed):
    """Random points in the root cube plus points exactly on depth-1..8 cell
    planes and on the root faces (the u == 0 / u == 1 clamps)."""
    rng = np.random.default_rng(seed)
    lo = np.asarray(tree.root_min, np.float64)
    e = float(tree.root_edge)
    p = lo + rng.random((n, 3)) * e
    grid = []
    for lvl in range(1, 9):
        k = rng.integers(0, 2 ** lvl + 1, size=(n // 16, 3))
        g = lo + k * (e / 2 ** lvl)
        jitter = rng.integers(0, 3, size=g.shape)  # keep some coordinates off-plane
        g = np.where(jitter == 0, lo + rng.random(g.shape) * e, g)
        grid.append(g)
    return np.concatenate([p, *grid, lo[None, :], (lo + e)[None, :]])


@pytest.mark.parametrize("name", ["rand400", "rand400m", "rand300i", "actors"])
def test_query_identical_with_jump_table(name):
    from paper_2507_18713_b200.octree import build_octree, query_batch
    sc = load_golden_scene(name)
    tree = build_octree(sc.static)
    pts = _probe_points(tree, 20000, 3)
    ref = query_batch(tree.with_jump(0), pts)
    for k in range(1, 9):
        got = query_batch(tree.with_jump(k), pts)
        for a, b in zip(ref, got):
            np.testing.assert_array_equal(a, b)


def test_query_and_march_identical_with_jump_table_s1m():
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200.octree import march_segments, query_batch
    from paper_2507_18713_b200.render_ray import build_scene_octrees
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    scene = get_scene("S1M", "init")
    tree = build_scene_octrees(scene).static
    assert tree.max_depth >= 6
    pts = _probe_points(tree, 200000, 5)
    ref = query_batch(tree.with_jump(0), pts)
    rays = gen_lidar_rays(configs.c3_lidar())
    sel = slice(0, None, 7)  # every 7th ray of the sweep (~33k rays, ~4.6M segments)
    o, d = rays.origins[sel], rays.dirs[sel]
    mref = [x.cpu().numpy() for x in march_segments(tree.with_jump(0), o, d)]
    for k in (1, 4, 7, 8):
        t = tree.with_jump(k)
        for a, b in zip(ref, query_batch(t, pts)):
            np.testing.assert_array_equal(a, b)
        for a, b in zip(mref, (x.cpu().numpy() for x in march_segments(t, o, d))):
            np.testing.assert_array_equal(a, b)


def test_lidar_and_ray_backward_identical_with_jump_table():
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_grad_buffer
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    scene = get_scene("S1M", "init")
    ds = DeviceScene.from_scene(scene)
    oc = RY.build_scene_octrees(scene)
    batch = gen_lidar_rays(configs.c3_lidar())
    outs = {}
    for k in (0, 7):
        o2 = dataclasses.replace(oc, static=oc.static.with_jump(k))
        ret = RY.render_lidar(ds, o2, batch)
        rec = RY.integrate_rays(ds, o2, batch.origins, batch.dirs, check_unit=False)
        dd = torch.sign(torch.nan_to_num(rec.depth.double()) - 10.0) / 1e5
        dc = torch.zeros((batch.origins.shape[0], 3), dtype=torch.float64, device=ds.device)
        g = torch.zeros((ds.n, 27), dtype=torch.float64, device=ds.device)
        backward_grad_buffer(rec, dc, dd, g, deterministic=True)
        outs[k] = (ret.depth.cpu().numpy(), rec.depth.cpu().numpy(), g.cpu().numpy())
    for a, b in zip(outs[0], outs[7]):
        np.testing.assert_array_equal(a, b)


def test_depth_only_ray_backward_equals_zero_colour_seeds():
    """backward_grad_buffer(d_color=None) (the depth-only instantiation, no
    colour terms) equals the colour path with zero colour seeds, bitwise
    (deterministic reduction)."""
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_grad_buffer
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    scene = get_scene("S1M", "init")
    ds = DeviceScene.from_scene(scene)
    oc = RY.build_scene_octrees(scene)
    batch = gen_lidar_rays(configs.c3_lidar())
    rec = RY.integrate_rays(ds, oc, batch.origins, batch.dirs, check_unit=False)
    dd = torch.sign(torch.nan_to_num(rec.depth.double()) - 10.0) / 1e5
    zc = torch.zeros((batch.origins.shape[0], 3), dtype=torch.float64, device=ds.device)
    outs = []
    for dc in (zc, None):
        for det in (True, False):
            g = torch.zeros((ds.n, 27), dtype=torch.float64, device=ds.device)
            backward_grad_buffer(rec, dc, dd, g, deterministic=det)
            outs.append(g.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[2])  # deterministic: bitwise
    np.testing.assert_allclose(outs[1], outs[3], rtol=1e-9, atol=1e-15)  # atomics: order only
    assert np.count_nonzero(outs[2][:, 4:25]) == 0 and np.count_nonzero(outs[2][:, :4]) > 0
