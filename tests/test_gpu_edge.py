"""GPU: the reference suite's edge cases and known answers, run through the
CUDA path, plus full-size (BASELINE config) checks against the oracle on
bounded samples and size-independent invariants."""

import numpy as np
import pytest
import torch

from conftest import oracle_voxels
from oracle import salf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _scene(lo, hi, base, levels, cells, vlevels=None, a=2.0, seed=0):
    from paper_2507_18713_b200.scene import Scene, SceneBounds, SparseVoxelSet
    from paper_2507_18713_b200.scenes import f32_roundtrip
    b = SceneBounds(np.asarray(lo, float), np.asarray(hi, float), base, levels)
    v = SparseVoxelSet(b, 1000)
    n = len(cells)
    rng = np.random.default_rng(seed)
    if n:
        v.set_arrays(np.zeros(n) if vlevels is None else vlevels, cells,
                     rng.uniform(-1 / np.sqrt(3), 1 / np.sqrt(3), (n, 4)),
                     rng.uniform(-1 / np.sqrt(3), 1 / np.sqrt(3), (n, 3, 3)),
                     rng.uniform(-0.5, 0.5, (n, 3, 4)), np.log(np.broadcast_to(a, (n,))),
                     np.log(np.full(n, 0.2)))
    return f32_roundtrip(Scene(bounds=b, static=v))


def _cam(pos=(0, 0, 0), w=32, h=32, f=40.0, cx=None, cy=None, target=None, kind="pinhole"):
    from paper_2507_18713_b200.sensors import CameraModel, look_at_quaternion
    q = look_at_quaternion(pos, target) if target is not None else np.array([1.0, 0, 0, 0])
    return CameraModel(kind=kind, width=w, height=h, fx=f, fy=f, cx=w / 2 if cx is None else cx,
                       cy=h / 2 if cy is None else cy, position=np.asarray(pos, float), quaternion=q)


def _raster64(scene, cam, bg=(0.0, 0.0, 0.0)):
    """f64 outputs from the raster saved state (colour, opacity, depth, weight sum)."""
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    fb, st = RR.rasterize(flatten_scene(scene), cam, background=bg, return_state=True, exact_color=True)
    s = st.saved.cpu().numpy()
    T = s[:, 5]
    col = s[:, :3] + T[:, None] * np.asarray(bg)
    depth = np.where(s[:, 3] > 0.5, s[:, 4] / np.where(s[:, 3] > 0, s[:, 3], 1), np.nan)
    return col, 1 - T, depth, s[:, 3], fb


def _ray64(scene, o, d, bg=(0.0, 0.0, 0.0)):
    from paper_2507_18713_b200 import render_ray as RY
    rec = RY.integrate_rays(scene, RY.build_scene_octrees(scene), o, d, background=bg, exact_color=True)
    s = rec.saved.cpu().numpy()
    T = s[:, 5]
    col = s[:, :3] + T[:, None] * np.asarray(bg)
    depth = np.where(s[:, 3] > 0.5, s[:, 4] / np.where(s[:, 3] > 0, s[:, 3], 1), np.nan)
    return col, 1 - T, depth, s[:, 3], rec


# ---- reference-suite known answers (test_render_raster.py / test_render_ray.py) ------

def test_empty_scene_background():
    from paper_2507_18713_b200 import render_raster as RR, render_ray as RY
    sc = _scene([0, 0, 0], [2, 2, 2], 1.0, 2, np.zeros((0, 3), int))
    fb = RR.rasterize_scene(sc, _cam(w=32, h=32, f=30.0), background=(0.1, 0.2, 0.3))
    assert torch.allclose(fb.color.cpu(), torch.tensor([0.1, 0.2, 0.3]))
    assert bool((fb.opacity == 0).all()) and bool(torch.isnan(fb.depth).all())
    rec = RY.integrate_rays(sc, RY.build_scene_octrees(sc), [[-1, 1, 1]], [[1.0, 0, 0]],
                            background=(0.2, 0.3, 0.4))
    assert np.allclose(rec.out_color.cpu().numpy(), [0.2, 0.3, 0.4])
    assert float(rec.opacity[0]) == 0.0 and bool(torch.isnan(rec.depth[0]))


def test_non_pinhole_rejected():
    from paper_2507_18713_b200 import render_raster as RR
    sc = _scene([0, 0, 0], [2, 2, 2], 1.0, 2, np.zeros((0, 3), int))
    with pytest.raises(ValueError, match="pinhole"):
        RR.rasterize_scene(sc, _cam(kind="equirect", w=8, h=8))


def test_non_unit_direction_rejected():
    from paper_2507_18713_b200 import octree as OC
    sc = _scene([0, 0, 0], [2, 2, 2], 1.0, 3, [[0, 0, 0]])
    with pytest.raises(ValueError, match="unit norm"):
        OC.march(OC.build_octree(sc.static), [0.5, 0.5, 0.5], [1.0, 1.0, 0.0])


def test_query_outside_root_raises():
    from paper_2507_18713_b200 import octree as OC
    sc = _scene([0, 0, 0], [2, 2, 2], 1.0, 3, [[0, 0, 0]])
    with pytest.raises(ValueError):
        OC.query(OC.build_octree(sc.static), [5.0, 0.5, 0.5])


def test_march_known_answers():
    """test_octree.py:149-171, :215-219."""
    from paper_2507_18713_b200 import octree as OC
    sc = _scene([0, 0, 0], [4, 4, 4], 1.0, 2, [[i, 0, 0] for i in range(4)])
    segs = OC.march(OC.build_octree(sc.static), [-1.0, 0.5, 0.5], [1.0, 0, 0])
    assert [s[0] for s in segs] == [0, 1, 2, 3]
    sc2 = _scene([0, 0, 0], [2, 2, 2], 1.0, 3, [[0, 0, 0]])
    buf = OC.build_octree(sc2.static)
    segs = OC.march(buf, [0.5, 0.5, 0.5], [1.0, 0, 0])
    assert len(segs) == 1 and segs[0][1] == 0.0 and segs[0][2] == pytest.approx(0.5)
    sc3 = _scene([0, 0, 0], [2, 2, 2], 1.0, 3, [[0, 0, 0], [1, 0, 0]])
    segs = OC.march(OC.build_octree(sc3.static), [-1.0, 0.5, 0.5], [1.0, 0, 0], t_max=1.5)
    assert len(segs) == 1 and segs[0][2] <= 1.5


def test_single_voxel_raster_equals_ray_at_principal_pixel():
    """test_render_raster.py:110-123: 1e-6 colour, 1e-9 depth."""
    sc = _scene([-2, -2, -2], [2, 2, 2], 1.0, 3, [[1, 1, 1]], a=50.0, seed=3)
    cam = _cam(pos=(-0.5, -0.5, -1.8), w=33, h=33, f=40.0, cx=16.5, cy=16.5)
    col, _, depth, _, _ = _raster64(sc, cam)
    rcol, _, rdepth, _, _ = _ray64(sc, [cam.position], [[0, 0, 1.0]])
    pix = 16 * 33 + 16
    assert np.max(np.abs(col[pix] - rcol[0])) < 1e-6
    assert depth[pix] == pytest.approx(rdepth[0], abs=1e-9)


def test_depth_single_opaque_segment():
    """test_render_ray.py:121-126."""
    sc = _scene([0, 0, 0], [2, 2, 2], 1.0, 2, [[0, 0, 0]], a=1000.0, seed=5)
    _, _, depth, _, _ = _ray64(sc, [[-1.0, 0.5, 0.5]], [[1.0, 0, 0]])
    assert depth[0] == pytest.approx(1.5, abs=1e-9)


def test_weights_plus_residual_is_one():
    """test_render_ray.py:274-285 invariants on a random scene."""
    from conftest import load_golden_scene
    sc = load_golden_scene("rand300i")
    rng = np.random.default_rng(42)
    o = rng.uniform(-1, 9, (500, 3))
    d = rng.normal(size=(500, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    _, op, _, wsum, rec = _ray64(sc, o, d)
    assert np.allclose(wsum + (1 - op), 1.0, atol=1e-6)
    assert int(rec.status.max()) == 0


def test_zero_loss_and_background_only_give_zero_grads():
    """test_backward.py:38-60."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_records
    from conftest import load_golden_scene
    sc = load_golden_scene("fd10")
    rec = RY.integrate_rays(sc, RY.build_scene_octrees(sc), np.random.default_rng(1).uniform(0, 4, (15, 3)),
                            np.tile([[0.0, 0.0, 1.0]], (15, 1)))
    g = backward_records(rec, sc, np.zeros((15, 3)), np.zeros(15))["static"]
    assert all(np.all(v == 0.0) for v in g.values())
    sc1 = _scene([0, 0, 0], [2, 2, 2], 1.0, 2, [[0, 0, 0]], seed=1)
    rec = RY.integrate_rays(sc1, RY.build_scene_octrees(sc1), [[-1.0, 1.5, 1.5]], [[1.0, 0, 0]])
    g = backward_records(rec, sc1, np.ones((1, 3)), np.ones(1))["static"]
    assert all(np.all(v == 0.0) for v in g.values())


@pytest.mark.parametrize("mode", ["sdf", "raw"])
@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_raster_backward_density_modes(mode, exact):
    """Raster backward in both density modes (scene.py:245-253) and both
    precisions against the oracle composition (raster pairs -> _composite ->
    backward_records), elementwise (tests/parity.py)."""
    import dataclasses
    from conftest import assert_grads, magnitude
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    rng = np.random.default_rng(11)
    cells = np.unique(rng.integers(0, 8, (120, 3)), axis=0)
    sc = _scene([0, 0, 0], [4, 4, 4], 0.5, 2, cells, a=3.0, seed=11)
    sc = dataclasses.replace(sc, density_mode=mode)
    cam = _cam(pos=(5.3, 4.7, 3.9), w=40, h=36, f=36.0, target=(2.0, 2.0, 2.0))
    bg = (0.05, 0.1, 0.15)
    fb, st = RR.rasterize(flatten_scene(sc), cam, background=bg, return_state=True, exact_color=exact)
    dc = rng.normal(size=(36, 40, 3)) * 1e-2
    dd = rng.normal(size=(36, 40)) * 1e-3
    g = RR.rasterize_backward(st, dc, dd)
    vox = oracle_voxels(sc)
    ocam = O.Camera("pinhole", 40, 36, 36.0, 36.0, 20.0, 18.0, position=cam.position,
                    quaternion=cam.quaternion)
    rec = O.raster_records(vox, ocam, background=bg)
    want = O.backward_records(rec, vox, dc.reshape(-1, 3), dd.reshape(-1))
    assert np.isfinite(rec["out_color"]).all() and np.abs(want["w_s"]).max() > 0
    assert_grads(g, want, magnitude(rec, vox, dc, dd))


def test_fisheye_invalid_pixels_keep_background():
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.sensors import CameraModel, camera_rays
    from conftest import load_golden_scene
    sc = load_golden_scene("rand300")
    cam = CameraModel(kind="fisheye_equidistant", width=40, height=30, fx=6.0, fy=6.0, cx=20.0, cy=15.0,
                      position=np.array([13.0, 11.0, 7.0]))
    b = camera_rays(cam)
    assert not bool(b.valid.all())
    col, op, depth = RY.render_rays_image(sc, RY.build_scene_octrees(sc), b, background=(0.3, 0.2, 0.1))
    inv = ~b.valid.reshape(30, 40)
    assert torch.allclose(col[inv].cpu(), torch.tensor([0.3, 0.2, 0.1]))
    assert bool((op[inv] == 0).all()) and bool(torch.isnan(depth[inv]).all())


def test_raster_repeat_bitwise_deterministic():
    from paper_2507_18713_b200 import render_raster as RR
    from conftest import load_golden_scene
    from paper_2507_18713_b200.scene import flatten_scene
    flat = flatten_scene(load_golden_scene("rand400"))
    cam = _cam(pos=(12.0, 12.0, 6.0), target=(4.0, 4.0, 2.0), w=40, h=40, f=45.0)
    a, b = RR.rasterize(flat, cam), RR.rasterize(flat, cam)
    assert torch.equal(a.color, b.color)


# ---- full-size configurations (BASELINE configs) on bounded oracle samples ------------

@pytest.fixture(scope="module")
def s1m():
    from paper_2507_18713_b200.scenes import get_scene
    return get_scene("S1M", "init")


def test_c2_reference_bins_full_size(s1m):
    """C2 at 1920x1080 on S1M: the reference CSR has 102.1M instances;
    a sample of tiles is bit-identical to the oracle's binning of those tiles."""
    from paper_2507_18713_b200 import configs, render_raster as RR
    from paper_2507_18713_b200.device import DeviceScene
    cam = configs.c2_camera()
    ds = DeviceScene.from_scene(s1m)
    p = RR._project(ds, cam, 0.05, 16)
    off, ent, n_inst, _ = RR._bin_sync(ds, cam, 0.05, 16, p, mode=0)
    assert 100_000_000 < n_inst < 104_000_000
    vox = oracle_voxels(s1m)
    ocam = O.Camera("pinhole", cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy,
                    position=cam.position, quaternion=cam.quaternion)
    off_h = off.cpu().numpy()
    for (tx, ty) in [(0, 0), (60, 34), (119, 67), (17, 50)]:
        _, _, ooff, oent = O.cull_and_bin(vox, ocam, window=(tx, ty, tx, ty))
        t = ty * 120 + tx
        got = ent[off_h[t]:off_h[t + 1]].cpu().numpy()
        np.testing.assert_array_equal(got, oent[ooff[t]:ooff[t + 1]])


@pytest.mark.parametrize("yaw", [0.0, 135.0])
def test_c2_certified_forward_equals_fp64_decisions(s1m, yaw):
    """The default (certified mixed-precision) forward against the fp64
    reference-order forward on a whole 1080p frame of S1M: every pixel's stop
    index and depth-NaN mask identical, values within fp32 rounding."""
    from paper_2507_18713_b200 import configs, render_raster as RR
    from paper_2507_18713_b200.device import DeviceScene
    ds = DeviceScene.from_scene(s1m)
    cam = configs.c2_camera(yaw)
    fa, sa = RR.rasterize(ds, cam, return_state=True)
    fe, se = RR.rasterize(ds, cam, return_state=True, exact_color=True)
    assert torch.equal(sa.saved[:, 6], se.saved[:, 6])
    assert torch.equal(torch.isnan(fa.depth), torch.isnan(fe.depth))
    assert not torch.isnan(fa.opacity).any()
    assert float((fa.color - fe.color).abs().max()) < 1e-5
    assert float((fa.opacity - fe.opacity).abs().max()) < 1e-5
    m = ~torch.isnan(fe.depth)
    assert float(((fa.depth[m] - fe.depth[m]).abs() / fe.depth[m]).max()) < 1e-5


def test_c2_deterministic_backward_full_size(s1m):
    """C2 at full size: deterministic mode bitwise stable across reruns and
    within fp32 partial-sum rounding of the atomic mode."""
    from paper_2507_18713_b200 import configs, render_raster as RR
    from paper_2507_18713_b200.device import DeviceScene
    cam = configs.c2_camera()
    h, w = cam.height, cam.width
    g = torch.Generator(device="cuda").manual_seed(9)
    dc = (torch.randint(0, 2, (h, w, 3), device="cuda", generator=g).double() * 2 - 1) / (h * w * 3)
    dd = torch.zeros((h, w), dtype=torch.float64, device="cuda")
    fb, st = RR.rasterize(DeviceScene.from_scene(s1m), cam, return_state=True)
    a = RR.rasterize_backward(st, dc, dd, as_dict=False, deterministic=True)
    b = RR.rasterize_backward(st, dc, dd, as_dict=False, deterministic=True)
    assert torch.equal(a, b)
    c = RR.rasterize_backward(st, dc, dd, as_dict=False)
    err = ((a - c).abs().max(dim=0).values / c.abs().max(dim=0).values.clamp_min(1e-30)).max()
    assert float(err) < 1e-6


def test_c3_deterministic_ray_backward_full_size(s1m):
    """C3 LiDAR sweep at full size (32M segments): deterministic ray backward
    bitwise stable across reruns and equal to the atomic mode up to order."""
    from paper_2507_18713_b200 import configs, render_ray as RY
    from paper_2507_18713_b200.backward import backward_grad_buffer
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    lb = gen_lidar_rays(configs.c3_lidar())
    rec = RY.integrate_rays(DeviceScene.from_scene(s1m), RY.build_scene_octrees(s1m), lb.origins, lb.dirs)
    g = torch.Generator(device="cuda").manual_seed(2)
    dd = (torch.randint(0, 2, (lb.n,), device="cuda", generator=g).double() * 2 - 1) / lb.n
    dc = torch.zeros((lb.n, 3), dtype=torch.float64, device="cuda")
    a = backward_grad_buffer(rec, dc, dd, deterministic=True)
    b = backward_grad_buffer(rec, dc, dd, deterministic=True)
    assert torch.equal(a, b)
    c = backward_grad_buffer(rec, dc, dd)
    err = ((a - c).abs().max(dim=0).values / c.abs().max(dim=0).values.clamp_min(1e-30)).max()
    assert float(err) < 1e-6


@pytest.mark.parametrize("sensor", ["c3_lidar", "c4_fisheye"])
def test_certified_ray_forward_equals_fp64_decisions(s1m, sensor):
    """The default (certified mixed-precision) ray forward vs the fp64 one on
    a full C3 sweep and a full C4-camera frame over S1M: per-ray segment
    counts (the product early stop) and depth-NaN masks identical, values
    within fp32 rounding."""
    from paper_2507_18713_b200 import configs, render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.sensors import camera_rays, gen_lidar_rays
    ds = DeviceScene.from_scene(s1m)
    oc = RY.build_scene_octrees(s1m)
    if sensor == "c3_lidar":
        b = gen_lidar_rays(configs.c3_lidar())
        valid = None
    else:
        b = camera_rays(configs.c4_camera())
        valid = b.valid
    fa = RY.integrate_rays(ds, oc, b.origins, b.dirs, valid=valid)
    fe = RY.integrate_rays(ds, oc, b.origins, b.dirs, valid=valid, exact_color=True)
    assert int(fa.status.max()) == 0 and int(fe.status.max()) == 0
    assert torch.equal(fa.saved[:, 6], fe.saved[:, 6])
    assert torch.equal(torch.isnan(fa.depth), torch.isnan(fe.depth))
    m = ~torch.isnan(fe.depth)
    assert float(((fa.depth[m] - fe.depth[m]).abs() / fe.depth[m]).max()) < 1e-5
    assert float((fa.opacity - fe.opacity).abs().max()) < 1e-5
    assert float((fa.out_color - fe.out_color).abs().max()) < 1e-5


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_certified_forward_stress_sharp_fields(seed):
    """Stress for the certified forward's error model: random multi-level
    scenes with sharp SDF transfers (b down to 4e-4), large |W_s| and dense
    opacity, viewed from several poses; raster and ray path decisions (stop
    index / segment counts, depth-NaN masks) must equal the fp64 path's."""
    from paper_2507_18713_b200 import render_raster as RR, render_ray as RY
    from paper_2507_18713_b200.scene import Scene, SceneBounds, SparseVoxelSet, flatten_scene
    from paper_2507_18713_b200.scenes import f32_roundtrip
    rng = np.random.default_rng(100 + seed)
    b = SceneBounds(np.zeros(3), np.full(3, 8.0), 1.0, 4)
    # at most one voxel per level-0 cell (levels 0..2), so no voxel contains another
    taken, L, C = set(), [], []
    for lv in (2, 1, 0):
        for ijk in np.unique(rng.integers(0, 8 * 2 ** lv, (250, 3)), axis=0):
            key0 = tuple(int(q) >> lv for q in ijk)
            if key0 not in taken:
                taken.add(key0)
                L.append(lv)
                C.append(ijk)
    n = len(L)
    v = SparseVoxelSet(b, 10 * n)
    ws = rng.normal(scale=3.0, size=(n, 4))
    v.set_arrays(np.array(L), np.array(C), ws, rng.normal(size=(n, 3, 3)), rng.normal(scale=0.5, size=(n, 3, 4)),
                 np.log(rng.uniform(5.0, 400.0, n)), np.log(rng.uniform(4e-4, 0.2, n)))
    sc = f32_roundtrip(Scene(bounds=b, static=v))
    flat = flatten_scene(sc)
    oc = RY.build_scene_octrees(sc)
    for k in range(3):
        pos = rng.uniform(-3.0, 11.0, 3) + 0.0137
        cam = _cam(pos=pos, w=96, h=80, f=70.0, target=rng.uniform(2.0, 6.0, 3))
        fa, sa = RR.rasterize(flat, cam, return_state=True)
        fe, se = RR.rasterize(flat, cam, return_state=True, exact_color=True)
        assert torch.equal(sa.saved[:, 6], se.saved[:, 6])
        assert torch.equal(torch.isnan(fa.depth), torch.isnan(fe.depth))
        assert float((fa.color - fe.color).abs().max()) < 1e-4
        o = np.tile(pos, (4000, 1))
        d = rng.normal(size=(4000, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        ra = RY.integrate_rays(sc, oc, o, d)
        re = RY.integrate_rays(sc, oc, o, d, exact_color=True)
        assert torch.equal(ra.saved[:, 6], re.saved[:, 6]) and torch.equal(ra.saved[:, 7], re.saved[:, 7])
        assert torch.equal(torch.isnan(ra.depth), torch.isnan(re.depth))


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_ray_path_raw_density(exact):
    """Raw density mode (scene.py:250-252) through the ray path: forward and
    backward against the oracle (integrate_rays + backward_records)."""
    import dataclasses
    from conftest import assert_grads, assert_image, magnitude
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_records
    rng = np.random.default_rng(21)
    cells = np.unique(rng.integers(0, 8, (150, 3)), axis=0)
    sc = dataclasses.replace(_scene([0, 0, 0], [4, 4, 4], 0.5, 2, cells, a=3.0, seed=21), density_mode="raw")
    o = rng.uniform(-1, 5, (600, 3)) + 0.0137
    d = rng.normal(size=(600, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rec = RY.integrate_rays(sc, RY.build_scene_octrees(sc), o, d, background=(0.1, 0.2, 0.3), exact_color=exact)
    vox = oracle_voxels(sc)
    ref = O.integrate_rays(vox, O.build_octree(vox), o, d, background=(0.1, 0.2, 0.3))
    assert_image(rec.out_color.cpu().numpy(), ref["out_color"], "color")
    assert_image(rec.opacity.cpu().numpy(), ref["opacity"], "opacity")
    assert_image(rec.depth.cpu().numpy(), ref["depth"], "depth")
    dc = rng.normal(size=(600, 3)) * 1e-2
    dd = rng.normal(size=600) * 1e-3
    g = backward_records(rec, sc, dc, dd)["static"]
    want = O.backward_records(ref, vox, dc, dd)
    assert_grads(g, want, magnitude(ref, vox, dc, dd))


def test_tile_launch_order(s1m):
    """salf_raster_tile_order: a permutation of the tiles, longest lists first
    (lengths saturated at 65535), ties in tile order -- the launch order of
    the backward (scheduling only)."""
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200 import render_raster as RR
    fb, st = RR.rasterize(s1m, configs.c2_camera(), return_state=True)
    dc = torch.zeros((1080, 1920, 3), dtype=torch.float64, device="cuda")
    dd = torch.zeros((1080, 1920), dtype=torch.float64, device="cuda")
    RR.rasterize_backward(st, dc, dd, as_dict=False)
    lens = (st.offsets[1:] - st.offsets[:-1]).cpu().numpy()
    want = np.argsort(-np.minimum(lens, 65535), kind="stable")
    np.testing.assert_array_equal(st.tile_order.cpu().numpy(), want)
