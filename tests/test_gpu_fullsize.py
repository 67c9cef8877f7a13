"""GPU parity at the BASELINE.json sizes (S1M / S2M, 1080p, full LiDAR sweeps):
the CUDA path against the oracle on bounded samples of each full-size run,
checked ELEMENT BY ELEMENT (tests/parity.py):

* C2 forward: 32 random tiles of the 1080p frame -- colour, opacity, depth;
* C2 backward: L1 seeds on 8 of those tiles, all five parameter classes;
* C3: 4096 rays of the 128 x 1800 sweep -- depth, opacity, gradients of a
  depth loss; hit lists of 400 of them bit for bit;
* C4: 4096 valid rays of the fisheye + rolling-shutter frame on S2M --
  colour, opacity, depth; hit lists of 300 bit for bit;
* C5: the whole 8-camera + 2-LiDAR training step on S1M (train_step.rig_step:
  forward, globally normalised L1 seeds, raster + ray backward), with the
  loss seeded on 2 tiles per camera and 1024 rays per LiDAR, against the
  oracle's raster_records / integrate_rays -> backward_records summed over
  the sensors (reference trainer.py:156-161, backward.py:35-101)."""

import numpy as np
import pytest
import torch

from conftest import assert_grads, assert_image, magnitude, oracle_voxels
from oracle import salf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(scope="module")
def s1m():
    from paper_2507_18713_b200.scenes import get_scene
    return get_scene("S1M", "init")


@pytest.fixture(scope="module")
def vox1m(s1m):
    return oracle_voxels(s1m)


@pytest.fixture(scope="module")
def tree1m(vox1m):
    return O.build_octree(vox1m)


@pytest.fixture(scope="module")
def ds1m(s1m):
    from paper_2507_18713_b200.device import DeviceScene
    return DeviceScene.from_scene(s1m)


@pytest.fixture(scope="module")
def oc1m(s1m):
    from paper_2507_18713_b200 import render_ray as RY
    return RY.build_scene_octrees(s1m)


def _ocam(cam):
    return O.Camera(cam.kind, cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.distortion,
                    cam.position, cam.quaternion, cam.readout_duration, cam.linear_velocity,
                    cam.angular_velocity)


def _tile_mask(tiles, h, w, tiles_x, tile=16):
    m = np.zeros((h, w), bool)
    for t in tiles:
        ty, tx = divmod(int(t), tiles_x)
        m[ty * tile:(ty + 1) * tile, tx * tile:(tx + 1) * tile] = True
    return m


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def test_c2_forward_and_backward_sampled_tiles(ds1m, vox1m):
    """C2 (1080p, S1M): the default certified forward on 32 random tiles and the
    default mixed backward with L1 seeds on 8 of them, elementwise."""
    from paper_2507_18713_b200 import configs, render_raster as RR
    cam = configs.c2_camera()
    h, w = cam.height, cam.width
    ocam = _ocam(cam)
    proj = O.project_voxels(vox1m, ocam)
    rng = np.random.default_rng(11)
    tiles = rng.choice(120 * 68, 32, replace=False)
    ref = O.rasterize(vox1m, ocam, tiles=tiles, proj=proj)
    sel = _tile_mask(tiles, h, w, 120)
    fb, st = RR.rasterize(ds1m, cam, return_state=True)
    assert_image(_np(fb.color)[sel], ref["color"][sel], "color")
    assert_image(_np(fb.opacity)[sel], ref["opacity"][sel], "opacity")
    assert_image(_np(fb.depth)[sel], ref["depth"][sel], "depth")
    assert np.isnan(ref["depth"][sel]).sum() < sel.sum()  # some returns, some sky
    btiles = tiles[:8]
    bsel = _tile_mask(btiles, h, w, 120)
    gt = rng.uniform(0, 1, (h, w, 3))
    dc = np.where(bsel[..., None], np.sign(ref["color"] - gt) / (3 * bsel.sum()), 0.0)
    rec = O.raster_records(vox1m, ocam, tiles=btiles, proj=proj)
    want = O.backward_records(rec, vox1m, dc.reshape(-1, 3), np.zeros(h * w))
    g = RR.rasterize_backward(st, dc, None)
    assert np.abs(want["w_s"]).max() > 0
    assert_grads(g, want, magnitude(rec, vox1m, dc, np.zeros(h * w)))


def test_c3_lidar_sampled_rays(ds1m, oc1m, vox1m, tree1m):
    """C3 (128 x 1800 on S1M): 4096 rays -- depth / opacity and the gradients of
    a depth L1 loss elementwise, hit lists of 400 bit for bit, every ray
    terminates, 32.3M segments per sweep."""
    from paper_2507_18713_b200 import configs, render_ray as RY
    from paper_2507_18713_b200.device import grads_to_dict
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    lb = gen_lidar_rays(configs.c3_lidar())
    ret = RY.render_lidar(ds1m, oc1m, lb)
    assert int(ret.status.max()) == 0
    assert 31_000_000 < int(ret.saved[:, 6].sum()) < 34_000_000
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(lb.n, 4096, replace=False))
    o, d = lb.origins[idx].cpu().numpy(), lb.dirs[idx].cpu().numpy()
    orec = O.integrate_rays(vox1m, tree1m, o, d)
    assert_image(_np(ret.depth).reshape(-1)[idx], orec["depth"], "depth")
    assert_image(_np(ret.opacity).reshape(-1)[idx], orec["opacity"], "opacity")
    ray, vid, t0, t1 = (x.cpu().numpy() for x in RY.segments(ds1m, oc1m, o[:400], d[:400]))
    ref = O.integrate_rays(vox1m, tree1m, o[:400], d[:400])
    for a, k in ((ray, "ray"), (vid, "vid"), (t0, "t0"), (t1, "t1")):
        np.testing.assert_array_equal(a, ref[k])
    gtr = rng.uniform(1, 30, idx.size)
    ok = np.isfinite(orec["depth"])
    dd_s = np.where(ok, np.sign(np.nan_to_num(orec["depth"]) - gtr) / max(ok.sum(), 1), 0.0)
    want = O.backward_records(orec, vox1m, np.zeros((idx.size, 3)), dd_s)
    dd = np.zeros(lb.n)
    dd[idx] = dd_s
    g, _, _ = RY.lidar_backward(ret, torch.as_tensor(dd, device="cuda"))
    assert_grads(grads_to_dict(g), want, magnitude(orec, vox1m, np.zeros((idx.size, 3)), dd_s))


def test_c4_fisheye_rolling_shutter_sampled_rays():
    """C4 (1920x1080 fisheye + rolling shutter on S2M): rays equal the oracle's
    (1e-12), 4096 valid pixels elementwise, hit lists of 300 bit for bit."""
    from paper_2507_18713_b200 import configs, render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import camera_rays
    sc = get_scene("S2M", "init")
    cam = configs.c4_camera()
    b = camera_rays(cam)
    ref_rays = O.camera_rays(_ocam(cam))
    assert np.max(np.abs(b.dirs.cpu().numpy() - ref_rays["dirs"])) < 1e-12
    assert np.max(np.abs(b.origins.cpu().numpy() - ref_rays["origins"])) < 1e-12
    np.testing.assert_array_equal(b.valid.cpu().numpy(), ref_rays["valid"])
    ds = DeviceScene.from_scene(sc)
    oc = RY.build_scene_octrees(sc)
    col, op, dep = RY.render_rays_image(ds, oc, b)
    valid = np.flatnonzero(ref_rays["valid"])
    idx = np.sort(np.random.default_rng(3).choice(valid, 4096, replace=False))
    o, d = ref_rays["origins"][idx], ref_rays["dirs"][idx]
    vox = oracle_voxels(sc)
    tree = O.build_octree(vox)
    ref = O.integrate_rays(vox, tree, o, d)
    assert_image(_np(col).reshape(-1, 3)[idx], ref["out_color"], "color")
    assert_image(_np(op).reshape(-1)[idx], ref["opacity"], "opacity")
    assert_image(_np(dep).reshape(-1)[idx], ref["depth"], "depth")
    ray, vid, t0, t1 = (x.cpu().numpy() for x in RY.segments(ds, oc, o[:300], d[:300]))
    r3 = O.integrate_rays(vox, tree, o[:300], d[:300])
    for a, k in ((ray, "ray"), (vid, "vid"), (t0, "t0"), (t1, "t1")):
        np.testing.assert_array_equal(a, r3[k])


def test_c5_rig_step_full_size(s1m, ds1m, oc1m, vox1m, tree1m):
    """C5 at full size: train_step.rig_step over the 8 x 1080p + 2 x 128x1800
    rig on S1M.  Targets equal the rendered outputs except on 2 tiles per
    camera and 1024 rays per LiDAR, so the global L1 seeds (normalised by the
    counts of ALL pixels / returns, losses.py:29-30, :44-45) are non-zero only
    there; the accumulated gradient equals the oracle's backward_records summed
    over the sensors' sampled records, elementwise."""
    from paper_2507_18713_b200 import configs, render_raster as RR, render_ray as RY
    from paper_2507_18713_b200.device import grads_to_dict
    from paper_2507_18713_b200.parallel import split_work
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    from paper_2507_18713_b200.train_step import rig_step
    cams, lidars = configs.c5_rig()
    sensors = cams + lidars
    rng = np.random.default_rng(55)
    targets, samples = [], []
    for cam in cams:
        c = RR.rasterize(ds1m, cam).color.double()
        tiles = rng.choice(120 * 68, 2, replace=False)
        m = torch.as_tensor(_tile_mask(tiles, cam.height, cam.width, 120), device="cuda")
        sgn = torch.as_tensor(rng.choice([-1.0, 1.0], (cam.height, cam.width, 3)), device="cuda")
        targets.append(torch.where(m[..., None], c + 0.05 * sgn, c))
        samples.append(tiles)
    for lid in lidars:
        dep = RY.render_lidar(ds1m, oc1m, gen_lidar_rays(lid)).depth.reshape(-1).double()
        fin = torch.isfinite(dep).cpu().numpy()
        idx = np.sort(rng.choice(np.flatnonzero(fin), 1024, replace=False))
        gt = dep.clone()
        gt[torch.as_tensor(idx, device="cuda")] += torch.as_tensor(rng.choice([-0.5, 0.5], idx.size),
                                                                   device="cuda")
        targets.append(gt)
        samples.append(idx)
    grad = torch.zeros((ds1m.n, 27), dtype=torch.float64, device="cuda")
    _, counts = rig_step(ds1m, oc1m, sensors, targets, split_work(sensors, 1), grad)
    n_c, n_d = float(counts[0]), float(counts[1])
    assert n_c == 8 * 1080 * 1920 * 3
    # oracle: the sampled records of every sensor -> backward_records, summed
    want = mag = None
    for i, (s, gt, smp) in enumerate(zip(sensors, targets, samples)):
        gt = gt.cpu().numpy()
        if i < len(cams):
            ocam = _ocam(s)
            rec = O.raster_records(vox1m, ocam, tiles=smp)
            sel = _tile_mask(smp, s.height, s.width, 120).reshape(-1)
            dc = np.where(sel[:, None], np.sign(rec["out_color"] - gt.reshape(-1, 3)) / n_c, 0.0)
            dd = np.zeros(rec["n_rays"])
        else:
            lr = O.lidar_rays(O.Lidar(s.beam_elevations, s.azimuth_start, s.azimuth_end, s.steps, s.scan_period,
                                      s.position, s.quaternion, s.linear_velocity, s.angular_velocity))
            rec = O.integrate_rays(vox1m, tree1m, lr["origins"][smp], lr["dirs"][smp])
            dc = np.zeros((smp.size, 3))
            dd = 10.0 * np.sign(rec["depth"] - gt[smp]) / n_d
        g = O.backward_records(rec, vox1m, dc, dd)
        m = magnitude(rec, vox1m, dc, dd)
        want = g if want is None else {k: want[k] + g[k] for k in g}
        mag = m if mag is None else {k: mag[k] + m[k] for k in m}
    assert np.abs(want["w_s"]).max() > 0
    assert_grads(grads_to_dict(grad), want, mag)
