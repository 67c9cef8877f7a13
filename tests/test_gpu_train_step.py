"""GPU: the C5 multi-sensor step (cameras rasterized in row bands, LiDAR in ray
blocks, global L1 normalisation) equals the oracle's composition of the
reference backward over all sensors, and sharding over virtual ranks sums to
the same gradient."""

import numpy as np
import pytest
import torch

from conftest import assert_grads, grads_close_normwise, load_golden_scene, magnitude, oracle_voxels
from oracle import salf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _rig():
    from paper_2507_18713_b200.sensors import CameraModel, LidarModel, look_at_quaternion
    cams = []
    for pos in ([13.0, 11.0, 7.0], [-4.0, 9.0, 5.0]):
        cams.append(CameraModel(kind="pinhole", width=48, height=40, fx=45.0, fy=45.0, cx=24.0, cy=20.0,
                                position=np.array(pos), quaternion=look_at_quaternion(pos, [4.0, 4.0, 2.0])))
    lid = LidarModel(beam_elevations=np.linspace(-0.5, 0.3, 8), steps=60, position=np.array([4.013, 3.987, 2.5]),
                     linear_velocity=np.array([1.0, 0.0, 0.0]))
    return cams + [lid]


def _targets(sensors):
    rng = np.random.default_rng(9)
    out = []
    for s in sensors:
        if hasattr(s, "width"):
            out.append(torch.as_tensor(rng.uniform(0, 1, (s.height, s.width, 3)), device="cuda"))
        else:
            out.append(torch.as_tensor(rng.uniform(1, 8, s.beam_elevations.shape[0] * s.steps), device="cuda"))
    return out


def _oracle_grad(sc, sensors, targets, depth_weight=10.0):
    vox = oracle_voxels(sc)
    tree = O.build_octree(vox)
    recs = []
    for s, gt in zip(sensors, targets):
        gt = gt.cpu().numpy()
        if hasattr(s, "width"):
            cam = O.Camera("pinhole", s.width, s.height, s.fx, s.fy, s.cx, s.cy, position=s.position,
                           quaternion=s.quaternion)
            recs.append(("c", O.raster_records(vox, cam), gt.reshape(-1, 3)))
        else:
            lid = O.Lidar(s.beam_elevations, s.azimuth_start, s.azimuth_end, s.steps, s.scan_period, s.position,
                          s.quaternion, s.linear_velocity, s.angular_velocity)
            rays = O.lidar_rays(lid)
            recs.append(("l", O.integrate_rays(vox, tree, rays["origins"], rays["dirs"]), gt))
    n_c = sum(r["out_color"].size for k, r, _ in recs if k == "c")
    n_d = sum(int((np.isfinite(r["depth"]) & np.isfinite(gt)).sum()) for k, r, gt in recs if k == "l")
    tot = mag = None
    for k, r, gt in recs:
        if k == "c":
            dc = np.sign(r["out_color"] - gt) / n_c
            dd = np.zeros(r["n_rays"])
        else:
            ok = np.isfinite(r["depth"]) & np.isfinite(gt)
            dd = np.where(ok, depth_weight * np.sign(np.nan_to_num(r["depth"]) - gt) / n_d, 0.0)
            dc = np.zeros((r["n_rays"], 3))
        g = O.backward_records(r, vox, dc, dd)
        m = magnitude(r, vox, dc, dd)
        tot = g if tot is None else {q: tot[q] + g[q] for q in g}
        mag = m if mag is None else {q: mag[q] + m[q] for q in m}
    return tot, mag


def test_rig_step_matches_oracle_and_sharding_is_exact():
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene, grads_to_dict
    from paper_2507_18713_b200.parallel import assign, split_work
    from paper_2507_18713_b200.train_step import rig_backward, rig_forward, rig_step
    sc = load_golden_scene("rand300")
    ds = DeviceScene.from_scene(sc)
    oc = RY.build_scene_octrees(sc)
    sensors = _rig()
    targets = _targets(sensors)
    grad = torch.zeros((ds.n, 27), dtype=torch.float64, device="cuda")
    rig_step(ds, oc, sensors, targets, split_work(sensors, 1), grad)
    want, mag = _oracle_grad(sc, sensors, targets)
    assert_grads(grads_to_dict(grad), want, mag)
    # four virtual ranks: bands + ray blocks, counts summed between the phases
    per = assign(split_work(sensors, 4, tile=16), 4)
    assert sum(len(p) for p in per) > len(sensors)  # cameras really are cut into bands
    states = [rig_forward(ds, oc, sensors, targets, items) for items in per]
    counts = sum(fs.counts for fs in states)
    g2 = torch.zeros_like(grad)
    for fs in states:
        rig_backward(fs, g2, counts)
    assert grads_close_normwise(grads_to_dict(g2), grads_to_dict(grad)) < 1e-6


def test_rig_step_two_processes_gloo(tmp_path):
    """C5 step as two processes (gloo, both on cuda:0): each rank rasterizes /
    marches its share, the counts, gradient rows and losses are all-reduced
    inside rig_step (parallel.allreduce_grad_, f64 transport), and rank 0's
    buffer equals the one-process step and the oracle composition."""
    import socket
    import torch.multiprocessing as mp
    from _rig_worker import run
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene, grads_to_dict
    from paper_2507_18713_b200.parallel import split_work
    from paper_2507_18713_b200.train_step import rig_step
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(run, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    r = np.load(out)
    sc = load_golden_scene("rand300")
    ds = DeviceScene.from_scene(sc)
    oc = RY.build_scene_octrees(sc)
    sensors = _rig()
    targets = _targets(sensors)
    grad = torch.zeros((ds.n, 27), dtype=torch.float64, device="cuda")
    losses, counts = rig_step(ds, oc, sensors, targets, split_work(sensors, 1), grad)
    np.testing.assert_array_equal(r["counts"], counts.cpu().numpy())
    np.testing.assert_allclose(r["losses"], losses.cpu().numpy(), rtol=1e-12)
    assert grads_close_normwise(grads_to_dict(torch.as_tensor(r["grad"])), grads_to_dict(grad)) < 1e-12
    want, mag = _oracle_grad(sc, sensors, targets)
    assert_grads(grads_to_dict(torch.as_tensor(r["grad"])), want, mag)


def test_adam_and_regularisers_match_reference(golden):
    """Adam (optim.py:48-62) and eikonal / empty / LiDAR-opacity regularisers
    (losses.py:49-249) on the device vs the reference's own outputs."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import grads_to_dict
    from paper_2507_18713_b200.optim import (AdamConfig, TrainableScene, loss_eikonal, loss_empty,
                                             loss_opacity_lidar)
    sc = load_golden_scene("fd10")
    ts = TrainableScene(sc)
    oc = RY.build_scene_octrees(sc)
    g = ts.zero_grad()
    l_e = loss_eikonal(ts, np.arange(ts.n), g)
    np.testing.assert_allclose(grads_to_dict(g)["w_s"], golden["reg_eik_w_s"], rtol=1e-10, atol=1e-14)
    g = ts.zero_grad()
    l_m = loss_empty(ts, golden["reg_outer"], g)
    gd = grads_to_dict(g)
    for k in ("w_s", "log_a", "log_b"):
        np.testing.assert_allclose(gd[k], golden["reg_emp_" + k], rtol=1e-10, atol=1e-14)
    g = ts.zero_grad()
    l_o = loss_opacity_lidar(ts, oc.static, golden["reg_points"], g)
    gd = grads_to_dict(g)
    for k in ("w_s", "log_a", "log_b"):
        np.testing.assert_allclose(gd[k], golden["reg_opa_" + k], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose([l_e, l_m, l_o], golden["reg_loss"], rtol=1e-10)
    names = ("w_s", "w_c", "w_sh", "log_a", "log_b")
    for i in range(3):
        gb = np.concatenate([golden[f"adam_g{i}_{k}"].reshape(ts.n, -1) for k in names], axis=1)
        ts.adam_step(torch.as_tensor(gb, device="cuda"), AdamConfig(lr_decay_every=2))
    got = ts.to_numpy()
    for k in names:
        np.testing.assert_allclose(got[k], golden["adam_p_" + k], rtol=1e-13, atol=1e-15)
    # the render-side scene was refreshed from the updated block
    assert np.allclose(ts.ds.prm[:, :4].cpu().numpy(), got["w_s"].astype(np.float32))


@pytest.mark.parametrize("case", ["fd10", "rand60s"])
def test_smoothness_regulariser_matches_reference(golden, case):
    """loss_smooth (losses.py:95-185): face pairs found by device octree queries,
    deduplicated in the reference's iteration order; value and gradients."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import grads_to_dict
    from paper_2507_18713_b200.optim import TrainableScene, loss_smooth
    sc = load_golden_scene(case)
    ts = TrainableScene(sc)
    oc = RY.build_scene_octrees(sc)
    g = ts.zero_grad()
    if case == "fd10":
        idx, pre = np.arange(ts.n), "reg_smo_"
        want_loss = golden["reg_smooth_loss"][0]
    else:
        idx, pre = golden["reg_smooth2_idx"], "reg_smo2_"
        want_loss = golden["reg_smooth2_loss"][0]
    val = loss_smooth(ts, oc.static, idx, g)
    assert val == pytest.approx(want_loss, rel=1e-10)
    gd = grads_to_dict(g)
    for k in ("w_s", "w_c", "w_sh"):
        np.testing.assert_allclose(gd[k], golden[pre + k], rtol=1e-9, atol=1e-13)


@pytest.mark.parametrize("gt_dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("masked", [False, True])
def test_fused_l1_color_seed(gt_dtype, masked):
    """backward.l1_color_seed (one kernel) == losses.py:22-31 restated with torch ops."""
    from paper_2507_18713_b200.backward import l1_color_seed, loss_color_seed
    g = torch.Generator(device="cuda").manual_seed(3)
    c = torch.rand((37, 29, 3), device="cuda", generator=g)
    gt = torch.rand((37, 29, 3), device="cuda", generator=g).to(gt_dtype)
    gt[0, 0] = c[0, 0].to(gt_dtype)  # sign(0) = 0
    mask = (torch.rand(37 * 29, device="cuda", generator=g) > 0.3) if masked else None
    d, lsum = l1_color_seed(c, gt, mask)
    mref = mask if masked else torch.ones(37 * 29, dtype=torch.bool, device="cuda")
    want = loss_color_seed(c.reshape(-1, 3), gt.reshape(-1, 3)[mref], mref).reshape(37, 29, 3)
    assert torch.equal(d, want)
    diff = (c.double() - gt.double()).reshape(-1, 3)[mref]
    torch.testing.assert_close(lsum, diff.abs().sum(), rtol=1e-12, atol=0)


def test_trainable_scene_with_actors_covers_static_rows_only():
    """a scene with actors trains the static owner only -- the device
    scene, the parameter block and the Adam moments all have the static row
    count, an Adam step refreshes exactly those rows, and densify keeps them
    consistent (the actor voxels never enter the block)."""
    from paper_2507_18713_b200.optim import TrainableScene
    sc = load_golden_scene("actors")
    assert sc.actors and sum(a.voxels.n for a in sc.actors) > 0
    ts = TrainableScene(sc)
    m = sc.static.n
    assert ts.n == m == ts.params.shape[0] == ts.m.shape[0] == ts.ds.geo.shape[0]
    prm0 = ts.ds.prm.clone()
    g = torch.zeros_like(ts.params)
    g[:, 0] = 1.0
    ts.adam_step(g)
    torch.cuda.synchronize()
    assert ts.ds.prm.shape == prm0.shape
    # w_s[0] moved by -lr on every static row, nothing else changed
    d = (ts.ds.prm - prm0).double()
    assert torch.allclose(d[:, 0], torch.full_like(d[:, 0], -0.01), atol=1e-6)
    assert float(d[:, 1:].abs().max()) == 0.0
