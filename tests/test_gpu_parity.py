"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle on identical inputs.

Bars (north star): bit-exact tile CSR / sort order / hit lists / octree node
tables; <= 1e-4 relative for rendered colour, opacity, depth and gradients,
ELEMENT BY ELEMENT (tests/parity.py: images |a-b| <= 1e-4 |b| + 1e-7;
gradients |a-b| <= 1e-4 |b| + 1e-5 x the oracle's conditioning scale)."""

import numpy as np
import pytest
import torch

from conftest import (assert_grads, assert_image, grads_close_normwise, load_golden_scene, magnitude,
                      oracle_camera, oracle_lidar, oracle_voxels)
from oracle import salf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _cam(d):
    from paper_2507_18713_b200.sensors import CameraModel
    return CameraModel.from_dict(d)


def _flat(name):
    from paper_2507_18713_b200.scene import flatten_scene
    return flatten_scene(load_golden_scene(name))


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def assert_image_close(got, want):
    assert_image(got, want)


@pytest.fixture(scope="module")
def rand300_mag(golden, golden_meta):
    """Conditioning scale of the rand300 raster-backward golden (oracle raster records)."""
    sc = load_golden_scene("rand300")
    vox = oracle_voxels(sc)
    rec = O.raster_records(vox, oracle_camera(golden_meta["rand300_cam"]), background=(0.05, 0.1, 0.15))
    return magnitude(rec, vox, golden["rand300_rbw_dcolor"], golden["rand300_rbw_ddepth"])


@pytest.fixture(scope="module")
def ray_mag(golden):
    """Conditioning scales of the integ / fd ray-backward goldens (oracle ray records)."""
    out = {}
    for case, name in (("integ", "rand300i"), ("fd", "fd10")):
        bg = (0.2, 0.1, 0.3) if case == "integ" else golden["fd_bg"]
        vox = oracle_voxels(load_golden_scene(name))
        rec = O.integrate_rays(vox, O.build_octree(vox), golden[case + "_o"], golden[case + "_d"], background=bg)
        out[case] = magnitude(rec, vox, golden[case + "_dcolor"], golden[case + "_ddepth"])
    return out


# ---- rasterizer -----------------------------------------------------------------

def test_project_voxels_bit_exact(golden, golden_meta):
    from paper_2507_18713_b200 import render_raster as RR
    rmin, rmax, zc, culled = RR.project_voxels(_flat("rand400"), _cam(golden_meta["rand400_cam"]))
    np.testing.assert_array_equal(culled, golden["rand400_culled"])
    np.testing.assert_array_equal(zc, golden["rand400_zc"])
    np.testing.assert_array_equal(rmin, golden["rand400_rmin"])
    np.testing.assert_array_equal(rmax, golden["rand400_rmax"])


def test_cull_and_bin_bit_exact(golden, golden_meta):
    from paper_2507_18713_b200 import render_raster as RR
    bins = RR.cull_and_bin(_flat("rand400"), _cam(golden_meta["rand400_cam"]))
    np.testing.assert_array_equal(bins.offsets, golden["rand400_offsets"])
    np.testing.assert_array_equal(bins.entries, golden["rand400_entries"])


def test_cull_and_bin_c1_bit_exact(golden, golden_meta):
    """C1: S20k (reference CLI bytes) at 256^2: 385,735 instances, bit for bit."""
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    from paper_2507_18713_b200.scenes import make_init_scene
    bins = RR.cull_and_bin(flatten_scene(make_init_scene("S20k")), _cam(golden_meta["c1_cam"]))
    np.testing.assert_array_equal(bins.offsets, golden["c1_offsets"])
    np.testing.assert_array_equal(bins.entries, golden["c1_entries"])


def test_render_bins_are_subsequences(golden, golden_meta):
    """Tightened render lists keep the reference order and drop only straddlers."""
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    from paper_2507_18713_b200.scenes import make_init_scene
    flat = flatten_scene(make_init_scene("S20k"))
    cam = _cam(golden_meta["c1_cam"])
    fit = RR.render_bins(flat, cam)
    off, ent = golden["c1_offsets"], golden["c1_entries"]
    assert fit.entries.size < ent.size
    for t in range(len(off) - 1):
        ref = ent[off[t]:off[t + 1]]
        got = fit.entries[fit.offsets[t]:fit.offsets[t + 1]]
        assert np.array_equal(ref[np.isin(ref, got)], got), f"tile {t} order differs"


@pytest.mark.parametrize("exact", [True, False])
def test_rasterize_matches_reference(golden, golden_meta, exact):
    from paper_2507_18713_b200 import render_raster as RR
    fb = RR.rasterize(_flat("rand400"), _cam(golden_meta["rand400_cam"]), background=(0.1, 0.2, 0.3),
                      exact_color=exact)
    assert_image_close(_np(fb.color), golden["rand400_color"])
    assert_image_close(_np(fb.opacity), golden["rand400_opacity"])
    assert_image_close(_np(fb.depth), golden["rand400_depth"])


def test_rasterize_c1_matches_reference(golden, golden_meta):
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    from paper_2507_18713_b200.scenes import make_init_scene
    fb = RR.rasterize(flatten_scene(make_init_scene("S20k")), _cam(golden_meta["c1_cam"]))
    assert_image_close(_np(fb.color), golden["c1_color"])
    assert_image_close(_np(fb.opacity), golden["c1_opacity"])
    assert_image_close(_np(fb.depth), golden["c1_depth"])


def test_tile_size_is_scheduling_only(golden_meta):
    """test_render_raster.py:140-150: tile 1 == tile 16 bit for bit."""
    from paper_2507_18713_b200 import render_raster as RR
    flat, cam = _flat("rand400"), _cam(golden_meta["rand400_cam"])
    a = RR.rasterize(flat, cam, tile=16)
    b = RR.rasterize(flat, cam, tile=1)
    assert torch.equal(a.color, b.color) and torch.equal(a.opacity, b.opacity)
    assert torch.equal(torch.nan_to_num(a.depth, 7.0), torch.nan_to_num(b.depth, 7.0))


@pytest.mark.parametrize("tile", [1, 5, 8, 13])
@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_tile_size_scheduling_backward(golden, golden_meta, tile, exact):
    """The tile size only schedules work: frames and gradients for tile sizes
    1..16 (incl. non-divisors of the image) agree with tile 16 (gradients up
    to fp32 partial-sum order)."""
    from paper_2507_18713_b200 import render_raster as RR
    cam = _cam(golden_meta["rand300_cam"])
    flat = _flat("rand300")
    h, w = cam.height, cam.width
    dc, dd = golden["rand300_rbw_dcolor"].reshape(h, w, 3), golden["rand300_rbw_ddepth"].reshape(h, w)
    fa, sa = RR.rasterize(flat, cam, tile=16, return_state=True, exact_color=exact)
    fb, sb = RR.rasterize(flat, cam, tile=tile, return_state=True, exact_color=exact)
    assert torch.equal(fa.color, fb.color) and torch.equal(fa.opacity, fb.opacity)
    ga = RR.rasterize_backward(sa, dc, dd, as_dict=False)
    gb = RR.rasterize_backward(sb, dc, dd, as_dict=False)
    err = ((ga - gb).abs().max(dim=0).values / ga.abs().max(dim=0).values.clamp_min(1e-30)).max()
    assert float(err) < 1e-5, float(err)


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_raster_backward_matches_reference_composition(golden, golden_meta, exact, rand300_mag):
    """exact: the fp64 backward; mixed: the default fp64-geometry / fp32-field backward."""
    from paper_2507_18713_b200 import render_raster as RR
    cam = _cam(golden_meta["rand300_cam"])
    fb, st = RR.rasterize(_flat("rand300"), cam, background=(0.05, 0.1, 0.15), return_state=True,
                          exact_color=exact)
    h, w = cam.height, cam.width
    g = RR.rasterize_backward(st, golden["rand300_rbw_dcolor"].reshape(h, w, 3),
                              golden["rand300_rbw_ddepth"].reshape(h, w))
    want = {k: golden["rand300_rbw_g_" + k] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    assert_grads(g, want, rand300_mag)


# ---- octree / ray path ----------------------------------------------------------

def test_octree_and_query_bit_exact(golden):
    from paper_2507_18713_b200.octree import build_octree, query_batch
    tree = build_octree(load_golden_scene("rand400m").static)
    np.testing.assert_array_equal(tree.nodes_id, golden["march_nodes_id"])
    np.testing.assert_array_equal(tree.nodes_leaf, golden["march_nodes_leaf"])
    fl, vid, corner, edge = query_batch(tree, golden["query_p"])
    np.testing.assert_array_equal(fl, golden["query_flag"])
    np.testing.assert_array_equal(vid, golden["query_vid"])
    np.testing.assert_array_equal(corner, golden["query_corner"])
    np.testing.assert_array_equal(edge, golden["query_edge"])


def test_march_hit_list_bit_exact(golden):
    from paper_2507_18713_b200.octree import build_octree, march_batch
    tree = build_octree(load_golden_scene("rand400m").static)
    ray, vid, t0, t1 = march_batch(tree, golden["march_o"], golden["march_d"])
    for a, k in ((ray, "ray"), (vid, "vid"), (t0, "t0"), (t1, "t1")):
        np.testing.assert_array_equal(a, golden["march_" + k])


@pytest.mark.parametrize("exact", [True, False])
def test_integrate_rays_matches_reference(golden, exact):
    from paper_2507_18713_b200 import render_ray as RY
    sc = load_golden_scene("rand300i")
    rec = RY.integrate_rays(sc, RY.build_scene_octrees(sc), golden["integ_o"], golden["integ_d"],
                            background=(0.2, 0.1, 0.3), exact_color=exact)
    assert int(rec.status.max()) == 0
    assert_image_close(_np(rec.out_color), golden["integ_color"])
    assert_image_close(_np(rec.opacity), 1.0 - golden["integ_tfinal"])
    assert_image_close(_np(rec.depth), golden["integ_depth"])
    # exact mode: the fp64 reference-order sums; default mode: 1 - exp(-Y) from the certified fp32 Y
    tol = dict(rtol=1e-12, atol=1e-13) if exact else dict(rtol=0, atol=2e-6)
    np.testing.assert_allclose(_np(rec.weight_sum), golden["integ_wsum"], **tol)
    if not exact:  # every reference decision certified: depth-NaN mask and the 0.5 threshold identical
        np.testing.assert_array_equal(_np(rec.weight_sum) > 0.5, golden["integ_wsum"] > 0.5)
    # early-stopped hit list (ray, vid, t0) bit-exact
    ray, vid, t0, t1 = (x.cpu().numpy() for x in RY.segments(sc, RY.build_scene_octrees(sc),
                                                                golden["integ_o"], golden["integ_d"]))
    np.testing.assert_array_equal(ray, golden["integ_ray"])
    np.testing.assert_array_equal(vid, golden["integ_vid"])
    np.testing.assert_array_equal(t0, golden["integ_t0"])
    np.testing.assert_array_equal(t1, golden["integ_t1"])


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
@pytest.mark.parametrize("case", ["integ", "fd"])
def test_ray_backward_matches_reference(golden, case, exact, ray_mag):
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_records
    name = {"integ": "rand300i", "fd": "fd10"}[case]
    bg = (0.2, 0.1, 0.3) if case == "integ" else golden["fd_bg"]
    sc = load_golden_scene(name)
    rec = RY.integrate_rays(sc, RY.build_scene_octrees(sc), golden[case + "_o"], golden[case + "_d"],
                            background=bg, exact_color=exact)
    g = backward_records(rec, sc, golden[case + "_dcolor"], golden[case + "_ddepth"])["static"]
    want = {k: golden[f"{case}_g_{k}"] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    assert_grads(g, want, ray_mag[case])


def test_ray_image_matches_reference(golden, golden_meta):
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.sensors import camera_rays
    sc = load_golden_scene("rand300")
    color, op, depth = RY.render_rays_image(sc, RY.build_scene_octrees(sc),
                                            camera_rays(_cam(golden_meta["rand300_cam"])))
    assert_image_close(_np(color), golden["rand300_ray_color"])
    assert_image_close(_np(op), golden["rand300_ray_opacity"])
    assert_image_close(_np(depth), golden["rand300_ray_depth"])


# ---- sensors --------------------------------------------------------------------

@pytest.mark.parametrize("name", ["pin", "fish", "eq", "lidar"])
def test_sensor_rays_match_reference(golden, golden_meta, name):
    from paper_2507_18713_b200 import sensors as S
    d = golden_meta["rays_" + name]
    if name == "lidar":
        b = S.gen_lidar_rays(S.sensor_from_dict(d), t0=0.5)
    else:
        b = S.camera_rays(S.CameraModel.from_dict(d))
    np.testing.assert_allclose(_np(b.origins), golden[f"rays_{name}_o"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(_np(b.dirs), golden[f"rays_{name}_d"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(_np(b.t_stamps), golden[f"rays_{name}_t"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(b.valid.cpu().numpy(), golden[f"rays_{name}_valid"])


def test_lidar_ranges_and_extension(golden):
    """render_lidar_ranges equals integrate_rays' depth; the intensity / ray-drop
    extension blends features with the reference's own weights (the blended
    feature is pinned through the oracle's weights; the head has no reference)."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.sensors import RayBatch
    sc = load_golden_scene("rand300i")
    oc = RY.build_scene_octrees(sc)
    o, d = golden["integ_o"], golden["integ_d"]
    n = o.shape[0]
    b = RayBatch(torch.as_tensor(o, device="cuda"), torch.as_tensor(d, device="cuda"),
                 torch.zeros(n, device="cuda"), torch.zeros((n, 2), device="cuda"),
                 torch.ones(n, dtype=torch.bool, device="cuda"), (n,))
    dep = RY.render_lidar_ranges(sc, oc, b)
    assert_image_close(_np(dep), golden["integ_depth"])
    rng = np.random.default_rng(5)
    feat = rng.uniform(-1, 1, (sc.static.n, 8)).astype(np.float32)
    head = rng.uniform(-0.5, 0.5, (2, 13)).astype(np.float32)
    ret = RY.render_lidar(sc, oc, b, features=feat, head=head, want_feature=True)
    # oracle: F = sum_i w_i f_vid_i over included segments, with the reference's weights
    vox = oracle_voxels(sc)
    rec = O.integrate_rays(vox, O.build_octree(vox), o, d)
    w = np.where(rec["included"], rec["t_before"] * np.clip(rec["alpha"], 0, O.ALPHA_MAX), 0.0)
    F = np.zeros((n, 8))
    np.add.at(F, rec["ray"], w[:, None] * feat[rec["vid"]].astype(np.float64))
    np.testing.assert_allclose(_np(ret.feature), F, atol=1e-5)
    D = np.nan_to_num(rec["depth"], nan=0.0)
    z = F @ head[:, :8].T.astype(np.float64) + D[:, None] * head[:, 8] + d @ head[:, 9:12].T + head[:, 12]
    ref = 1.0 / (1.0 + np.exp(-z))
    np.testing.assert_allclose(_np(ret.intensity), ref[:, 0], atol=1e-5)
    np.testing.assert_allclose(_np(ret.drop_prob), ref[:, 1], atol=1e-5)


def test_lidar_extension_backward():
    """Backward of the intensity / ray-drop extension: head, feature and field
    gradients against the oracle's restatement of the reference chain with the
    colour replaced by the blended feature."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.sensors import RayBatch
    from conftest import load_golden_scene as lgs
    sc = lgs("rand300i")
    oc = RY.build_scene_octrees(sc)
    rng = np.random.default_rng(11)
    n = 300
    o = rng.uniform(-1, 9, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    b = RayBatch(torch.as_tensor(o, device="cuda"), torch.as_tensor(d, device="cuda"),
                 torch.zeros(n, device="cuda"), torch.zeros((n, 2), device="cuda"),
                 torch.ones(n, dtype=torch.bool, device="cuda"), (n,))
    feat = rng.uniform(-1, 1, (sc.static.n, 8)).astype(np.float32)
    head = rng.uniform(-0.5, 0.5, (2, 13)).astype(np.float32)
    ret = RY.render_lidar(sc, oc, b, features=feat, head=head, want_feature=True)
    d_dep, d_int, d_drop = rng.normal(size=n) * 0.1, rng.normal(size=n), rng.normal(size=n)
    grad, fgrad, hgrad = RY.lidar_backward(ret, d_dep, features=feat, head=head, d_intensity=d_int,
                                           d_drop=d_drop)
    vox = oracle_voxels(sc)
    rec = O.integrate_rays(vox, O.build_octree(vox), o, d)
    w = np.where(rec["included"], rec["t_before"] * np.clip(rec["alpha"], 0, O.ALPHA_MAX), 0.0)
    F = np.zeros((n, 8))
    np.add.at(F, rec["ray"], w[:, None] * feat[rec["vid"]].astype(np.float64))
    valid = rec["weight_sum"] > 0.5
    D = np.where(valid, np.nan_to_num(rec["depth"]), 0.0)
    z_in = np.concatenate([F, D[:, None], d], 1)
    W = head.astype(np.float64)
    out = 1.0 / (1.0 + np.exp(-(z_in @ W[:, :12].T + W[:, 12])))
    dz = np.stack([d_int, d_drop], 1) * out * (1 - out)
    h_ref = np.concatenate([dz.T @ z_in, dz.sum(0)[:, None]], 1)
    np.testing.assert_allclose(hgrad.cpu().numpy(), h_ref, rtol=1e-4, atol=1e-6)
    dF = dz @ W[:, :8]
    dd = d_dep + np.where(valid, dz @ W[:, 8], 0.0)
    g_ref, f_ref = O.feature_backward(rec, vox, feat.astype(np.float64), dF, dd)
    from parity import GRAD_COND, X_FLOOR, assert_ok, elementwise, grad_report
    g_mag, f_mag = O.feature_backward(rec, vox, feat.astype(np.float64), dF, dd, magnitude=True, x_floor=X_FLOOR)
    fg = fgrad.cpu().numpy()
    assert_ok(elementwise(fg, f_ref, floor=1e-9 * np.abs(f_ref).max(), mag=f_mag, cond=GRAD_COND, name="feature"))
    from paper_2507_18713_b200.device import grads_to_dict
    assert_ok(grad_report(grads_to_dict(grad[: sc.static.n]), g_ref, g_mag, keys=("w_s", "log_a", "log_b")))


def test_dynamic_actors_ray_path(golden):
    """integrate_rays with two moving/rotating actors (render_ray.py:161-239):
    merged hit lists bit-identical to the reference's, colours/depths within
    1e-4, backward gradients per owner (static + each actor) within 1e-4."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_records
    sc = load_golden_scene("actors")
    assert [a.actor_id for a in sc.actors] == ["cart", "box"]
    oc = RY.build_scene_octrees(sc)
    rec = RY.integrate_rays(sc, oc, golden["act_o"], golden["act_d"], golden["act_t"],
                            background=(0.1, 0.2, 0.05), exact_color=True)
    assert_image_close(_np(rec.out_color), golden["act_color"])
    assert_image_close(_np(rec.opacity), golden["act_opacity"])
    assert_image_close(_np(rec.depth), golden["act_depth"])
    # actor segments of the merged list, in the reference's (ray, t0, owner, vid) order
    r = rec.ex_rec.cpu().numpy()
    start = rec.ex_start.cpu().numpy()
    ray = np.repeat(np.arange(len(start) - 1), np.diff(start))
    m = golden["act_owner"] >= 0
    np.testing.assert_array_equal(ray, golden["act_ray"][m])
    np.testing.assert_array_equal(r[: ray.size, 20].astype(int), golden["act_owner"][m])
    offs = {0: 0, 1: sc.actors[0].voxels.n}
    np.testing.assert_array_equal(r[: ray.size, 21].astype(int) - np.array([offs[o] for o in golden["act_owner"][m]]),
                                  golden["act_vid"][m])
    np.testing.assert_array_equal(r[: ray.size, 0], golden["act_t0"][m])
    g = backward_records(rec, sc, golden["act_dcolor"], golden["act_ddepth"])
    for own in ("static", "cart", "box"):
        want = {k: golden[f"act_g_{own}_{k}"] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
        assert_grads(g[own], want)


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_dynamic_actors_raster_path(golden, golden_meta, exact):
    """rasterize with the actors flattened at t = 0.7 (rotated voxels,
    render_raster.py:63-129, :185-198): bit-exact CSR, colours, and the raster
    backward through rotated voxels."""
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scene import flatten_scene
    sc = load_golden_scene("actors")
    flat = flatten_scene(sc, 0.7)
    cam = _cam(golden_meta["actr_cam"])
    bins = RR.cull_and_bin(flat, cam)
    np.testing.assert_array_equal(bins.offsets, golden["actr_offsets"])
    np.testing.assert_array_equal(bins.entries, golden["actr_entries"])
    fb, st = RR.rasterize(flat, cam, background=(0.1, 0.2, 0.05), return_state=True, exact_color=exact)
    assert_image_close(_np(fb.color), golden["actr_color"])
    assert_image_close(_np(fb.depth), golden["actr_depth"])
    g = RR.rasterize_backward(st, golden["actr_dcolor"].reshape(48, 64, 3), np.zeros((48, 64)))
    want = {k: golden["actr_g_" + k] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    assert_grads(g, want)


@pytest.mark.parametrize("exact", [True, False], ids=["fp64", "mixed"])
def test_raster_backward_deterministic_mode(golden, golden_meta, exact, rand300_mag):
    """Deterministic gradient mode: the
    reference composition to 1e-4 and bitwise identical across reruns."""
    from paper_2507_18713_b200 import render_raster as RR
    cam = _cam(golden_meta["rand300_cam"])
    fb, st = RR.rasterize(_flat("rand300"), cam, background=(0.05, 0.1, 0.15), return_state=True,
                          exact_color=exact)
    h, w = cam.height, cam.width
    dc, dd = golden["rand300_rbw_dcolor"].reshape(h, w, 3), golden["rand300_rbw_ddepth"].reshape(h, w)
    runs = [RR.rasterize_backward(st, dc, dd, as_dict=False, deterministic=True) for _ in range(3)]
    assert all(torch.equal(runs[0], r) for r in runs[1:])
    want = {k: golden["rand300_rbw_g_" + k] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    from paper_2507_18713_b200.device import grads_to_dict
    assert_grads(grads_to_dict(runs[0]), want, rand300_mag)
    atomic = RR.rasterize_backward(st, dc, dd, as_dict=False)
    # the atomic mode adds each warp's fp32 entry totals in fp64, the deterministic mode rounds
    # a tile's sum over its warps to one fp32 partial row: they differ by that rounding
    # (<= 2^-24 of a tile partial), bounded here per parameter column
    col_max = atomic.abs().amax(dim=0, keepdim=True).clamp_min(1e-300)
    assert bool(((runs[0] - atomic).abs() <= 1e-6 * atomic.abs() + 1e-6 * col_max).all())


@pytest.mark.parametrize("case", ["integ", "fd"])
def test_ray_backward_deterministic_mode(golden, case, ray_mag):
    """Ray-path deterministic gradients: reference values to 1e-4, bitwise
    identical across reruns, and equal to the atomic mode up to summation order."""
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import backward_grad_buffer
    from paper_2507_18713_b200.device import grads_to_dict
    name = {"integ": "rand300i", "fd": "fd10"}[case]
    bg = (0.2, 0.1, 0.3) if case == "integ" else golden["fd_bg"]
    sc = load_golden_scene(name)
    rec = RY.integrate_rays(sc, RY.build_scene_octrees(sc), golden[case + "_o"], golden[case + "_d"],
                            background=bg, exact_color=True)
    dc, dd = golden[case + "_dcolor"], golden[case + "_ddepth"]
    runs = [backward_grad_buffer(rec, dc, dd, deterministic=True) for _ in range(3)]
    assert all(torch.equal(runs[0], r) for r in runs[1:])
    want = {k: golden[f"{case}_g_{k}"] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    assert_grads(grads_to_dict(runs[0][: sc.static.n]), want, ray_mag[case])
    torch.testing.assert_close(runs[0], backward_grad_buffer(rec, dc, dd), rtol=1e-6, atol=1e-12)
