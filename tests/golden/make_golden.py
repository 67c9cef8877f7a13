"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where the read-only reference is importable):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every expected array below is produced by calling the reference's own public
functions (salf.render_raster / render_ray / octree / backward / sensors) on
scenes that are first round-tripped through the salf.v1 container, so the
GPU side loads exactly the same bytes.  The outputs are committed; nothing at
test time (or on the GPU box) needs /root/reference.
"""

from __future__ import annotations

import json
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from conftest import make_random_scene, random_rays  # noqa: E402  (reference test helpers)
from fd_fixture import build_fixture  # noqa: E402
from salf import backward as R_bw  # noqa: E402
from salf import container as R_io  # noqa: E402
from salf import octree as R_oct  # noqa: E402
from salf import render_raster as R_ras  # noqa: E402
from salf import render_ray as R_ray  # noqa: E402
from salf import sensors as R_sen  # noqa: E402
from salf.bench import scale_camera  # noqa: E402
from salf.losses import loss_color, loss_depth  # noqa: E402
from salf.scene import Scene, SceneBounds, SparseVoxelSet  # noqa: E402
from salf.synthetic import look_at_quaternion  # noqa: E402

SCENES = HERE / "scenes"


def cam_at(position, target, width=64, height=64, f=80.0):
    return R_sen.CameraModel(kind="pinhole", width=width, height=height, fx=f, fy=f,
                             cx=width / 2.0, cy=height / 2.0,
                             position=np.asarray(position, np.float64),
                             quaternion=look_at_quaternion(position, target))


def roundtrip(name, scene):
    """Save as salf.v1 and reload: params become the f32 values both sides use."""
    R_io.save_scene(scene, SCENES / name)
    return R_io.load_scene(SCENES / name)


def cam_dict(cam):
    return R_io.sensor_to_dict(cam)


def raster_band(args):
    path, cam_d, r0, r1 = args
    scene = R_io.load_scene(path)
    cam = R_io.sensor_from_dict(cam_d)
    flat = R_ras.flatten_scene(scene)
    # rows r0..r1 of a full-size frame: render a camera cropped to the band
    # by shifting cy (tiles are rows of 16, r0 is a multiple of 16)
    band = R_sen.CameraModel(kind="pinhole", width=cam.width, height=r1 - r0, fx=cam.fx, fy=cam.fy,
                             cx=cam.cx, cy=cam.cy - r0, position=cam.position,
                             quaternion=cam.quaternion)
    fb = R_ras.rasterize(flat, band)
    return r0, fb.color, fb.opacity, fb.depth


def raster_records_reference(flat, cam, background):
    """Raster pairs -> RenderRecords using reference functions only."""
    bins = R_ras.cull_and_bin(flat, cam)
    batch = R_sen.gen_camera_rays(cam)
    dirs = batch.dirs
    t_near = R_ras.NEAR_PLANE / (dirs @ cam.rotation_matrix())[:, 2]
    h, w, tile = cam.height, cam.width, bins.tile
    rays, vids, t0s, t1s, os_, ds_ = [], [], [], [], [], []
    for t in range(bins.tiles_x * bins.tiles_y):
        ent = bins.entries[bins.offsets[t]:bins.offsets[t + 1]]
        if ent.size == 0:
            continue
        ty, tx = divmod(t, bins.tiles_x)
        rr = np.arange(ty * tile, min((ty + 1) * tile, h))
        cc = np.arange(tx * tile, min((tx + 1) * tile, w))
        px = (rr[:, None] * w + cc[None, :]).ravel()
        pp, vv = np.repeat(px, ent.size), np.tile(ent, px.size)
        o, d, t_in, t_out = R_ras._pair_fields(flat, np.broadcast_to(cam.position, (pp.size, 3)),
                                               dirs[pp], vv)
        t0 = np.maximum(np.maximum(t_in, t_near[pp]), 0.0)
        hit = t_out > t0 + 1e-12
        rays.append(pp[hit]); vids.append(vv[hit]); t0s.append(t0[hit]); t1s.append(t_out[hit])
        os_.append(o[hit]); ds_.append(d[hit])
    ray = np.concatenate(rays); vid = np.concatenate(vids)
    t0 = np.concatenate(t0s); t1 = np.concatenate(t1s)
    o_all, d_all = np.concatenate(os_), np.concatenate(ds_)
    order = np.argsort(ray, kind="stable")
    ray, vid, t0, t1 = ray[order], vid[order], t0[order], t1[order]
    from salf.scene import eval_color, eval_sdf, sdf_to_density, segment_opacity
    tm = 0.5 * (t0 + t1)
    o = o_all[order]  # pair-frame origin / direction (rotated for actor voxels, :191-196)
    d = d_all[order]
    x = (o + tm[:, None] * d) / (0.5 * flat.edges[vid])[:, None]
    s = eval_sdf(x, flat.w_s[vid])
    sig = sdf_to_density(s, np.exp(flat.log_a[vid]), np.exp(flat.log_b[vid]))
    alpha = segment_opacity(sig, t1 - t0)
    color = eval_color(x, d, flat.w_c[vid], flat.w_sh[vid])
    bg = np.asarray(background, np.float64)
    (t_before, included, _w, out_color, opacity, depth, weight_sum, t_final,
     starts) = R_ray._composite(ray, alpha, color, tm, h * w, bg, R_ray.STOP_THRESHOLD)
    owner = np.full(ray.size, R_ray.STATIC_OWNER, np.int32)
    return R_ray.RenderRecords(
        n_rays=h * w, ray=ray, owner=owner, vid=vid, t0=t0, t1=t1, x=x, omega=d, s_field=s,
        sigma=sig, alpha=alpha, color=color, t_before=t_before, included=included,
        out_color=out_color, opacity=opacity, depth=depth, weight_sum=weight_sum, t_final=t_final,
        background=bg, density_mode="sdf", group_start=starts)


def _flat_set(flat, bounds):
    """A SparseVoxelSet view of flattened voxels (only the params are used by
    backward_records' 'static' owner)."""
    v = SparseVoxelSet(bounds, budget=flat.n + 1)
    v.level = np.zeros(flat.n, np.uint8)
    v.ijk = np.zeros((flat.n, 3), np.int32)
    v.w_s, v.w_c, v.w_sh, v.log_a, v.log_b = flat.w_s, flat.w_c, flat.w_sh, flat.log_a, flat.log_b
    v.rotation = flat.rotations
    return v


def main():
    SCENES.mkdir(parents=True, exist_ok=True)
    out = {}
    meta = {}

    # 1. binning / projection / raster on a random multi-level scene (test_render_raster.py:80-91)
    sc = roundtrip("rand400", make_random_scene(61, 400))
    cam = cam_at([12.0, 12.0, 6.0], [4.0, 4.0, 2.0])
    flat = R_ras.flatten_scene(sc)
    bins = R_ras.cull_and_bin(flat, cam)
    rmin, rmax, zc, culled = R_ras.project_voxels(flat, cam)
    fb = R_ras.rasterize(flat, cam, background=(0.1, 0.2, 0.3))
    out.update(rand400_offsets=bins.offsets, rand400_entries=bins.entries, rand400_rmin=rmin,
               rand400_rmax=rmax, rand400_zc=zc, rand400_culled=culled, rand400_color=fb.color,
               rand400_opacity=fb.opacity, rand400_depth=fb.depth)
    meta["rand400_cam"] = cam_dict(cam)

    # 2. raster vs ray on the L1 scene (test_render_raster.py:160-166)
    sc = roundtrip("rand300", make_random_scene(65, 300, a_range=(1.0, 6.0)))
    cam = cam_at([13.0, 11.0, 7.0], [4.0, 4.0, 2.0], width=96, height=96, f=90.0)
    fb = R_ras.rasterize_scene(sc, cam)
    oc = R_ray.build_scene_octrees(sc)
    color, opac, depth = R_ray.render_rays_image(sc, oc, R_sen.camera_rays(cam))
    out.update(rand300_raster_color=fb.color, rand300_raster_opacity=fb.opacity,
               rand300_raster_depth=fb.depth, rand300_ray_color=color, rand300_ray_opacity=opac,
               rand300_ray_depth=depth)
    meta["rand300_cam"] = cam_dict(cam)
    # raster backward oracle built from reference functions, L1 seeds vs a constant target
    flat = R_ras.flatten_scene(sc)
    rec = raster_records_reference(flat, cam, (0.05, 0.1, 0.15))
    gt = np.full((cam.height * cam.width, 3), 0.4)
    _, d_c = loss_color(rec, gt, np.ones(rec.n_rays, bool))
    gtd = np.full(rec.n_rays, 9.0)
    _, d_d = loss_depth(rec, gtd, np.ones(rec.n_rays, bool))
    g = R_bw.backward_records(rec, sc, d_c, 0.1 * d_d)["static"]
    out.update(rand300_rbw_out_color=rec.out_color, rand300_rbw_depth=rec.depth,
               rand300_rbw_dcolor=d_c, rand300_rbw_ddepth=0.1 * d_d,
               **{f"rand300_rbw_g_{k}": v for k, v in g.items()})

    # 3. march vs reference march_batch (test_octree.py:173-186)
    sc = roundtrip("rand400m", make_random_scene(21, 400))
    buf = R_oct.build_octree(sc.static)
    rng = np.random.default_rng(22)
    o, d = random_rays(rng, 500, [0, 0, 0], [8, 8, 8])
    ray, vid, t0, t1 = R_oct.march_batch(buf, o, d)
    out.update(march_o=o, march_d=d, march_ray=ray, march_vid=vid, march_t0=t0, march_t1=t1,
               march_nodes_id=buf.nodes_id, march_nodes_leaf=buf.nodes_leaf)
    qp = np.random.default_rng(23).uniform(0, 8, size=(3000, 3))
    fl, qv, qc, qe = R_oct.query_batch(buf, qp)
    out.update(query_p=qp, query_flag=fl, query_vid=qv, query_corner=qc, query_edge=qe)

    # 4. integrate with early stop (test_render_ray.py:137-154) + backward with L1 seeds
    sc = roundtrip("rand300i", make_random_scene(45, 300, a_range=(2.0, 8.0)))
    oc = R_ray.build_scene_octrees(sc)
    rng = np.random.default_rng(46)
    o, d = random_rays(rng, 100, [0, 0, 0], [8, 8, 8])
    rec = R_ray.integrate_rays(sc, oc, o, d, background=(0.2, 0.1, 0.3))
    cam_mask = np.arange(100) < 66
    gt_c = np.random.default_rng(47).uniform(0, 1, (66, 3))
    gt_r = np.random.default_rng(48).uniform(0.5, 6.0, 34)
    _, d_c = loss_color(rec, gt_c, cam_mask)
    _, d_d = loss_depth(rec, gt_r, ~cam_mask)
    g = R_bw.backward_records(rec, sc, d_c, 10.0 * d_d)["static"]
    out.update(integ_o=o, integ_d=d, integ_color=rec.out_color, integ_opacity=rec.opacity,
               integ_depth=rec.depth, integ_wsum=rec.weight_sum, integ_tfinal=rec.t_final,
               integ_ray=rec.ray, integ_vid=rec.vid, integ_t0=rec.t0, integ_t1=rec.t1,
               integ_dcolor=d_c, integ_ddepth=10.0 * d_d,
               **{f"integ_g_{k}": v for k, v in g.items()})

    # 5. the FD fixture scene (fd_fixture.py:16-50): ray backward
    fx = build_fixture(n_voxels=10, n_rays=50, seed=5)
    sc = roundtrip("fd10", fx["scene"])
    oc = R_ray.build_scene_octrees(sc)
    rec = R_ray.integrate_rays(sc, oc, fx["origins"], fx["dirs"], background=fx["background"])
    _, d_c = loss_color(rec, fx["gt_colors"], fx["cam_mask"])
    _, d_d = loss_depth(rec, fx["gt_ranges"], ~fx["cam_mask"])
    g = R_bw.backward_records(rec, sc, d_c, 10.0 * d_d)["static"]
    out.update(fd_o=fx["origins"], fd_d=fx["dirs"], fd_bg=fx["background"], fd_color=rec.out_color,
               fd_depth=rec.depth, fd_dcolor=d_c, fd_ddepth=10.0 * d_d,
               **{f"fd_g_{k}": v for k, v in g.items()})

    # 5b. regularisers + Adam on the FD scene (losses.py:49-249, optim.py:48-62)
    from salf.losses import loss_eikonal, loss_empty, loss_opacity_lidar, loss_smooth
    from salf.optim import AdamConfig, AdamState, adam_step
    vs = sc.static
    all_idx = np.arange(vs.n)
    outer = np.flatnonzero(sc.outer_voxel_mask())
    l_e, g_e = loss_eikonal(vs, all_idx)
    l_m, g_m = loss_empty(vs, outer)
    l_o, g_o = loss_opacity_lidar(vs, oc.static, fx["points"])
    l_s, g_s = loss_smooth(vs, oc.static, all_idx)
    out.update(reg_smooth_loss=np.array([l_s]), **{f"reg_smo_{k}": v for k, v in g_s.items()})
    sm = make_random_scene(13, 60)
    sm = roundtrip("rand60s", sm)
    oc_sm = R_ray.build_scene_octrees(sm)
    sm_idx = np.unique(np.random.default_rng(3).integers(0, sm.static.n, 40))
    l_s2, g_s2 = loss_smooth(sm.static, oc_sm.static, sm_idx)
    out.update(reg_smooth2_idx=sm_idx, reg_smooth2_loss=np.array([l_s2]),
               **{f"reg_smo2_{k}": v for k, v in g_s2.items()})
    out.update(reg_points=fx["points"], reg_outer=outer, reg_loss=np.array([l_e, l_m, l_o]),
               reg_eik_w_s=g_e["w_s"], **{f"reg_emp_{k}": v for k, v in g_m.items()},
               **{f"reg_opa_{k}": v for k, v in g_o.items()})
    params = {k: getattr(vs, k).copy() for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    st = AdamState.for_params(params)
    cfg = AdamConfig(lr_decay_every=2)
    rng = np.random.default_rng(77)
    gseq = [{k: rng.normal(size=v.shape) for k, v in params.items()} for _ in range(3)]
    for gs in gseq:
        adam_step(params, gs, st, cfg)
    out.update(**{f"adam_g{i}_{k}": v for i, gs in enumerate(gseq) for k, v in gs.items()},
               **{f"adam_p_{k}": v for k, v in params.items()})

    # 5c. dynamic actors (render_ray.py:161-239; test_render_ray.py:323-402, test_backward.py:62-81)
    from salf.scene import Actor, make_actor_bounds
    bounds = SceneBounds([0, 0, 0], [4, 4, 4], base_edge=1.0, max_levels=3)
    static = SparseVoxelSet(bounds, budget=100)
    static.add_voxels([0, 0, 0], [[0, 1, 1], [3, 1, 1], [1, 3, 2]], rng=np.random.default_rng(8), a=5.0)
    a_bounds = make_actor_bounds([2.0, 2.0, 2.0], 1.0, max_levels=2)
    av = SparseVoxelSet(a_bounds, budget=20)
    av.add_voxels([0, 0, 1, 1], [[0, 0, 0], [1, 1, 1], [0, 3, 2], [2, 1, 0]], rng=np.random.default_rng(7),
                  a=np.array([30.0, 8.0, 20.0, 12.0]))
    yaw = lambda deg: np.array([np.cos(np.deg2rad(deg) / 2), 0.0, 0.0, np.sin(np.deg2rad(deg) / 2)])
    cart = Actor("cart", np.array([2.0, 2, 2]), av, times=np.array([0.0, 1.0, 2.0]),
                 positions=np.array([[2.0, 2.0, 2.0], [2.4, 2.1, 2.0], [3.0, 2.0, 2.2]]),
                 quaternions=np.stack([yaw(0.0), yaw(35.0), yaw(90.0)]))
    bv = SparseVoxelSet(make_actor_bounds([1.0, 1.0, 1.0], 0.5, max_levels=2), budget=10)
    bv.add_voxels([0], [[1, 0, 1]], rng=np.random.default_rng(17), a=15.0)
    box = Actor("box", np.array([1.0, 1.0, 1.0]), bv, times=np.array([0.0, 2.0]),
                positions=np.array([[1.5, 2.5, 1.0], [1.5, 2.5, 1.0]]),
                quaternions=np.array([yaw(20.0), yaw(20.0)]))
    sc = Scene(bounds=bounds, static=static, actors=[cart, box])
    sc = roundtrip("actors", sc)
    oc = R_ray.build_scene_octrees(sc)
    rng = np.random.default_rng(9)
    o = rng.uniform(-1.0, 5.0, (400, 3))
    d = (2.2 + rng.uniform(-1.2, 1.2, (400, 3))) - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ts = rng.uniform(0.0, 2.0, 400)
    rec = R_ray.integrate_rays(sc, oc, o, d, t_stamps=ts, background=(0.1, 0.2, 0.05))
    gt = np.random.default_rng(10).uniform(0, 1, (400, 3))
    _, d_c = loss_color(rec, gt, np.ones(400, bool))
    _, d_d = loss_depth(rec, np.full(400, 2.5), np.ones(400, bool))
    g = R_bw.backward_records(rec, sc, d_c, 0.3 * d_d)
    # raster with the actors flattened at t = 0.7 (rotated voxels, render_raster.py:63-89)
    cam = cam_at([-3.0, -2.0, 4.5], [2.0, 2.0, 1.8], width=64, height=48, f=50.0)
    flat = R_ras.flatten_scene(sc, 0.7)
    bins = R_ras.cull_and_bin(flat, cam)
    fb = R_ras.rasterize(flat, cam, background=(0.1, 0.2, 0.05))
    rr = raster_records_reference(flat, cam, (0.1, 0.2, 0.05))
    _, d_c2 = loss_color(rr, np.full((64 * 48, 3), 0.3), np.ones(rr.n_rays, bool))
    sc_flat = Scene(bounds=sc.bounds, static=sc.static)  # owner layout for backward_records
    g2 = R_bw.backward_records(rr, Scene(bounds=sc.bounds, static=_flat_set(flat, sc.bounds)), d_c2,
                               np.zeros(rr.n_rays))["static"]
    out.update(actr_offsets=bins.offsets, actr_entries=bins.entries, actr_color=fb.color,
               actr_opacity=fb.opacity, actr_depth=fb.depth, actr_dcolor=d_c2,
               **{f"actr_g_{k}": v for k, v in g2.items()})
    meta["actr_cam"] = cam_dict(cam)
    out.update(act_o=o, act_d=d, act_t=ts, act_color=rec.out_color, act_opacity=rec.opacity,
               act_depth=rec.depth, act_ray=rec.ray, act_owner=rec.owner, act_vid=rec.vid, act_t0=rec.t0,
               act_dcolor=d_c, act_ddepth=0.3 * d_d,
               **{f"act_g_{own}_{k}": v for own, gg in g.items() for k, v in gg.items()})

    # 6. sensors
    pin = R_sen.CameraModel(kind="pinhole", width=32, height=24, fx=30.0, fy=31.0, cx=15.5, cy=12.25,
                            position=np.array([0.3, -0.2, 1.1]),
                            quaternion=look_at_quaternion([0.3, -0.2, 1.1], [2.0, 1.0, 0.0]))
    fish = R_sen.CameraModel(kind="fisheye_equidistant", width=40, height=30, fx=12.0, fy=12.5, cx=20.0,
                             cy=15.0, distortion=(0.05, -0.01, 0.002, 0.0),
                             position=np.array([-1.0, 0.5, 1.5]),
                             quaternion=look_at_quaternion([-1.0, 0.5, 1.5], [1.0, 0.0, 0.5]),
                             readout_duration=0.03, linear_velocity=np.array([10.0, 0.0, 0.0]),
                             angular_velocity=np.array([0.0, 0.0, 0.2]))
    eq = R_sen.CameraModel(kind="equirect", width=16, height=8, position=np.array([0.0, 0.0, 1.0]))
    lid = R_sen.LidarModel(beam_elevations=np.linspace(-0.4, 0.25, 8), steps=90, scan_period=0.1,
                           position=np.array([0.0137, -0.0213, 1.3]),
                           quaternion=np.array([0.9961946980917455, 0.0, 0.0, 0.08715574274765817]),
                           linear_velocity=np.array([5.0, 0.0, 0.0]),
                           angular_velocity=np.array([0.0, 0.0, 0.3]))
    for name, b in (("pin", R_sen.camera_rays(pin)), ("fish", R_sen.camera_rays(fish)),
                    ("eq", R_sen.camera_rays(eq)), ("lidar", R_sen.gen_lidar_rays(lid, t0=0.5))):
        out.update({f"rays_{name}_o": b.origins, f"rays_{name}_d": b.dirs,
                    f"rays_{name}_t": b.t_stamps, f"rays_{name}_valid": b.valid})
    meta.update(rays_pin=cam_dict(pin), rays_fish=cam_dict(fish), rays_eq=cam_dict(eq),
                rays_lidar=R_io.sensor_to_dict(lid))

    # 7. C1: S20k (reference CLI scene) with cam_eval_000 scaled to 256^2
    s20 = Path("/tmp/gen/S_0.3")
    sc = R_io.load_scene(s20)
    sensors = json.loads((s20 / "sensors.json").read_text())["sensors"]
    cam = scale_camera(R_io.sensor_from_dict(sensors["cam_eval_000"]), 256)
    flat = R_ras.flatten_scene(sc)
    bins = R_ras.cull_and_bin(flat, cam)
    out.update(c1_offsets=bins.offsets, c1_entries=bins.entries.astype(np.int32))
    meta["c1_cam"] = cam_dict(cam)
    with ProcessPoolExecutor(8) as ex:
        parts = list(ex.map(raster_band, [(str(s20), cam_dict(cam), r, r + 32)
                                          for r in range(0, 256, 32)]))
    col = np.zeros((256, 256, 3)); opa = np.zeros((256, 256)); dep = np.zeros((256, 256))
    for r0, c, op, de in parts:
        col[r0:r0 + c.shape[0]] = c; opa[r0:r0 + c.shape[0]] = op; dep[r0:r0 + c.shape[0]] = de
    out.update(c1_color=col, c1_opacity=opa, c1_depth=dep)
    buf = R_oct.build_octree(sc.static)
    out.update(c1_nodes_id=buf.nodes_id, c1_nodes_leaf=buf.nodes_leaf)

    np.savez_compressed(HERE / "golden.npz", **out)
    (HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    # digests of the reference CLI scenes (the bench inputs)
    import hashlib
    dig = {}
    for name, d in (("S20k", "S_0.3"), ("S1M", "S_0.07"), ("S2M", "S_0.055")):
        p = Path("/tmp/gen") / d / "voxels.bin"
        if p.exists():
            dig[name] = hashlib.sha256(p.read_bytes()).hexdigest()
    (HERE / "scene_digests.json").write_text(json.dumps(dig, indent=1, sort_keys=True) + "\n")
    print("wrote", HERE / "golden.npz", sum(v.nbytes for v in out.values()) / 1e6, "MB raw")


if __name__ == "__main__":
    main()
