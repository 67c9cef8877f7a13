"""Elementwise parity report of the default (mixed-precision) and fp64 paths
against the oracle on the golden cases and full-size (C2/C3/C4) samples.

  python tools/parity_report.py [--out gpurun_out/parity_report.json] [--quick]

Writes one JSON document (tests/parity.py reports per output / gradient class).
GPU only; the oracle is the checker."""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import GOLDEN, load_golden_scene, oracle_voxels  # noqa: E402
from oracle import salf_oracle as O  # noqa: E402
from parity import grad_magnitude, grad_report, image_report  # noqa: E402


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def ocam_of(cam):
    return O.Camera(cam.kind, cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.distortion,
                    cam.position, cam.quaternion, cam.readout_duration, cam.linear_velocity,
                    cam.angular_velocity)


def golden_cases(out):
    from paper_2507_18713_b200 import render_raster as RR, render_ray as RY
    from paper_2507_18713_b200.backward import backward_records
    from paper_2507_18713_b200.scene import flatten_scene
    from paper_2507_18713_b200.sensors import CameraModel
    gd = np.load(GOLDEN / "golden.npz")
    meta = json.loads((GOLDEN / "golden_meta.json").read_text())
    cam = CameraModel.from_dict(meta["rand300_cam"])
    sc = load_golden_scene("rand300")
    h, w = cam.height, cam.width
    dc, dd = gd["rand300_rbw_dcolor"], gd["rand300_rbw_ddepth"]
    vox = oracle_voxels(sc)
    rec = O.raster_records(vox, ocam_of(cam), background=(0.05, 0.1, 0.15))
    mag = grad_magnitude(O, rec, vox, dc, dd)
    want = {k: gd["rand300_rbw_g_" + k] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
    for exact in (False, True):
        fb, st = RR.rasterize(flatten_scene(sc), cam, background=(0.05, 0.1, 0.15), return_state=True,
                              exact_color=exact)
        g = RR.rasterize_backward(st, dc.reshape(h, w, 3), dd.reshape(h, w))
        out[f"rand300_raster_grad_{'fp64' if exact else 'mixed'}"] = grad_report(g, want, mag)
        out[f"rand300_raster_grad_{'fp64' if exact else 'mixed'}_nomag"] = grad_report(g, want)
    for case, name in (("integ", "rand300i"), ("fd", "fd10")):
        bg = (0.2, 0.1, 0.3) if case == "integ" else gd["fd_bg"]
        sc = load_golden_scene(name)
        vox = oracle_voxels(sc)
        orec = O.integrate_rays(vox, O.build_octree(vox), gd[case + "_o"], gd[case + "_d"], background=bg)
        mag = grad_magnitude(O, orec, vox, gd[case + "_dcolor"], gd[case + "_ddepth"])
        want = {k: gd[f"{case}_g_{k}"] for k in ("w_s", "w_c", "w_sh", "log_a", "log_b")}
        for exact in (False, True):
            r = RY.integrate_rays(sc, RY.build_scene_octrees(sc), gd[case + "_o"], gd[case + "_d"],
                                  background=bg, exact_color=exact)
            g = backward_records(r, sc, gd[case + "_dcolor"], gd[case + "_ddepth"])["static"]
            tag = f"{case}_ray_{'fp64' if exact else 'mixed'}"
            out[tag + "_grad"] = grad_report(g, want, mag)
            out[tag + "_grad_nomag"] = grad_report(g, want)
            out[tag + "_color"] = image_report(_np(r.out_color), orec["out_color"], "color")
            out[tag + "_depth"] = image_report(_np(r.depth), orec["depth"], "depth")
            out[tag + "_opacity"] = image_report(_np(r.opacity), orec["opacity"], "opacity")


def c2_cases(out, s1m, n_fwd_tiles, n_bwd_tiles):
    from paper_2507_18713_b200 import configs, render_raster as RR
    from paper_2507_18713_b200.device import DeviceScene
    cam = configs.c2_camera()
    h, w = cam.height, cam.width
    ds = DeviceScene.from_scene(s1m)
    vox = oracle_voxels(s1m)
    ocam = ocam_of(cam)
    t0 = time.time()
    proj = O.project_voxels(vox, ocam)
    rng = np.random.default_rng(11)
    tiles = rng.choice(120 * 68, n_fwd_tiles, replace=False)
    ref = O.rasterize(vox, ocam, tiles=tiles, proj=proj)
    out["c2_oracle_fwd_s"] = time.time() - t0
    sel = np.zeros((h, w), bool)
    for t in tiles:
        ty, tx = divmod(int(t), 120)
        sel[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    for exact in (False, True):
        fb = RR.rasterize(ds, cam, exact_color=exact)
        tag = "c2_fp64" if exact else "c2_mixed"
        out[tag + "_color"] = image_report(_np(fb.color)[sel], ref["color"][sel], "color")
        out[tag + "_opacity"] = image_report(_np(fb.opacity)[sel], ref["opacity"][sel], "opacity")
        out[tag + "_depth"] = image_report(_np(fb.depth)[sel], ref["depth"][sel], "depth")
    # backward: L1 seeds (random target) on n_bwd_tiles tiles
    btiles = tiles[:n_bwd_tiles]
    bsel = np.zeros((h, w), bool)
    for t in btiles:
        ty, tx = divmod(int(t), 120)
        bsel[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    gt = rng.uniform(0, 1, (h, w, 3))
    dc = np.where(bsel[..., None], np.sign(ref["color"] - gt) / (3 * bsel.sum()), 0.0)
    t0 = time.time()
    rec = O.raster_records(vox, ocam, tiles=btiles, proj=proj)
    want = O.backward_records(rec, vox, dc.reshape(-1, 3), np.zeros(h * w))
    mag = grad_magnitude(O, rec, vox, dc.reshape(-1, 3), np.zeros(h * w))
    out["c2_oracle_bwd_s"] = time.time() - t0
    for exact in (False, True):
        fb, st = RR.rasterize(ds, cam, return_state=True, exact_color=exact)
        g = RR.rasterize_backward(st, dc, None)
        tag = "c2_fp64" if exact else "c2_mixed"
        out[tag + "_grad"] = grad_report(g, want, mag)
        out[tag + "_grad_nomag"] = grad_report(g, want)


def c3_cases(out, s1m, n_rays):
    from paper_2507_18713_b200 import configs, render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene, grads_to_dict
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    ds = DeviceScene.from_scene(s1m)
    oc = RY.build_scene_octrees(s1m)
    lb = gen_lidar_rays(configs.c3_lidar())
    ret = RY.render_lidar(ds, oc, lb)
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(lb.n, n_rays, replace=False))
    o, d = lb.origins[idx].cpu().numpy(), lb.dirs[idx].cpu().numpy()
    vox = oracle_voxels(s1m)
    t0 = time.time()
    tree = O.build_octree(vox)
    out["c3_oracle_octree_s"] = time.time() - t0
    t0 = time.time()
    orec = O.integrate_rays(vox, tree, o, d)
    out["c3_oracle_integrate_s"] = time.time() - t0
    out["c3_mixed_depth"] = image_report(_np(ret.depth).reshape(-1)[idx], orec["depth"], "depth")
    out["c3_mixed_opacity"] = image_report(_np(ret.opacity).reshape(-1)[idx], orec["opacity"], "opacity")
    gtr = rng.uniform(1, 30, n_rays)
    ok = np.isfinite(orec["depth"])
    dd_s = np.where(ok, np.sign(np.nan_to_num(orec["depth"]) - gtr) / max(ok.sum(), 1), 0.0)
    want = O.backward_records(orec, vox, np.zeros((n_rays, 3)), dd_s)
    mag = grad_magnitude(O, orec, vox, np.zeros((n_rays, 3)), dd_s)
    dd = np.zeros(lb.n)
    dd[idx] = dd_s
    g, _, _ = RY.lidar_backward(ret, torch.as_tensor(dd, device="cuda"))
    out["c3_mixed_grad"] = grad_report(grads_to_dict(g), want, mag)
    out["c3_mixed_grad_nomag"] = grad_report(grads_to_dict(g), want)


def c4_cases(out, n_rays):
    from paper_2507_18713_b200 import configs, render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import camera_rays
    sc = get_scene("S2M", "init")
    cam = configs.c4_camera()
    b = camera_rays(cam)
    ds = DeviceScene.from_scene(sc)
    oc = RY.build_scene_octrees(sc)
    col, op, dep = RY.render_rays_image(ds, oc, b)
    valid = np.flatnonzero(b.valid.cpu().numpy().reshape(-1))
    idx = np.sort(np.random.default_rng(3).choice(valid, n_rays, replace=False))
    o, d = b.origins.reshape(-1, 3)[idx].cpu().numpy(), b.dirs.reshape(-1, 3)[idx].cpu().numpy()
    vox = oracle_voxels(sc)
    t0 = time.time()
    ref = O.integrate_rays(vox, O.build_octree(vox), o, d)
    out["c4_oracle_s"] = time.time() - t0
    out["c4_mixed_color"] = image_report(_np(col).reshape(-1, 3)[idx], ref["out_color"], "color")
    out["c4_mixed_opacity"] = image_report(_np(op).reshape(-1)[idx], ref["opacity"], "opacity")
    out["c4_mixed_depth"] = image_report(_np(dep).reshape(-1)[idx], ref["depth"], "depth")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/parity_report.json")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="golden,c2,c3,c4")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    out = {}
    only = a.only.split(",")
    if "golden" in only:
        golden_cases(out)
    if {"c2", "c3"} & set(only):
        from paper_2507_18713_b200.scenes import get_scene
        s1m = get_scene("S1M", "init")
        if "c2" in only:
            c2_cases(out, s1m, 8 if a.quick else 32, 2 if a.quick else 8)
        if "c3" in only:
            c3_cases(out, s1m, 512 if a.quick else 4096)
    if "c4" in only:
        c4_cases(out, 512 if a.quick else 4096)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(out, indent=1))
    for k, v in out.items():
        if isinstance(v, dict) and "ok" in v:
            print(f"{k:40s} ok={v['ok']} viol={v['violations']}/{v['n']} worst_rel={v['worst_rel_above_floor']:.2e}")
        elif isinstance(v, dict):
            for kk, r in v.items():
                print(f"{k + '.' + kk:40s} ok={r['ok']} viol={r['violations']}/{r['n']} "
                      f"worst_rel={r['worst_rel_above_floor']:.2e} under_floor={r['n_under_floor']}")
        else:
            print(k, v)


if __name__ == "__main__":
    main()
