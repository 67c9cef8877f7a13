"""Per-pixel breakdown of the worst C2 gradient elements (mixed backward vs the oracle).

  python tools/diag_grad.py [--n 3]

For the worst violating voxels of the parity report's C2 case it reseeds the
loss one pixel at a time and prints each pixel's GPU vs oracle contribution,
plus the pixel's saved state (stop index, T_final) and the oracle's hits."""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import oracle_voxels  # noqa: E402
from oracle import salf_oracle as O  # noqa: E402
from parity import grad_magnitude, grad_report  # noqa: E402

KEYS = ("w_s", "w_c", "w_sh", "log_a", "log_b")
OFF = {"w_s": 0, "w_c": 4, "w_sh": 13, "log_a": 25, "log_b": 26}
SIZE = {"w_s": 4, "w_c": 9, "w_sh": 12, "log_a": 1, "log_b": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3)
    a = ap.parse_args()
    from paper_2507_18713_b200 import configs, render_raster as RR
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from parity_report import ocam_of
    s1m = get_scene("S1M", "init")
    cam = configs.c2_camera()
    h, w = cam.height, cam.width
    ds = DeviceScene.from_scene(s1m)
    vox = oracle_voxels(s1m)
    ocam = ocam_of(cam)
    proj = O.project_voxels(vox, ocam)
    rng = np.random.default_rng(11)
    tiles = rng.choice(120 * 68, 32, replace=False)
    btiles = tiles[:8]
    ref = O.rasterize(vox, ocam, tiles=btiles, proj=proj)
    bsel = np.zeros((h, w), bool)
    for t in btiles:
        ty, tx = divmod(int(t), 120)
        bsel[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    gt = rng.uniform(0, 1, (h, w, 3))
    dc = np.where(bsel[..., None], np.sign(ref["color"] - gt) / (3 * bsel.sum()), 0.0)
    rec = O.raster_records(vox, ocam, tiles=btiles, proj=proj)
    want = O.backward_records(rec, vox, dc.reshape(-1, 3), np.zeros(h * w))
    mag = grad_magnitude(O, rec, vox, dc.reshape(-1, 3), np.zeros(h * w))
    fb, st = RR.rasterize(ds, cam, return_state=True)
    g = RR.rasterize_backward(st, dc, None)
    rep = grad_report(g, want, mag)
    saved = st.saved.cpu().numpy()
    for k in KEYS:
        r = rep[k]
        print(k, r["violations"], r["worst"])
        if r["violations"] == 0:
            continue
        x = np.asarray(g[k], np.float64).reshape(-1)
        y = np.asarray(want[k], np.float64).reshape(-1)
        mm = np.asarray(mag[k], np.float64).reshape(-1)
        bad = np.flatnonzero(np.abs(x - y) > 1e-4 * np.abs(y) + 1e-5 * mm)
        bad = bad[np.argsort(-np.abs(x - y)[bad] / np.abs(y[bad]))][: a.n]
        for idx in bad:
            v, comp = divmod(int(idx), SIZE[k])
            col = OFF[k] + comp
            segs = np.flatnonzero(rec["vid"] == v)
            pix = np.unique(rec["ray"][segs])
            print(f"  voxel {v} comp {k}[{comp}] got {x[idx]:.6e} want {y[idx]:.6e} mag {mm[idx]:.3e} "
                  f"pixels {pix.size} segments {segs.size}")
            for p in pix[:12]:
                dcp = np.zeros_like(dc).reshape(-1, 3)
                dcp[p] = dc.reshape(-1, 3)[p]
                gp = RR.rasterize_backward(st, dcp.reshape(h, w, 3), None, as_dict=False)[v, col].item()
                wp = O.backward_records(rec, vox, dcp, np.zeros(h * w))[k].reshape(-1)[idx]
                sv = saved[p]
                rs = segs[rec["ray"][segs] == p]
                inc = rec["included"][rs]
                print(f"    px {p}: gpu {gp:.6e} oracle {wp:.6e} rel {abs(gp - wp) / max(abs(wp), 1e-300):.2e} "
                      f"| n_stop {int(sv[6])} n_inc {int(sv[7])} T_fin {sv[5]:.4e} | oracle seg inc {inc.tolist()} "
                      f"alpha {rec['alpha'][rs].round(6).tolist()} c {rec['color'][rs].round(6).tolist()} "
                      f"tb {rec['t_before'][rs].round(6).tolist()} delta/edge {((rec['t1'][rs] - rec['t0'][rs]) / vox.edges[v]).tolist()} "
                      f"sigma {rec['sigma'][rs].tolist()} x {rec['x'][rs].tolist()} s {rec['s_field'][rs].tolist()}")


if __name__ == "__main__":
    main()
