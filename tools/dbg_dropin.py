"""Debug: one trainer-shaped batch through the reference and the drop-in backend."""
import copy, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT / "baseline/_ref"), str(ROOT / "tests"), str(ROOT)]
import salf, salf.container
from salf.sensors import CameraModel, LidarModel, camera_rays, gen_camera_rays, gen_lidar_rays
from salf.synthetic import look_at_quaternion
from salf.render_ray import build_scene_octrees, integrate_rays
from salf.backward import backward_records
from salf.losses import loss_color, loss_depth
scene = salf.container.load_scene(ROOT / "tests/golden/scenes/rand300")
pos = np.array([13.0137, 11.0213, 7.0])
cam = CameraModel(kind="pinhole", width=64, height=48, fx=60.0, fy=60.0, cx=32.0, cy=24.0, position=pos,
                  quaternion=look_at_quaternion(pos, [4.0, 4.0, 2.0]))
lid = LidarModel(beam_elevations=np.radians(np.linspace(-25, 15, 16)), steps=90, position=np.array([4.0137, 3.9787, 3.3]))
cb, lb = gen_camera_rays(cam), gen_lidar_rays(lid)
rng = np.random.default_rng(0)
ci, li = rng.integers(0, cb.n, 512), rng.integers(0, lb.n, 128)
o = np.concatenate([cb.origins[ci], lb.origins[li]]); d = np.concatenate([cb.dirs[ci], lb.dirs[li]])
mask = np.zeros(o.shape[0], bool); mask[:512] = True
gt_c = rng.uniform(0, 1, (512, 3)); gt_d = rng.uniform(1, 10, 128)
def run():
    oc = salf.render_ray.build_scene_octrees(scene)
    rec = salf.render_ray.integrate_rays(scene, oc, o, d)
    lc, dc = loss_color(rec, gt_c, mask)
    ld, dd = loss_depth(rec, gt_d, ~mask)
    g = salf.backward.backward_records(rec, scene, dc, 10 * dd)
    return rec, lc, ld, g
r_ref = run()
from paper_2507_18713_b200 import dropin
be = dropin.install(salf)
r_gpu = run()
print("losses", r_ref[1], r_gpu[1], r_ref[2], r_gpu[2])
for f in ("out_color", "depth", "opacity", "weight_sum", "t_final"):
    a, b = getattr(r_gpu[0], f), getattr(r_ref[0], f)
    m = np.isfinite(b)
    print(f, "nan-mismatch", int((np.isnan(a) != np.isnan(b)).sum()), "max abs", np.abs(a[m] - b[m]).max())
print("segments", r_gpu[0].n_segments, r_ref[0].n_segments)
for k in ("w_s", "w_c", "w_sh", "log_a", "log_b"):
    a, b = r_gpu[3]["static"][k], r_ref[3]["static"][k]
    print(k, "max abs", np.abs(a - b).max(), "max |ref|", np.abs(b).max())
# reference backward on OUR records (isolates forward vs backward)
be.uninstall()
g2 = salf.backward.backward_records(r_gpu[0], scene, *[x for x in (None, None)] ) if False else None

# --- trainer step-by-step
from salf.trainer import RayDataset, TrainConfig, train_loop
from salf.render_ray import render_lidar_ranges, render_rays_image
target = copy.deepcopy(scene); target.static.w_c = target.static.w_c * 0.8; target.static.log_a = target.static.log_a + 0.3
octs = build_scene_octrees(target)
img, _, _ = render_rays_image(target, octs, camera_rays(cam))
rng_l = render_lidar_ranges(target, octs, gen_lidar_rays(lid))
hit = np.isfinite(rng_l.ravel())
ds = RayDataset(cam_origins=cb.origins, cam_dirs=cb.dirs, cam_colors=img.reshape(-1, 3), lidar_origins=lb.origins,
                lidar_dirs=lb.dirs, lidar_ranges=rng_l.ravel(), points=lb.origins[hit] + rng_l.ravel()[hit, None] * lb.dirs[hit])
cfg = TrainConfig(steps=20, batch_rays=512, batch_lidar=128, seed=3, log_every=1)
captured = {"ref": [], "gpu": []}
import salf.trainer as T
orig_bw = T.backward_records
def cap(tag):
    def f(rec, sc, dc, dd):
        g = T._cur_bw(rec, sc, dc, dd)
        d = {k: v.copy() for k, v in g["static"].items()}
        d["_dc"], d["_dd"] = np.array(dc), np.array(dd)
        d["_oc"], d["_dep"], d["_ws"] = rec.out_color.copy(), rec.depth.copy(), rec.weight_sum.copy()
        captured[tag].append(d)
        return g
    return f
s_ref, s_gpu = copy.deepcopy(scene), copy.deepcopy(scene)
T._cur_bw = orig_bw; T.backward_records = cap("ref")
m_ref = train_loop(s_ref, ds, cfg)
T.backward_records = orig_bw
be = dropin.install(salf)
T._cur_bw = T.backward_records; T.backward_records = cap("gpu")
m_gpu = train_loop(s_gpu, ds, cfg)
for a, b in zip(m_gpu, m_ref):
    print(a["step"], a["loss_total"], b["loss_total"], a["loss_color"] - b["loss_color"], a["loss_depth"] - b["loss_depth"])
a, b = captured["gpu"][0], captured["ref"][0]
for k in ("_dc", "_dd", "_oc", "_dep", "_ws"):
    x, y = a[k], b[k]
    print(k, x.shape, "nan mism", int((np.isnan(x) != np.isnan(y)).sum()), "max", np.nanmax(np.abs(x - y)))
bad = np.flatnonzero((a["w_s"] == 0).any(1) != (b["w_s"] == 0).any(1))
print("voxels with zero-pattern mismatch", bad[:10], a["w_s"][bad[:3]], b["w_s"][bad[:3]])
for i, (a, b) in enumerate(zip(captured["gpu"], captured["ref"])):
    for k in ("w_s", "log_a"):
        za, zb = a[k] == 0, b[k] == 0
        print(i, k, "zero-pattern mismatch", int((za != zb).sum()), "max abs", np.abs(a[k] - b[k]).max())
