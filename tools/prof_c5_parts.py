import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
"""Per-phase device time of the C5 rig step on one GPU: each camera's raster
forward / backward, each LiDAR's forward / backward, Adam, and the whole
rig_step (tools/gpu, diagnostic only)."""
import json

import torch

from paper_2507_18713_b200 import configs
from paper_2507_18713_b200 import render_raster as RR
from paper_2507_18713_b200 import render_ray as RY
from paper_2507_18713_b200.backward import backward_grad_buffer
from paper_2507_18713_b200.optim import TrainableScene
from paper_2507_18713_b200.parallel import split_work
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import gen_lidar_rays
from paper_2507_18713_b200.train_step import rig_step


def timeit(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


scene = get_scene("S1M", "init")
ts = TrainableScene(scene)
ds = ts.ds
oc = RY.build_scene_octrees(scene)
cams, lidars = configs.c5_rig()
grad = ts.zero_grad()
out = {"cams": []}
for c in cams:
    fb, st = RR.rasterize(ds, c, return_state=True)
    dc = torch.sign(torch.randn(c.height, c.width, 3, dtype=torch.float64, device=ds.device)) / 1e6
    dd = torch.zeros((c.height, c.width), dtype=torch.float64, device=ds.device)
    f = timeit(lambda: RR.rasterize(ds, c, return_state=True))
    b = timeit(lambda: RR.rasterize_backward(st, dc, None, grad, as_dict=False))  # colour-only, as rig_step
    out["cams"].append({"fwd_ms": f, "bwd_ms": b, "instances": int(st.n_instances) if hasattr(st, "n_instances") else None})
out["lidars"] = []
for l in lidars:
    rays = gen_lidar_rays(l, device=ds.device)
    rec = RY.integrate_rays(ds, oc, rays.origins, rays.dirs, check_unit=False)
    dd = torch.sign(torch.randn(rays.origins.shape[0], dtype=torch.float64, device=ds.device)) / 1e5
    dcz = torch.zeros((rays.origins.shape[0], 3), dtype=torch.float64, device=ds.device)
    f = timeit(lambda: RY.integrate_rays(ds, oc, rays.origins, rays.dirs, check_unit=False))
    b = timeit(lambda: backward_grad_buffer(rec, dcz, dd, grad))
    out["lidars"].append({"fwd_ms": f, "bwd_ms": b})
out["adam_ms"] = timeit(lambda: ts.adam_step(grad))
sensors = cams + lidars
g = torch.Generator().manual_seed(5)
targets = [torch.rand((c.height, c.width, 3), generator=g, dtype=torch.float64).to(ds.device) for c in cams] + [
    (1.0 + 20.0 * torch.rand(l.beam_elevations.shape[0] * l.steps, generator=g, dtype=torch.float64)).to(ds.device)
    for l in lidars]
items = split_work(sensors, 1)
out["items"] = [(it.kind, it.sensor, it.lo, it.hi) for it in items]


def step():
    grad.zero_()
    rig_step(ts.ds, oc, sensors, targets, items, grad)
    ts.adam_step(grad)


out["step_ms"] = timeit(step, n=3)
out["sum_parts_ms"] = sum(c["fwd_ms"] + c["bwd_ms"] for c in out["cams"]) + sum(
    l["fwd_ms"] + l["bwd_ms"] for l in out["lidars"]) + out["adam_ms"]
print(json.dumps(out))
