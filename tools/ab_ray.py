"""A/B timing of the ray path for the library named by $SALF_LIB: C3 LiDAR
sweep (forward, and forward + depth backward) on S1M, C4 fisheye + rolling
shutter frame on S2M.  usage: SALF_LIB=... python tools/ab_ray.py [tag]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2507_18713_b200 import configs, render_ray as RY
from paper_2507_18713_b200.backward import backward_grad_buffer
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import camera_rays, gen_lidar_rays

tag = sys.argv[1] if len(sys.argv) > 1 else "lib"


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


sc = get_scene("S1M", "init")
ds = DeviceScene.from_scene(sc)
oc = RY.build_scene_octrees(sc)
lb = gen_lidar_rays(configs.c3_lidar())
out = {"tag": tag}
out["c3_lidar_ms"] = timeit(lambda: RY.render_lidar(ds, oc, lb, need_state=False))
out["c3_lidar_state_ms"] = timeit(lambda: RY.render_lidar(ds, oc, lb))
out["c3_fwd_ms"] = timeit(lambda: RY.integrate_rays(ds, oc, lb.origins, lb.dirs))
rec = RY.integrate_rays(ds, oc, lb.origins, lb.dirs)
dd = torch.sign(torch.randn(lb.n, device="cuda", dtype=torch.float64)) / lb.n
dc = torch.zeros((lb.n, 3), device="cuda", dtype=torch.float64)
grad = torch.zeros((ds.n, 27), device="cuda", dtype=torch.float64)
out["c3_bwd_ms"] = timeit(lambda: backward_grad_buffer(rec, dc, dd, grad))
out["c3_bwd_depth_only_ms"] = timeit(lambda: backward_grad_buffer(rec, None, dd, grad))
out["c3_digest"] = [float(rec.saved[:, 6].sum()), float(torch.nan_to_num(rec.depth.double()).sum())]
del ds, oc
s2 = get_scene("S2M", "init")
ds2 = DeviceScene.from_scene(s2)
oc2 = RY.build_scene_octrees(s2)
cb = camera_rays(configs.c4_camera())
out["c4_ms"] = timeit(lambda: RY.integrate_rays(ds2, oc2, cb.origins, cb.dirs, valid=cb.valid, need_state=False), n=5)
r2 = RY.integrate_rays(ds2, oc2, cb.origins, cb.dirs, valid=cb.valid)
out["c4_digest"] = [float(r2.saved[:, 6].sum()), float(torch.nan_to_num(r2.depth.double()).sum())]
print(json.dumps(out))
