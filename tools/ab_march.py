"""A/B timing of the marcher descent variants (SALF_MARCH_VARIANT) on C3."""
import os, sys, json, subprocess
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
code = r'''
import sys, json; sys.path.insert(0, "%s")
import torch, numpy as np
from paper_2507_18713_b200 import configs, render_ray as RY
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import gen_lidar_rays
out = {}
for regime in sys.argv[1:]:
    sc = get_scene("S1M", regime); ds = DeviceScene.from_scene(sc); oc = RY.build_scene_octrees(sc)
    lb = gen_lidar_rays(configs.c3_lidar())
    f = lambda: RY.integrate_rays(ds, oc, lb.origins, lb.dirs)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    out[regime] = a.elapsed_time(b) / 20
print(json.dumps(out))
''' % ROOT
for v in sys.argv[1].split(","):
    env = dict(os.environ, SALF_MARCH_VARIANT=v)
    r = subprocess.run([sys.executable, "-c", code] + sys.argv[2:], env=env, capture_output=True, text=True)
    print("variant", v, r.stdout.strip(), r.stderr.strip()[-300:])
