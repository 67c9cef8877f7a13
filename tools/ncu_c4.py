"""Short workload for ncu: the C4 fisheye + rolling-shutter frame (S2M, ray path)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2507_18713_b200 import configs, render_ray as RY
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import camera_rays
sc = get_scene("S2M", "init")
ds = DeviceScene.from_scene(sc)
oc = RY.build_scene_octrees(sc)
cb = camera_rays(configs.c4_camera())
for _ in range(3):
    RY.integrate_rays(ds, oc, cb.origins, cb.dirs, valid=cb.valid)
torch.cuda.synchronize()
print("ok")
