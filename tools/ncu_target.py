"""Short workload for ncu captures: C2 raster fwd+bwd and C3 LiDAR fwd+bwd on S1M (init)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2507_18713_b200 import configs, render_raster as RR, render_ray as RY
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import gen_lidar_rays

regime = sys.argv[1] if len(sys.argv) > 1 else "init"
sc = get_scene("S1M", regime)
ds = DeviceScene.from_scene(sc)
cam = configs.c2_camera()
dc = torch.full((1080, 1920, 3), 1e-6, device="cuda", dtype=torch.float64)
dd = None  # colour-only loss, as bench.py
oc = RY.build_scene_octrees(sc)
lb = gen_lidar_rays(configs.c3_lidar())
for _ in range(3):
    fb, st = RR.rasterize(ds, cam, return_state=True)
    RR.rasterize_backward(st, dc, dd, as_dict=False)
    ret = RY.render_lidar(ds, oc, lb)
    RY.lidar_backward(ret, torch.sign(torch.nan_to_num(ret.depth.double()) - 10.0) / 1e5)
torch.cuda.synchronize()
print("ok")
