import sys, torch
sys.path.insert(0,'.')
from paper_2507_18713_b200 import configs, render_ray as RY
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import gen_lidar_rays
sc=get_scene("S1M","init"); ds=DeviceScene.from_scene(sc); oc=RY.build_scene_octrees(sc); lb=gen_lidar_rays(configs.c3_lidar())
for _ in range(3): r=RY.render_lidar(ds, oc, lb)
torch.cuda.synchronize()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): r=RY.render_lidar(ds, oc, lb)
b.record(); torch.cuda.synchronize()
print(sys.argv[1], a.elapsed_time(b)/20, float(r.saved[:,6].sum()))
