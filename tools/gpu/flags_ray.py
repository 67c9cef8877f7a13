import sys, torch
sys.path.insert(0, '.')
from paper_2507_18713_b200 import configs, render_ray as RY
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.sensors import gen_lidar_rays, camera_rays
for regime in ("init", "surface-dense"):
    sc = get_scene("S1M", regime); ds = DeviceScene.from_scene(sc); oc = RY.build_scene_octrees(sc)
    lb = gen_lidar_rays(configs.c3_lidar())
    r = RY.render_lidar(ds, oc, lb)
    cb = camera_rays(configs.c4_camera())
    r2 = RY.integrate_rays(ds, oc, cb.origins, cb.dirs, valid=cb.valid)
    print(regime, "lidar flagged", int(((r.status & 8) != 0).sum()), "of", lb.n, "| c4 flagged", int(((r2.status & 8) != 0).sum()), "of", cb.n)
