"""Quick timing probe of every hot kernel (development aid, not the bench)."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2507_18713_b200 import render_raster as RR, render_ray as RY, configs, sensors as S
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scene import flatten_scene

def timeit(fn, n=5):
    fn(); torch.cuda.synchronize()
    ts=[]
    for _ in range(n):
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))

res={}
for regime in sys.argv[1:] or ["surface","init"]:
    t=time.time(); sc=get_scene("S1M", regime); res[f"load_{regime}_s"]=time.time()-t
    res[f"S1M_{regime}_voxels"]=sc.static.n
    ds=DeviceScene.from_scene(sc)
    cam=configs.c2_camera()
    fb=RR.rasterize(ds, cam); torch.cuda.synchronize()
    res[f"c2_fwd_ms_{regime}"]=timeit(lambda: RR.rasterize(ds, cam))
    p=RR._project(ds, cam, 0.05, 16)
    _,_,ninst,_=RR._bin_sync(ds, cam, 0.05, 16, p, 1)
    res[f"c2_instances_fit_{regime}"]=ninst
    fb,st=RR.rasterize(ds, cam, return_state=True)
    dc=torch.full((1080,1920,3),1e-6,device='cuda',dtype=torch.float64); dd=torch.zeros((1080,1920),device='cuda',dtype=torch.float64)
    res[f"c2_bwd_ms_{regime}"]=timeit(lambda: RR.rasterize_backward(st, dc, dd, as_dict=False), n=3)
    t=time.time(); oc=RY.build_scene_octrees(sc); res[f"octree_build_s_{regime}"]=time.time()-t
    from paper_2507_18713_b200.octree import build_octree_device
    build_octree_device(sc.static); torch.cuda.synchronize()
    t=time.time(); build_octree_device(sc.static); torch.cuda.synchronize(); res[f"octree_build_device_s_{regime}"]=time.time()-t
    lb=S.gen_lidar_rays(configs.c3_lidar())
    res[f"c3_ms_{regime}"]=timeit(lambda: RY.integrate_rays(ds, oc, lb.origins, lb.dirs))
    rec=RY.integrate_rays(ds, oc, lb.origins, lb.dirs)
    res[f"c3_segments_{regime}"]=float(rec.n_segments.sum().item())
    res[f"c3_status_{regime}"]=int(rec.status.max().item())
    print(json.dumps(res), flush=True)
print(json.dumps(res))
