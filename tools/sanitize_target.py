"""Small workload for compute-sanitizer: raster fwd+bwd (default, deterministic,
fp64 modes), ray fwd+bwd, LiDAR, densify, effects on the golden scenes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import torch
from conftest import load_golden_scene
from paper_2507_18713_b200 import render_raster as RR, render_ray as RY
from paper_2507_18713_b200.backward import backward_grad_buffer
from paper_2507_18713_b200.densify import DensifyConfig, densify_and_prune
from paper_2507_18713_b200.scene import flatten_scene
from paper_2507_18713_b200.sensors import CameraModel, look_at_quaternion

sc = load_golden_scene("rand300")
pos = np.array([13.0, 11.0, 7.0])
cam = CameraModel(kind="pinhole", width=48, height=40, fx=45.0, fy=45.0, cx=24.0, cy=20.0, position=pos,
                  quaternion=look_at_quaternion(pos, [4.0, 4.0, 2.0]))
flat = flatten_scene(sc)
dc = torch.full((40, 48, 3), 1e-3, device="cuda", dtype=torch.float64)
dd = torch.full((40, 48), 1e-4, device="cuda", dtype=torch.float64)
for exact in (False, True):
    fb, st = RR.rasterize(flat, cam, return_state=True, exact_color=exact)
    RR.rasterize_backward(st, dc, dd)
    RR.rasterize_backward(st, dc, dd, deterministic=True)
oc = RY.build_scene_octrees(sc)
rng = np.random.default_rng(3)
o = rng.uniform(-1, 9, (300, 3))
d = rng.normal(size=(300, 3))
d /= np.linalg.norm(d, axis=1, keepdims=True)
rec = RY.integrate_rays(sc, oc, o, d)
backward_grad_buffer(rec, np.full((300, 3), 1e-3), np.full(300, 1e-3))
backward_grad_buffer(rec, np.full((300, 3), 1e-3), np.full(300, 1e-3), deterministic=True)
densify_and_prune(sc.static, rng.random(sc.static.n), DensifyConfig(budget=sc.static.n + 400))
RY.trace_effects(sc, oc, o, d, 0.0, [RY.InjectedSphere([4, 4, 3], 1.0, "glass")], [0, 0, 1])
torch.cuda.synchronize()
print("sanitize target ok")
# descent jump tables of every depth (query + march)
from paper_2507_18713_b200.octree import march_segments, query_batch
pts = rng.uniform(-1, 9, (500, 3)).clip(oc.static.root_min, oc.static.root_min + oc.static.root_edge)
for k in range(0, 9):
    t = oc.static.with_jump(k)
    query_batch(t, pts)
    march_segments(t, o, d)
torch.cuda.synchronize()
print("jump tables ok")
# round 2: hand-written sort (multi-CTA, device count), capacity re-bin, hit-word backward on a
# bigger frame, device actor rays + merge, inference ray / LiDAR paths
from paper_2507_18713_b200 import _lib
lib = _lib.load()
for kb, end in ((4, 13), (8, 64)):
    n = 50_000
    keys = torch.randint(0, 1 << 13, (n,), device="cuda", dtype=torch.int32 if kb == 4 else torch.int64)
    vals = torch.arange(n, device="cuda", dtype=torch.int32)
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    nd = torch.tensor([n - 123], device="cuda", dtype=torch.int64)
    wsb = lib.salf_sort_pairs_workspace_bytes(n, kb, 0, end)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.salf_sort_pairs(keys.data_ptr(), vals.data_ptr(), ko.data_ptr(), vo.data_ptr(), kb, nd.data_ptr(),
                                   n, 0, end, ws.data_ptr(), wsb, _lib.stream_ptr()), "sort")
# splitter bucket sort (the depth rank): device count, all-equal keys (one key, split on the value)
for const in (False, True):
    n = 60_000
    keys = (torch.zeros(n, device="cuda", dtype=torch.int64) + 7 if const
            else torch.randint(0, 1 << 40, (n,), device="cuda", dtype=torch.int64))
    vals = torch.arange(n, device="cuda", dtype=torch.int32)
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    nd = torch.tensor([n - 999], device="cuda", dtype=torch.int64)
    wsb = lib.salf_sort_pairs_unique_workspace_bytes()
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.salf_sort_pairs_unique(keys.data_ptr(), vals.data_ptr(), ko.data_ptr(), vo.data_ptr(),
                                          nd.data_ptr(), n, ws.data_ptr(), wsb, _lib.stream_ptr()), "sort_unique")
# non-16 tile (one CTA per tile, partial warps rounded up) forward + backward
fb13, st13 = RR.rasterize(flat, cam, tile=13, return_state=True)
RR.rasterize_backward(st13, dc, dd)
big = CameraModel(kind="pinhole", width=320, height=256, fx=300.0, fy=300.0, cx=160.0, cy=128.0, position=pos,
                  quaternion=look_at_quaternion(pos, [4.0, 4.0, 2.0]))
RR._CAPACITY[("cuda:0", 1)] = 5  # forces the re-bin path
fb, st = RR.rasterize(flat, big, return_state=True)
RR.rasterize_backward(st, torch.full((256, 320, 3), 1e-3, device="cuda", dtype=torch.float64), None)
act = load_golden_scene("actors")
oca = RY.build_scene_octrees(act)
rec = RY.integrate_rays(act, oca, o, d, np.linspace(0.0, 0.5, 300))
RR.rasterize_scene(act, cam, 0.25)
RY.integrate_rays(sc, oc, o, d, need_state=False)
from paper_2507_18713_b200.sensors import LidarModel, gen_lidar_rays
lb = gen_lidar_rays(LidarModel(beam_elevations=np.linspace(-0.4, 0.2, 8), steps=64, position=np.array([4.013, 3.987, 2.5])))
RY.render_lidar(sc, oc, lb, need_state=False)
ret = RY.render_lidar(sc, oc, lb)
RY.lidar_backward(ret, torch.full((lb.n,), 1e-3, device="cuda", dtype=torch.float64))
torch.cuda.synchronize()
print("round-2 paths ok")
