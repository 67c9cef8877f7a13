"""Counts of the backward's chord refinement at C2 (diagnostics build:
tools/ab_build.sh diag -DSALF_DIAG_CHORD; SALF_LIB=build_ab/diag/libsalf_b200.so)."""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2507_18713_b200 import _lib, configs, render_raster as RR
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene

torch.cuda.set_device(0)
ds = DeviceScene.from_scene(get_scene("S1M", "init"))
cam = configs.c2_camera()
lib = _lib.load()
fn = ctypes.CDLL(str(_lib.LIB_PATH)).salf_debug_counters
cnt = (ctypes.c_ulonglong * 4)()
fb, st = RR.rasterize(ds, cam, return_state=True)
dc = torch.full((1080, 1920, 3), 1e-6, device="cuda", dtype=torch.float64)
fn(cnt, 1)
RR.rasterize_backward(st, dc, None, as_dict=False)
torch.cuda.synchronize()
fn(cnt, 0)
print({"fp32_hits": cnt[0], "under_cheap_bound": cnt[1], "refined_fp64": cnt[2]})
