"""A/B timing of the C2 raster forward / backward (S1M, 1080p) for the library
named by $SALF_LIB (default: the in-tree build), plus the fast-mode gradient
against the fp64 exact-mode gradient on the same frame (normwise per class).

usage: SALF_LIB=... python tools/ab_raster.py [init|surface] [tag]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2507_18713_b200 import configs, render_raster as RR
from paper_2507_18713_b200.device import DeviceScene
from paper_2507_18713_b200.scenes import get_scene

regime = sys.argv[1] if len(sys.argv) > 1 else "init"
tag = sys.argv[2] if len(sys.argv) > 2 else "lib"
torch.cuda.set_device(0)
ds = DeviceScene.from_scene(get_scene("S1M", regime))
cam = configs.c2_camera()
g = torch.Generator(device="cuda").manual_seed(0)
h, w = cam.height, cam.width
dc = (torch.randint(0, 2, (h, w, 3), device="cuda", generator=g).double() * 2 - 1) / (h * w * 3)
dd = (torch.randint(0, 2, (h, w), device="cuda", generator=g).double() * 2 - 1) / (h * w)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = {"tag": tag, "regime": regime}
for exact in (False, True):
    fb, st = RR.rasterize(ds, cam, return_state=True, exact_color=exact)
    grad = torch.zeros((ds.n, 27), dtype=torch.float64, device="cuda")
    key = "exact" if exact else "fast"
    out[f"{key}_fwd_ms"] = timeit(lambda: RR.rasterize(ds, cam, return_state=True, exact_color=exact))
    out[f"{key}_bwd_ms"] = timeit(lambda: RR.rasterize_backward(st, dc, dd, grad=grad.zero_(), as_dict=False))
    out[f"{key}_bwd_colour_only_ms"] = timeit(lambda: RR.rasterize_backward(st, dc, None, grad=grad.zero_(),
                                                                            as_dict=False))
    out[f"{key}_bwd_det_ms"] = timeit(lambda: RR.rasterize_backward(st, dc, dd, grad=grad.zero_(), as_dict=False,
                                                                    deterministic=True), n=5)
    grad.zero_()
    RR.rasterize_backward(st, dc, dd, grad=grad, as_dict=False)
    out[f"{key}_grad"] = grad.clone()
    out[f"{key}_rgb"] = fb.color.clone()
# forward decisions: fast (certified + fp64 redo) vs exact, per pixel
fa, sa = RR.rasterize(ds, cam, return_state=True, exact_color=False)
fe, se = RR.rasterize(ds, cam, return_state=True, exact_color=True)
na, ne = sa.saved[:, 6], se.saved[:, 6]
out["fwd_stop_index_mismatch"] = int((na != ne).sum())
out["fwd_depth_nan_mismatch"] = int((torch.isnan(fa.depth) != torch.isnan(fe.depth)).sum())
m = ~torch.isnan(fe.depth)
out["fwd_depth_max_rel"] = float(((fa.depth[m] - fe.depth[m]).abs() / fe.depth[m].abs()).max())
out["fwd_opacity_max_abs"] = float((fa.opacity - fe.opacity).abs().max())
out["fwd_color_max_abs_vs_exact"] = float((fa.color - fe.color).abs().max())
ga, gb = out.pop("fast_grad"), out.pop("exact_grad")
sl = {"w_s": slice(0, 4), "w_c": slice(4, 13), "w_sh": slice(13, 25), "log_a": slice(25, 26),
      "log_b": slice(26, 27)}
out["grad_normwise_err"] = {k: float((ga[:, s] - gb[:, s]).abs().max() / gb[:, s].abs().max().clamp_min(1e-30))
                            for k, s in sl.items()}
ra, rb = out.pop("fast_rgb"), out.pop("exact_rgb")
out["rgb_max_abs_err"] = float((ra - rb).abs().max())
import os
if os.environ.get("SALF_NO_REDO") == "1":
    out["flagged_pixels"] = int(torch.isnan(fa.opacity).sum())
print(json.dumps(out))
