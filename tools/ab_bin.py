"""A/B timing of the C2 frame binning alone (S1M, 1080p: projection + cull +
depth rank + tile expansion + tile sort) for the library named by $SALF_LIB,
plus a checksum of the CSR so variants can be compared for identity.

usage: SALF_LIB=... python tools/ab_bin.py [init|surface] [tag]"""
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
near, tile = RR.NEAR_PLANE, RR.TILE_SIZE
out = {"tag": tag, "regime": regime}
for mode in (0, 1):
    proj = RR._project(ds, cam, near, tile)
    off, ent, n, _ = RR._bin_sync(ds, cam, near, tile, proj, mode)
    out[f"mode{mode}_instances"] = int(n)
    out[f"mode{mode}_csr_hash"] = int((ent.long() * torch.arange(1, n + 1, device=ent.device) % 1000003).sum()
                                      + off.sum())
    ts = []
    for i in range(23):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        RR._bin(ds, cam, near, tile, proj, mode)
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    out[f"mode{mode}_bin_ms"] = float(np.median(ts))
    # device time alone: a spin kernel ahead of the start event keeps the host enqueue off the clock
    ts = []
    for i in range(23):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record()
        RR._bin(ds, cam, near, tile, proj, mode)
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    out[f"mode{mode}_bin_device_ms"] = float(np.median(ts))
    ts = []
    for i in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p = RR._project(ds, cam, near, tile)
        RR._bin(ds, cam, near, tile, p, mode)
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    out[f"mode{mode}_project_bin_ms"] = float(np.median(ts))
print(json.dumps(out))
