"""Kernel-time breakdown of one C5 rig training step on one GPU (torch.profiler)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2507_18713_b200 import configs, render_ray as RY
from paper_2507_18713_b200.optim import TrainableScene
from paper_2507_18713_b200.parallel import split_work
from paper_2507_18713_b200.scenes import get_scene
from paper_2507_18713_b200.train_step import rig_step

scene = get_scene("S1M", "init")
oc = RY.build_scene_octrees(scene)
ts = TrainableScene(scene)
cams, lidars = configs.c5_rig()
sensors = cams + lidars
g = torch.Generator().manual_seed(5)
targets = [torch.rand((c.height, c.width, 3), generator=g, dtype=torch.float64).to(ts.ds.device) for c in cams] + \
    [(1.0 + 20.0 * torch.rand(l.beam_elevations.shape[0] * l.steps, generator=g, dtype=torch.float64)).to(ts.ds.device)
     for l in lidars]
items = split_work(sensors, 1)
gbuf = ts.zero_grad()


def step():
    gbuf.zero_()
    rig_step(ts.ds, oc, sensors, targets, items, gbuf)
    ts.adam_step(gbuf)


for _ in range(2):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
step()
b.record()
torch.cuda.synchronize()
print("step ms", a.elapsed_time(b))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
