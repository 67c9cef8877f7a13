"""Worker for tests/test_gpu_train_step.py::test_rig_step_two_processes_gloo: one
rank of a world-2 C5-shaped training step (gloo process group, both ranks on
cuda:0), sharded by parallel.assign(split_work(...)) and summed by the
all-reduces inside train_step.rig_step."""
import sys

import numpy as np
import torch
import torch.distributed as dist


def run(rank: int, world: int, port: int, out_path: str) -> None:
    sys.path[:0] = [str(__import__("pathlib").Path(__file__).resolve().parent.parent)]
    from conftest import load_golden_scene
    from test_gpu_train_step import _rig, _targets
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.parallel import assign, split_work
    from paper_2507_18713_b200.train_step import rig_step
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sc = load_golden_scene("rand300")
    ds = DeviceScene.from_scene(sc)
    oc = RY.build_scene_octrees(sc)
    sensors = _rig()
    targets = _targets(sensors)
    items = assign(split_work(sensors, world), world)[rank]
    grad = torch.zeros((ds.n, 27), dtype=torch.float64, device="cuda")
    losses, counts = rig_step(ds, oc, sensors, targets, items, grad)
    if rank == 0:
        np.savez(out_path, grad=grad.cpu().numpy(), losses=losses.cpu().numpy(), counts=counts.cpu().numpy(),
                 n_items=len(items))
    dist.barrier()
    dist.destroy_process_group()
