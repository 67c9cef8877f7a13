"""Multi-sensor training step (C5): sharded forward, globally normalised L1
seeds, backward into one dense per-voxel gradient buffer, all-reduce.

Mirrors the loss/backward part of the reference's train_loop step
(trainer.py:156-161: integrate/rasterize, loss_color, loss_depth,
backward_records); regularisers, Adam and densification are later §8(f) rows.
Cameras are rasterized (pinhole) in row bands; LiDARs go through the ray path
in ray blocks (parallel.py).
"""

from __future__ import annotations

import torch

from . import _lib
from . import render_raster as RR
from . import render_ray as RY
from .backward import backward_grad_buffer
from .parallel import allreduce_, band_camera
from .sensors import CameraModel, gen_lidar_rays


def rig_step(ds, octree, sensors, targets, items, grad: torch.Tensor, depth_weight: float = 10.0):
    """One rank's share of a training step.

    sensors: list of CameraModel (pinhole) / LidarModel; targets[i]: (H, W, 3)
    gt colour for cameras, (beams*steps,) gt range for LiDARs (CUDA tensors).
    items: this rank's WorkItems.  Accumulates into `grad` (M, 27) and
    all-reduces it; returns (color_loss_sum, depth_loss_sum, counts)."""
    dev = ds.device
    fwd = []
    n_color = torch.zeros(1, dtype=torch.float64, device=dev)
    n_depth = torch.zeros(1, dtype=torch.float64, device=dev)
    l_color = torch.zeros(1, dtype=torch.float64, device=dev)
    l_depth = torch.zeros(1, dtype=torch.float64, device=dev)
    for it in items:
        s = sensors[it.sensor]
        if it.kind == "raster_band":
            cam = band_camera(s, it.lo, it.hi)
            fb, st = RR.rasterize(ds, cam, return_state=True)
            gt = targets[it.sensor][it.lo:it.hi].to(dev)
            diff = fb.color.double() - gt.double()
            n_color += diff.numel()
            l_color += diff.abs().sum()
            fwd.append((it, st, diff))
        else:
            rays = gen_lidar_rays(s, device=dev)
            o, d = rays.origins[it.lo:it.hi], rays.dirs[it.lo:it.hi]
            rec = RY.integrate_rays(ds, octree, o, d)
            gt = targets[it.sensor][it.lo:it.hi].to(dev).double()
            dep = rec.depth.double()
            ok = torch.isfinite(dep) & torch.isfinite(gt)
            diff = torch.where(ok, dep - gt, torch.zeros_like(dep))
            n_depth += ok.sum()
            l_depth += diff.abs().sum()
            fwd.append((it, rec, diff))
    # global normalisation: L1 means over all ranks' selected rays
    counts = torch.cat([n_color, n_depth])
    allreduce_(counts)
    for it, st, diff in fwd:
        if it.kind == "raster_band":
            dc = torch.sign(diff) / counts[0].clamp_min(1.0)
            dd = torch.zeros(diff.shape[:2], dtype=torch.float64, device=dev)
            RR.rasterize_backward(st, dc, dd, grad, as_dict=False)
        else:
            dd = depth_weight * torch.sign(diff) / counts[1].clamp_min(1.0)
            dc = torch.zeros((diff.shape[0], 3), dtype=torch.float64, device=dev)
            backward_grad_buffer(st, dc, dd, grad)
    allreduce_(grad)
    losses = torch.cat([l_color, l_depth])
    allreduce_(losses)
    return losses, counts
