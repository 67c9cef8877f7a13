"""Multi-sensor training step (C5): sharded forward, globally normalised L1
seeds, backward into one dense per-voxel gradient buffer, all-reduce.

Mirrors the loss/backward part of the reference's train_loop step
(trainer.py:156-161: integrate/rasterize, loss_color, loss_depth,
backward_records); regularisers, Adam and densification are later §8(f) rows.
Cameras are rasterized (pinhole) in row bands; LiDARs go through the ray path
in ray blocks (parallel.py).  The step is split in two phases so the global
normalisation counts (reference losses.py:29-30, :44-45) can be all-reduced
between them.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import torch

from . import render_raster as RR
from . import render_ray as RY
from ._lib import nvtx
from .backward import l1_color_seed
from .parallel import allreduce_, allreduce_grad_, band_camera
from .render_ray import raise_for_status
from .sensors import CameraModel, gen_lidar_rays


@dataclass
class ForwardState:
    items: list
    saved: list  # per item: (state, diff)
    counts: torch.Tensor  # [n_color_terms, n_depth_returns] of this rank
    losses: torch.Tensor  # [sum |C - gt|, sum |D - gt|] of this rank


def color_terms(sensors) -> int:
    """Global normaliser of the cameras' L1 colour loss (losses.py:29-30): every
    pixel of every camera counts, 3 channels each -- known without a reduction."""
    return sum(3 * s.width * s.height for s in sensors if isinstance(s, CameraModel))


def rig_forward(ds, octree, sensors, targets, items, check: bool = True) -> ForwardState:
    """Forward of this rank's work items; targets[i]: (H, W, 3) gt colour for
    cameras, (beams * steps,) gt range for LiDARs.  Camera bands get their
    colour seeds in the same pass (the fused salf_l1_seed kernel: sign(C - gt)
    over the GLOBAL colour count, and |C - gt| summed); LiDAR seeds wait for the
    all-reduced return count.  `check`: raise like the reference's marcher for
    LiDAR rays that hit the round cap or leave the root (one host sync over all
    blocks, after every launch is queued)."""
    dev = ds.device
    counts = torch.zeros(2, dtype=torch.float64, device=dev)
    losses = torch.zeros(2, dtype=torch.float64, device=dev)
    saved = []
    statuses = []
    n_color = color_terms(sensors)
    for it in items:
        s = sensors[it.sensor]
        if it.kind == "raster_band":
            fb, st = RR.rasterize(ds, band_camera(s, it.lo, it.hi), return_state=True)
            gt = torch.as_tensor(targets[it.sensor], device=dev)[it.lo:it.hi]
            dc, lsum = l1_color_seed(fb.color, gt, None, count=n_color)
            counts[0] += 3 * fb.color.shape[0] * fb.color.shape[1]
            losses[0] += lsum
            saved.append((st, dc))
        else:
            # LiDAR block: the depth-only sweep kernel (no colour field), replayed by lidar_backward
            rays = gen_lidar_rays(s, device=dev)
            blk = SimpleNamespace(origins=rays.origins[it.lo:it.hi], dirs=rays.dirs[it.lo:it.hi],
                                  shape=(it.hi - it.lo,), generated=True)  # generated: unit by construction
            rec = RY.render_lidar(ds, octree, blk)
            statuses.append(rec.status)
            gt = torch.as_tensor(targets[it.sensor], device=dev)[it.lo:it.hi].double()
            dep = rec.depth.double()
            ok = torch.isfinite(dep) & torch.isfinite(gt)
            diff = torch.where(ok, dep - gt, torch.zeros_like(dep))
            counts[1] += ok.sum()
            losses[1] += diff.abs().sum()
            saved.append((rec, diff))
    if check and statuses:
        raise_for_status(torch.cat(statuses))
    return ForwardState(items, saved, counts, losses)


def rig_backward(fs: ForwardState, grad: torch.Tensor, global_counts: torch.Tensor,
                 depth_weight: float = 10.0) -> torch.Tensor:
    """Backward into `grad` (M, 27): camera bands with the seeds of the forward,
    LiDAR blocks with L1 seeds over the global return count."""
    n_d = global_counts[1].clamp_min(1.0)
    for it, (st, seed) in zip(fs.items, fs.saved):
        if it.kind == "raster_band":
            RR.rasterize_backward(st, seed, None, grad, as_dict=False)  # cameras carry the colour loss only
        else:
            dd = depth_weight * torch.sign(seed) / n_d
            RY.lidar_backward(st, dd, grad=grad)  # depth-only seeds: no colour terms
    return grad


def rig_step(ds, octree, sensors, targets, items, grad: torch.Tensor, depth_weight: float = 10.0):
    """One rank's share of a training step; all-reduces the counts, the
    gradient buffer and the loss sums.  Returns (loss_sums, global_counts)."""
    with nvtx("rig_forward"):
        fs = rig_forward(ds, octree, sensors, targets, items)
    with nvtx("rig_allreduce_counts"):
        counts = allreduce_(fs.counts.clone())
    with nvtx("rig_backward"):
        rig_backward(fs, grad, counts, depth_weight)
    with nvtx("rig_allreduce_grad"):
        allreduce_grad_(grad)
    losses = allreduce_(fs.losses.clone())
    return losses, counts
