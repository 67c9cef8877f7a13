"""Multi-GPU sharding of the render path.

One process per GPU; the scene is replicated.  Work items are sensors, split
into row bands (pinhole cameras, multiples of the 16-pixel tile so a band
renders bit-identically to the same rows of the full frame) or ray blocks
(LiDAR / ray-path cameras), assigned to ranks by longest-processing-time
greedy on an estimated cost.  Forward needs no exchange; the training
backward sums per-voxel gradients with one all-reduce (NCCL over NVLink on
the GPU box, gloo in the CPU tests), after the L1 loss seeds were normalised
by globally all-reduced counts (reference losses.py:29-30, :44-45).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .sensors import PINHOLE, CameraModel, LidarModel


@dataclass(frozen=True)
class WorkItem:
    sensor: int  # index into the rig's sensor list
    kind: str  # "raster_band" | "ray_block"
    lo: int  # first row (band) or first ray (block)
    hi: int  # one past the last
    cost: float


def sensor_rays(s) -> int:
    if isinstance(s, LidarModel):
        return int(s.beam_elevations.shape[0] * s.steps)
    return int(s.width * s.height)


def split_work(sensors, world_size: int, tile: int = 16, ray_cost: float = 1.0,
               raster_cost: float = 1.0) -> list:
    """Cut sensors into items no larger than ~1/world of the total cost."""
    costs = []
    for s in sensors:
        per_ray = raster_cost if isinstance(s, CameraModel) and s.kind == PINHOLE else ray_cost
        costs.append(per_ray * sensor_rays(s))
    target = sum(costs) / max(world_size, 1)
    items = []
    for i, (s, c) in enumerate(zip(sensors, costs)):
        n_parts = max(1, int(np.ceil(c / target - 1e-9))) if world_size > 1 else 1
        if isinstance(s, CameraModel) and s.kind == PINHOLE:
            tiles_y = -(-s.height // tile)
            n_parts = min(n_parts, tiles_y)
            cuts = np.linspace(0, tiles_y, n_parts + 1).round().astype(int) * tile
            cuts[-1] = s.height
            for a, b in zip(cuts[:-1], cuts[1:]):
                if b > a:
                    items.append(WorkItem(i, "raster_band", int(a), int(b), c * (b - a) / s.height))
        else:
            n = sensor_rays(s)
            cuts = np.linspace(0, n, n_parts + 1).round().astype(int)
            for a, b in zip(cuts[:-1], cuts[1:]):
                if b > a:
                    items.append(WorkItem(i, "ray_block", int(a), int(b), c * (b - a) / n))
    return items


def assign(items: list, world_size: int) -> list:
    """LPT greedy: biggest item to the least-loaded rank; returns per-rank lists."""
    load = np.zeros(world_size)
    out = [[] for _ in range(world_size)]
    for it in sorted(items, key=lambda x: (-x.cost, x.sensor, x.lo)):
        r = int(np.argmin(load))
        out[r].append(it)
        load[r] += it.cost
    for lst in out:
        lst.sort(key=lambda x: (x.sensor, x.lo))
    return out


def band_camera(cam: CameraModel, r0: int, r1: int) -> CameraModel:
    """Rows [r0, r1) of a pinhole frame as a camera of its own (cy shifted)."""
    return replace(cam, height=r1 - r0, cy=cam.cy - r0)


def _world(group=None) -> int:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


def allreduce_(t, group=None):
    """Sum a tensor across ranks in place (no-op when not distributed)."""
    import torch.distributed as dist
    if _world(group) > 1:
        dist.all_reduce(t, group=group)
    return t


def allreduce_grad_(grad, group=None, sparse: bool = True, transport=None):
    """Sum the dense (M, 27) f64 per-voxel gradient buffer across ranks.

    The buffer travels in its own dtype (f64) by default, so world > 1 sums
    equal the world = 1 buffer up to the order of one addition per rank.
    `transport=torch.float32` is an explicit opt-in that halves the NVLink
    bytes at the cost of rounding each rank's partial sums to fp32 first.
    With `sparse`, only the rows some rank wrote move: the union of the ranks'
    non-zero-row masks (a 1-byte MAX all-reduce) selects the rows, which are
    gathered, summed and scattered back.  A frame touches ~20% of an S1M
    scene, so the sum moves ~5x fewer bytes; rows outside the union are zero
    on every rank, so the result is identical to the dense sum."""
    import torch
    import torch.distributed as dist
    if _world(group) <= 1:
        return grad
    transport = grad.dtype if transport is None else transport
    if not sparse:
        t = grad if transport == grad.dtype else grad.to(transport)
        dist.all_reduce(t, group=group)
        if t is not grad:
            grad.copy_(t)
        return grad
    mask = (grad != 0).any(dim=1).to(torch.uint8)
    dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)
    idx = mask.nonzero().squeeze(1)
    rows = grad.index_select(0, idx).to(transport)
    dist.all_reduce(rows, group=group)
    grad.index_copy_(0, idx, rows.to(grad.dtype))
    return grad
