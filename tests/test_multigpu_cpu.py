"""Host-side multi-rank logic on CPU: sharding/assignment and the gradient /
count all-reduce, exercised with torch.distributed gloo at world_size 2."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_18713_b200 import configs
from paper_2507_18713_b200.parallel import assign, band_camera, split_work


def test_split_covers_every_row_and_ray_once():
    cams, lidars = configs.c5_rig()
    sensors = cams + lidars
    for world in (1, 2, 3, 4, 8):
        items = split_work(sensors, world)
        for i, s in enumerate(sensors):
            mine = sorted((it.lo, it.hi) for it in items if it.sensor == i)
            total = s.height if i < len(cams) else s.beam_elevations.shape[0] * s.steps
            assert mine[0][0] == 0 and mine[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(mine, mine[1:]))
            if i < len(cams):
                assert all(lo % 16 == 0 for lo, _ in mine)  # bands align to tile rows


def test_lpt_balance():
    cams, lidars = configs.c5_rig()
    for world in (2, 4, 8):
        per = assign(split_work(cams + lidars, world), world)
        loads = [sum(it.cost for it in lst) for lst in per]
        assert max(loads) <= 1.35 * (sum(loads) / world)
        assert sum(len(x) for x in per) == len(split_work(cams + lidars, world))


def test_band_camera_is_row_window():
    cam = configs.c2_camera(width=64, height=48)
    b = band_camera(cam, 16, 32)
    assert b.height == 16 and b.cy == cam.cy - 16 and b.fx == cam.fx


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_18713_b200.parallel import allreduce_
    g = torch.full((5, 27), float(rank + 1), dtype=torch.float64)
    allreduce_(g)
    counts = torch.tensor([3.0 * (rank + 1), float(rank)], dtype=torch.float64)
    allreduce_(counts)
    out[rank] = (g.numpy().copy(), counts.numpy().copy())
    dist.destroy_process_group()


def test_gloo_allreduce_world2():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    for r in (0, 1):
        g, c = res[r]
        assert np.all(g == 3.0)
        np.testing.assert_array_equal(c, [9.0, 1.0])


def _grad_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_18713_b200.parallel import allreduce_grad_
    rng = np.random.default_rng(rank)
    m = 400
    g = np.zeros((m, 27))
    rows = rng.choice(m, size=60, replace=False)  # each rank touches its own rows (partly shared)
    g[rows] = rng.normal(size=(60, 27)) * (1.0 + 1e-12)  # NOT fp32-representable
    g[rows[:5], :3] = 0.0  # rows with some zero components stay touched
    dense = torch.as_tensor(g.copy())
    sparse = torch.as_tensor(g.copy())
    f32 = torch.as_tensor(g.copy())
    allreduce_grad_(dense, sparse=False)
    allreduce_grad_(sparse, sparse=True)
    allreduce_grad_(f32, sparse=True, transport=torch.float32)
    out[rank] = (g, dense.numpy().copy(), sparse.numpy().copy(), f32.numpy().copy())
    dist.destroy_process_group()


def test_gloo_sparse_grad_allreduce_equals_dense_world2():
    """parallel.allreduce_grad_: the touched-rows all-reduce (union of the
    ranks' non-zero-row masks) gives exactly the dense sum, and the default f64
    transport gives exactly the world-1 sum of the two ranks' f64 buffers
    (values that are not fp32-representable); fp32 transport is opt-in."""
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_grad_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    want = res[0][0] + res[1][0]
    want32 = (res[0][0].astype(np.float32) + res[1][0].astype(np.float32)).astype(np.float64)
    assert not np.array_equal(want, want32)
    for r in (0, 1):
        _, dense, sparse, f32 = res[r]
        np.testing.assert_array_equal(dense, sparse)
        np.testing.assert_array_equal(sparse, want)
        np.testing.assert_array_equal(f32, want32)
