"""Reverse mode through volume rendering -- drop-in for reference backward.py.

`backward_records(records, scene, d_color, d_depth)` (backward.py:35-101)
returns {'static': {param: grad}} like the reference.  For the ray path the
kernel re-marches each ray (no per-segment records are kept) and scatters
per-voxel gradients with warp-aggregated fp64 atomics into a dense
(M, 27) buffer.  Raster frames use `render_raster.rasterize_backward`.
Loss seeds (losses.py:22-46) are provided on the device.
"""

from __future__ import annotations

import torch

from . import _lib
from .device import grads_to_dict
from .render_ray import RenderRecords

PARAM_NAMES = ("w_s", "w_c", "w_sh", "log_a", "log_b")


def backward_grad_buffer(records: RenderRecords, d_color, d_depth,
                         grad: torch.Tensor | None = None, deterministic: bool = False) -> torch.Tensor:
    """Accumulate into / return the raw (M, 27) f64 gradient buffer.
    `deterministic=True`: per-segment rows + ordered per-voxel reduction
    instead of atomics (bitwise identical reruns).
    `d_color=None`: depth-only seeds (LiDAR), the kernel drops the colour terms."""
    lib = _lib.load()
    ds = records.scene
    dev = ds.device
    n = records.n_rays
    dc = _lib.as_f64(d_color, dev).reshape(n * 3) if d_color is not None else None
    dd = _lib.as_f64(d_depth, dev).reshape(n)
    if grad is None:
        grad = torch.zeros((max(ds.n, 1), _lib.GRAD_STRIDE), dtype=torch.float64, device=dev)
    if records.saved is None:
        raise ValueError("these records were rendered with need_state=False (inference): no backward")
    if n and records.ex_rec is not None:
        raise ValueError("records with actor segments: use backward_records")
    if n and deterministic:
        sc, t = ds.c_struct(), records.octree.c_struct()
        start = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        start[1:] = torch.cumsum(records.saved[:, 6].to(torch.int64), 0)
        slots = int(start[-1].item())
        wsb = lib.salf_ray_backward_det_workspace_bytes(slots, max(ds.n, 1))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        _lib.check(lib.salf_ray_backward_deterministic(
            _lib.ref(t), _lib.ref(sc), n, records.origins.data_ptr(), records.dirs.data_ptr(),
            _lib.ptr(records.valid), _lib.ref(records.opts), records.saved.data_ptr(), _lib.ptr(dc),
            dd.data_ptr(), grad.data_ptr(), start.data_ptr(), slots, ws.data_ptr(), wsb, _lib.stream_ptr()),
            "backward_records")
    elif n:
        sc, t = ds.c_struct(), records.octree.c_struct()
        _lib.check(lib.salf_ray_backward(_lib.ref(t), _lib.ref(sc), n, records.origins.data_ptr(),
                                         records.dirs.data_ptr(), _lib.ptr(records.valid),
                                         _lib.ref(records.opts), records.saved.data_ptr(),
                                         _lib.ptr(dc), dd.data_ptr(), grad.data_ptr(),
                                         _lib.stream_ptr()), "backward_records")
    return grad


def backward_records(records: RenderRecords, scene, d_color, d_depth) -> dict:
    """Parameter gradients per owner, 'static' and each actor id (backward.py:35-101)."""
    if records.ex_rec is None:
        grad = backward_grad_buffer(records, d_color, d_depth)
        out = {"static": grads_to_dict(grad[: records.scene.n])}
        for a in getattr(scene, "actors", []):
            out[a.actor_id] = grads_to_dict(torch.zeros((a.voxels.n, _lib.GRAD_STRIDE), dtype=torch.float64))
        return out
    lib = _lib.load()
    ds = records.scene
    dev = ds.device
    n = records.n_rays
    dc = _lib.as_f64(d_color, dev).reshape(n * 3)
    dd = _lib.as_f64(d_depth, dev).reshape(n)
    grad = torch.zeros((max(ds.n, 1), _lib.GRAD_STRIDE), dtype=torch.float64, device=dev)
    total = sum(c for _, _, c in records.actor_offsets)
    ex_grad = torch.zeros((max(total, 1), _lib.GRAD_STRIDE), dtype=torch.float64, device=dev)
    if n:
        sc, t = ds.c_struct(), records.octree.c_struct()
        _lib.check(lib.salf_ray_backward_merge(_lib.ref(t), _lib.ref(sc), n, records.origins.data_ptr(),
                                               records.dirs.data_ptr(), _lib.ptr(records.valid),
                                               _lib.ref(records.opts), records.ex_start.data_ptr(),
                                               records.ex_rec.data_ptr(), records.saved.data_ptr(),
                                               dc.data_ptr(), dd.data_ptr(), grad.data_ptr(),
                                               ex_grad.data_ptr(), _lib.stream_ptr()), "backward_records")
    out = {"static": grads_to_dict(grad[: ds.n])}
    for actor_id, off, cnt in records.actor_offsets:
        out[actor_id] = grads_to_dict(ex_grad[off:off + cnt])
    return out


def loss_color_seed(out_color: torch.Tensor, gt: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
    """losses.py:22-31: dL/dC = sign(C - gt) / (n_selected * 3)."""
    d = torch.zeros(out_color.shape, dtype=torch.float64, device=out_color.device)
    idx = torch.nonzero(mask, as_tuple=True)[0]
    if idx.numel():
        diff = out_color[idx].double() - gt.double()
        d[idx] = torch.sign(diff) / diff.numel()
    return d


def l1_color_seed(out_color: torch.Tensor, gt: torch.Tensor, mask: torch.Tensor | None = None,
                  count: int | None = None):
    """Fused losses.py:22-31 (one kernel): returns (dL/dC (.., 3) f64, sum |C - gt|
    over the selection as a 0-d f64 device tensor).  mask selects pixels
    (None = all); the normaliser is count, or 3 x #selected.  Unlike
    loss_color_seed (the reference's signature: gt holds the selected rows
    only), gt here is full-frame, same shape as out_color; host tensors are
    copied to the device."""
    lib = _lib.load()
    pred = out_color.reshape(-1).contiguous()
    if pred.dtype != torch.float32:
        pred = pred.float()
    n = pred.numel()
    g = torch.as_tensor(gt)
    if g.numel() != n:
        raise ValueError(f"gt must be full-frame like out_color ({n} values), got {g.numel()} "
                         "(loss_color_seed takes the selected rows only)")
    g = g.to(device=pred.device).reshape(-1).contiguous()
    if g.dtype not in (torch.float32, torch.float64):
        g = g.double()
    m = None
    if mask is not None:
        m = mask.reshape(-1).to(torch.uint8).contiguous()
        if count is None:
            count = 3 * int(m.sum().item())
    elif count is None:
        count = n
    d = torch.empty(n, dtype=torch.float64, device=pred.device)
    loss = torch.zeros((), dtype=torch.float64, device=pred.device)
    _lib.check(lib.salf_l1_seed(n, pred.data_ptr(), g.data_ptr(), int(g.dtype == torch.float64), _lib.ptr(m), 3,
                                1.0 / max(count, 1), d.data_ptr(), loss.data_ptr(), _lib.stream_ptr()), "l1_seed")
    return d.reshape(out_color.shape), loss


def loss_depth_seed(depth: torch.Tensor, gt: torch.Tensor, mask: torch.Tensor,
                    count: int | None = None) -> torch.Tensor:
    """losses.py:34-46: dL/dD = sign(D - gt) / #valid (count overrides #valid, e.g. a
    global count all-reduced across ranks)."""
    d = torch.zeros(depth.shape[0], dtype=torch.float64, device=depth.device)
    idx = torch.nonzero(mask, as_tuple=True)[0]
    if idx.numel() == 0:
        return d
    dep = depth[idx].double()
    g = gt.double()
    ok = torch.isfinite(dep) & torch.isfinite(g)
    idx = idx[ok]
    if idx.numel():
        d[idx] = torch.sign(dep[ok] - g[ok]) / (count if count else idx.numel())
    return d
