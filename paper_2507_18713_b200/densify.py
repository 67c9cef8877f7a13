"""Densify / prune round on the device -- drop-in for reference densify.py
(`center_opacity` :39-46, `split_count` :49-50, `densify_and_prune` :53-94)
and the trainer's use of it with the Adam moment remap (trainer.py:194-206,
optim.py:35-40).

Per-voxel work runs in libsalf_b200 (csrc/salf_densify.cu): centre opacity
and the prune / eligible flags, the gradient-norm accumulator, the gather of
kept rows and the 8-child expansion of split rows (parameters inherited,
moments zeroed), and the device scene arrays of the new set.  The ranking
between them -- the reference's lexsort by gradient norm with index
tie-break, then flatnonzero -- is a stable device sort / selection.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .scene import DENSITY_SDF, SparseVoxelSet

SPLIT_DENOMINATOR = 8 * 5   # densify.py:22
PRUNE_OPACITY = 0.005       # densify.py:23
PARAMS = ("w_s", "w_c", "w_sh", "log_a", "log_b")


@dataclass
class DensifyConfig:
    """densify.py:31-36."""

    budget: int = 2_500_000
    prune_opacity: float = PRUNE_OPACITY
    interval: int = 400
    stop_fraction: float = 0.8


def split_count(budget: int, n: int, n_prune: int) -> int:
    """densify.py:49-50."""
    return max(0, (budget + n_prune - n) // SPLIT_DENOMINATOR)


def _block(v: SparseVoxelSet) -> np.ndarray:
    m = v.n
    b = np.empty((m, 27), np.float64)
    b[:, 0:4] = v.w_s
    b[:, 4:13] = v.w_c.reshape(m, 9)
    b[:, 13:25] = v.w_sh.reshape(m, 12)
    b[:, 25] = v.log_a
    b[:, 26] = v.log_b
    return b


def _flags(params, geo, level, mode, prune_opacity, max_levels, want_opacity=False):
    lib = _lib.load()
    n = level.numel()
    flags = torch.empty(max(n, 1), dtype=torch.uint8, device=level.device)
    opa = torch.empty(max(n, 1), dtype=torch.float64, device=level.device) if want_opacity else None
    _lib.check(lib.salf_densify_flags(n, params.data_ptr(), geo.data_ptr(), level.data_ptr(),
                                      _lib.DENSITY[mode], float(prune_opacity), int(max_levels),
                                      flags.data_ptr(), _lib.ptr(opa), _lib.stream_ptr()), "densify")
    return flags[:n], (opa[:n] if opa is not None else None)


def _geo_from_set(v: SparseVoxelSet, dev) -> torch.Tensor:
    geo = np.empty((max(v.n, 1), 4), np.float64)
    if v.n:
        geo[:v.n, :3] = v.centers()
        geo[:v.n, 3] = v.edges()
    return torch.as_tensor(geo, device=dev)


def center_opacity(vset: SparseVoxelSet, mode: str = DENSITY_SDF, device=None) -> np.ndarray:
    """densify.py:39-46: opacity at the voxel centre over its own edge length."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if vset.n == 0:
        return np.zeros(0)
    params = torch.as_tensor(_block(vset), device=dev)
    level = torch.as_tensor(vset.level.astype(np.uint8), device=dev)
    _f, opa = _flags(params, _geo_from_set(vset, dev), level, mode, PRUNE_OPACITY,
                     vset.bounds.max_levels, want_opacity=True)
    return opa.cpu().numpy()


def densify_device(params: torch.Tensor, geo: torch.Tensor, level: torch.Tensor, ijk: torch.Tensor,
                   grad_norms: torch.Tensor, cfg: DensifyConfig, max_levels: int, mode: str = DENSITY_SDF,
                   m: torch.Tensor | None = None, v: torch.Tensor | None = None) -> dict:
    """One prune + split round on device arrays: params (n, 27) f64, geo
    (n, 4) f64, level (n,) u8, ijk (n, 3) i32, grad_norms (n,) f64 and the
    optional Adam moments (n, 27).  Returns the new arrays, keep_idx and
    n_split (densify.py:53-94, optim.py:35-40)."""
    lib = _lib.load()
    dev = params.device
    n = level.numel()
    flags, _ = _flags(params, geo, level, mode, cfg.prune_opacity, max_levels)
    prune = (flags & 1).bool()
    eligible = (flags & 2).bool()
    n_prune = int(prune.sum().item())
    want = split_count(cfg.budget, n, n_prune)
    # np.lexsort((arange, -grad)): grad descending, ties by index (stable sort)
    order = torch.sort(-grad_norms.to(torch.float64), stable=True).indices
    cand = order[eligible[order]]
    split_idx = torch.sort(cand[:want]).values.contiguous()
    split = torch.zeros(n, dtype=torch.bool, device=dev)
    split[split_idx] = True
    keep_idx = torch.nonzero(~prune & ~split, as_tuple=True)[0].contiguous()
    n_keep, n_split = int(keep_idx.numel()), int(split_idx.numel())
    rows = n_keep + 8 * n_split
    if rows > cfg.budget:
        raise RuntimeError(f"densification exceeded the budget: {rows} > {cfg.budget}")
    out = {
        "level": torch.empty(max(rows, 1), dtype=torch.uint8, device=dev),
        "ijk": torch.empty((max(rows, 1), 3), dtype=torch.int32, device=dev),
        "params": torch.empty((max(rows, 1), 27), dtype=torch.float64, device=dev),
        "m": torch.empty((max(rows, 1), 27), dtype=torch.float64, device=dev) if m is not None else None,
        "v": torch.empty((max(rows, 1), 27), dtype=torch.float64, device=dev) if v is not None else None,
    }
    _lib.check(lib.salf_densify_apply(n_keep, keep_idx.data_ptr() if n_keep else 0, n_split,
                                      split_idx.data_ptr() if n_split else 0, level.data_ptr(),
                                      ijk.data_ptr(), params.data_ptr(), _lib.ptr(m), _lib.ptr(v),
                                      out["level"].data_ptr(), out["ijk"].data_ptr(),
                                      out["params"].data_ptr(), _lib.ptr(out["m"]), _lib.ptr(out["v"]),
                                      _lib.stream_ptr()), "densify")
    for k in ("level", "ijk", "params", "m", "v"):
        if out[k] is not None:
            out[k] = out[k][:rows]
    out.update(keep_idx=keep_idx, split_idx=split_idx, n_split=n_split, n_prune=n_prune)
    return out


def densify_and_prune(vset: SparseVoxelSet, grad_norms, cfg: DensifyConfig = DensifyConfig(),
                      mode: str = DENSITY_SDF, device=None):
    """densify.py:53-94: one prune + split round; returns (new set, kept old
    indices, n_split).  Candidates ranked by accumulated gradient norm (ties
    by index), finest-level voxels skipped; children inherit every parameter."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = vset.n
    params = torch.as_tensor(_block(vset), device=dev).contiguous()
    level = torch.as_tensor(vset.level.astype(np.uint8), device=dev)
    ijk = torch.as_tensor(np.ascontiguousarray(vset.ijk.astype(np.int32)), device=dev)
    g = torch.as_tensor(np.asarray(grad_norms, np.float64).reshape(n), device=dev)
    r = densify_device(params, _geo_from_set(vset, dev), level, ijk, g, cfg, vset.bounds.max_levels, mode)
    new = SparseVoxelSet(vset.bounds, budget=cfg.budget)
    b = r["params"].cpu().numpy()
    m = b.shape[0]
    new.set_arrays(r["level"].cpu().numpy(), r["ijk"].cpu().numpy(), b[:, 0:4], b[:, 4:13].reshape(m, 3, 3),
                   b[:, 13:25].reshape(m, 3, 4), b[:, 25], b[:, 26])
    keep_idx = r["keep_idx"].cpu().numpy().astype(np.int64)
    split_idx = r["split_idx"].cpu().numpy().astype(np.int64)
    rot = np.asarray(vset.rotation)
    new.rotation = np.concatenate([rot[keep_idx], np.repeat(rot[split_idx], 8, axis=0)])
    return new, keep_idx, int(r["n_split"])
