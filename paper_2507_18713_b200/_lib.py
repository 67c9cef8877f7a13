"""ctypes binding of libsalf_b200.so (C ABI declared in include/salf_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2507_18713_b200/csrc`).  There is no CPU fallback: if the
library or a CUDA device is missing, every render call raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import torch

import os

# SALF_LIB overrides the library path (A/B builds of the same ABI)
LIB_PATH = Path(os.environ.get("SALF_LIB") or Path(__file__).resolve().parent / "libsalf_b200.so")

SALF_OK, SALF_EINVAL, SALF_ENOTERM, SALF_ECUDA, SALF_EWORKSPACE = 0, 1, 2, 3, 4
KINDS = {"pinhole": 0, "fisheye_equidistant": 1, "equirect": 2}
DENSITY = {"sdf": 0, "raw": 1}
PRM_STRIDE = 28
SAVED_STRIDE = 8
GRAD_STRIDE = 27

c_double3 = C.c_double * 3
c_double9 = C.c_double * 9
c_double4 = C.c_double * 4
vp = C.c_void_p


class SceneT(C.Structure):
    _fields_ = [("n", C.c_int64), ("geo", vp), ("aux", vp), ("prm", vp), ("rot", vp),
                ("density_mode", C.c_int32), ("pad", C.c_int32)]


class CameraT(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("pad", C.c_int32), ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double), ("k", c_double4), ("position", c_double3), ("rot", c_double9),
                ("readout_duration", C.c_double), ("linear_velocity", c_double3),
                ("angular_velocity", c_double3), ("t0", C.c_double)]


class LidarT(C.Structure):
    _fields_ = [("n_beams", C.c_int32), ("steps", C.c_int32), ("azimuth_start", C.c_double),
                ("azimuth_end", C.c_double), ("scan_period", C.c_double),
                ("position", c_double3), ("rot", c_double9), ("linear_velocity", c_double3),
                ("angular_velocity", c_double3), ("t0", C.c_double)]


class OctreeT(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("nodes", vp), ("root_min", c_double3),
                ("root_edge", C.c_double), ("max_depth", C.c_int32), ("jump_levels", C.c_int32),
                ("jump", vp)]


class SphereT(C.Structure):
    _fields_ = [("center", c_double3), ("radius", C.c_double), ("ior", C.c_double), ("albedo", c_double3),
                ("material", C.c_int32), ("pad", C.c_int32)]


class RasterOptsT(C.Structure):
    _fields_ = [("background", c_double3), ("near", C.c_double), ("stop_threshold", C.c_double),
                ("tile", C.c_int32), ("exact_color", C.c_int32)]


# name -> (restype, argtypes); every symbol declared in include/salf_b200.h
SIGNATURES = {
    "salf_last_error": (C.c_char_p, []),
    "salf_device_sm_count": (C.c_int, []),
    "salf_project_voxels": (C.c_int, [vp, vp, C.c_double, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_raster_bin_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64, C.c_int32]),
    "salf_raster_bin": (C.c_int, [vp, vp, C.c_double, C.c_int32, C.c_int32, vp, vp, vp, vp,
                                  C.c_size_t, C.c_int64, vp, vp, vp, vp]),
    "salf_sort_pairs_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int32, C.c_int32]),
    "salf_sort_pairs": (C.c_int, [vp, vp, vp, vp, C.c_int32, vp, C.c_int64, C.c_int32, C.c_int32, vp,
                                  C.c_size_t, vp]),
    "salf_sort_pairs_unique_workspace_bytes": (C.c_size_t, []),
    "salf_sort_pairs_unique": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, C.c_size_t, vp]),
    "salf_raster_composite": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_raster_hitbits_words": (C.c_size_t, [C.c_int64, C.c_int32]),
    "salf_raster_backward": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_raster_backward_det_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64]),
    "salf_raster_tile_order_workspace_bytes": (C.c_size_t, [C.c_int32]),
    "salf_raster_tile_order": (C.c_int, [vp, C.c_int32, vp, vp, C.c_size_t, vp]),
    "salf_ray_backward_det_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64]),
    "salf_ray_backward_deterministic": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int64,
                                                  vp, C.c_size_t, vp]),
    "salf_raster_backward_deterministic": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp,
                                                     vp, vp, C.c_size_t, vp]),
    "salf_camera_rays": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "salf_lidar_rays": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "salf_lidar_batch": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_camera_batch": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "salf_octree_build_host": (C.c_int, [C.c_int64, vp, vp, C.c_int32, vp, C.c_int64, vp, vp]),
    "salf_octree_query": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp]),
    "salf_octree_jump_bytes": (C.c_size_t, [C.c_int32]),
    "salf_octree_jump_build": (C.c_int, [vp, C.c_int32, vp, vp]),
    "salf_march": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp, C.c_double, C.c_int32, vp, vp, vp,
                             vp, vp, vp, vp]),
    "salf_ray_forward": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_ray_backward": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_lidar_forward": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_lidar_backward": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_adam_step": (C.c_int, [C.c_int64, vp, vp, vp, vp, C.c_double, C.c_double, C.c_double,
                                 C.c_double, C.c_int64, vp]),
    "salf_scene_refresh": (C.c_int, [vp, C.c_int64, vp, vp, vp]),
    "salf_loss_eikonal": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp]),
    "salf_center_alpha": (C.c_int, [vp, vp, C.c_int32, C.c_int64, vp, vp, vp]),
    "salf_loss_empty_grad": (C.c_int, [vp, vp, C.c_int32, C.c_int64, vp, vp, vp]),
    "salf_loss_opacity_lidar": (C.c_int, [vp, vp, C.c_int32, C.c_int64, vp, vp, vp, vp, vp]),
    "salf_loss_smooth": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp]),
    "salf_fp64_peak": (C.c_int, [vp, C.c_int32, C.c_int32, vp]),
    "salf_fp32_peak": (C.c_int, [vp, C.c_int32, C.c_int32, vp]),
    "salf_effects_wave": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int32, vp, vp, vp, vp, vp,
                                    vp, vp, vp, vp, vp, vp]),
    "salf_decode_records": (C.c_int, [C.c_int64, vp, vp, C.c_double, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_l1_seed": (C.c_int, [C.c_int64, vp, vp, C.c_int32, vp, C.c_int32, C.c_double, vp, vp, vp]),
    "salf_densify_flags": (C.c_int, [C.c_int64, vp, vp, vp, C.c_int32, C.c_double, C.c_int32, vp, vp, vp]),
    "salf_grad_norm_acc": (C.c_int, [C.c_int64, vp, vp, vp]),
    "salf_densify_apply": (C.c_int, [C.c_int64, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                     vp]),
    "salf_voxel_geometry": (C.c_int, [C.c_int64, vp, vp, vp, C.c_double, vp, vp, vp, vp, vp]),
    "salf_octree_ancestor_keys": (C.c_int, [C.c_int64, vp, vp, C.c_int32, vp, vp, vp, vp]),
    "salf_octree_fill": (C.c_int, [C.c_int64, C.c_int64, vp, vp, vp, vp, vp]),
    "salf_actor_rays": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_shade_segments": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp, vp, C.c_int32, C.c_int64, C.c_int32,
                                      vp, vp]),
    "salf_ray_forward_merge": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "salf_ray_backward_merge": (C.c_int, [vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                          vp]),
}

_lib = None


def load(require_cuda: bool = True):
    """Load the shared library (fails loudly; no fallback)."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("paper_2507_18713_b200 needs a CUDA device (sm_100a); none is visible")
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(make -C paper_2507_18713_b200/csrc) first")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, where: str = "") -> None:
    if rc == SALF_OK:
        return
    msg = load(require_cuda=False).salf_last_error().decode("utf-8", "replace")
    if rc == SALF_EINVAL:
        raise ValueError(msg)
    if rc == SALF_ENOTERM:
        raise RuntimeError(msg)
    raise RuntimeError(f"{where}: {msg}" if where else msg)


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ref(struct):
    return C.byref(struct)


def as_f64(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.array(x, dtype=np.float64, order="C"), device=device)


# NVTX ranges around the phases of a frame (SALF_NVTX=1; e.g. `ncu --nvtx
# --nvtx-include "raster_backward/"`): a no-op context otherwise.
NVTX = os.environ.get("SALF_NVTX", "0") == "1"


class _NoRange:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_NO_RANGE = _NoRange()


def nvtx(name: str):
    return torch.cuda.nvtx.range(name) if NVTX else _NO_RANGE
