"""Tile rasterizer for pinhole cameras -- drop-in for reference render_raster.py.

Same entry points and arguments as the reference (`project_voxels` :97,
`cull_and_bin` :143, `rasterize` :201, `rasterize_scene` :304); the work runs
in libsalf_b200 (csrc/salf_raster.cu).  Outputs are CUDA tensors (float32
image planes); `Framebuffer.numpy()` converts for host callers.

Two bin lists exist for one frame:
  * reference bins (`cull_and_bin`): the reference's CSR bit for bit,
    including near-plane-straddling voxels in every tile;
  * render bins (used by `rasterize`): each tile's list restricted to voxels
    whose clipped footprint reaches the tile -- a per-tile subsequence of the
    reference list that drops only pairs with alpha = 0 exactly, so the
    composited result is unchanged.
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceScene, as_device_scene, grads_to_dict
from .scene import FlatVoxels, Scene, flatten_scene
from .sensors import PINHOLE, CameraModel

TILE_SIZE = 16
NEAR_PLANE = 0.05
STOP_THRESHOLD = 0.99


@dataclass
class Framebuffer:
    color: torch.Tensor  # (H, W, 3) f32
    opacity: torch.Tensor  # (H, W) f32
    depth: torch.Tensor  # (H, W) f32, NaN = no return

    def numpy(self):
        return Framebuffer(self.color.cpu().numpy().astype(np.float64),
                           self.opacity.cpu().numpy().astype(np.float64),
                           self.depth.cpu().numpy().astype(np.float64))


@dataclass
class TileBins:
    tiles_x: int
    tiles_y: int
    tile: int
    offsets: np.ndarray  # (tiles + 1,) int64
    entries: np.ndarray  # voxel indices, (center depth, index) order per tile


@dataclass
class RasterState:
    """What the backward needs from one rasterized frame."""

    scene: DeviceScene
    cam: CameraModel
    opts: _lib.RasterOptsT
    offsets: torch.Tensor
    entries: torch.Tensor
    saved: torch.Tensor
    n_instances: int
    vrange: torch.Tensor | None = None  # per-voxel footprint rows (entry culling per warp)
    tile_order: torch.Tensor | None = None  # launch order of the tiles (longest lists first)
    hitbits: torch.Tensor | None = None  # included-hit words per (tile, pixel, 32 entries) (default mode)


def _timed(events, name):
    """Profiling hook: append (name, start, end) CUDA events around one launch."""
    if events is None:
        return None
    e = (name, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    e[1].record()
    events.append(e)
    return e


def _require_pinhole(cam: CameraModel) -> None:
    if cam.kind != PINHOLE:
        raise ValueError(f"rasterizer supports pinhole cameras only, got {cam.kind!r}")


class _Workspace:
    """Per-device grow-only scratch (the C ABI never allocates)."""

    def __init__(self):
        self.buf = {}

    def get(self, device, nbytes: int, slot: str = "bin") -> torch.Tensor:
        key = (str(device), slot)
        t = self.buf.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self.buf[key] = t
        return t


_WS = _Workspace()
_CAPACITY: dict = {}


def _project(ds: DeviceScene, cam: CameraModel, near: float, tile: int, want_rect: bool = False):
    lib = _lib.load()
    m = max(ds.n, 1)
    dev = ds.device
    out = dict(
        span_ref=torch.empty((m, 4), dtype=torch.int32, device=dev),
        span_fit=torch.empty((m, 4), dtype=torch.int32, device=dev),
        zkey=torch.empty(m, dtype=torch.int64, device=dev),
        vrange=torch.empty((m, 2), dtype=torch.int32, device=dev),  # footprint rows, columns
    )
    if want_rect:
        out["rect"] = torch.empty((m, 4), dtype=torch.float64, device=dev)
        out["zc"] = torch.empty(m, dtype=torch.float64, device=dev)
        out["culled"] = torch.empty(m, dtype=torch.uint8, device=dev)
    sc, cs = ds.c_struct(), cam.c_struct(rolling=False)
    _lib.check(lib.salf_project_voxels(
        _lib.ref(sc), _lib.ref(cs), float(near), int(tile), _lib.ptr(out.get("rect")),
        _lib.ptr(out.get("zc")), _lib.ptr(out.get("culled")), out["span_ref"].data_ptr(),
        out["span_fit"].data_ptr(), out["zkey"].data_ptr(), out["vrange"].data_ptr(), _lib.stream_ptr()),
        "project_voxels")
    return out


def _bin(ds: DeviceScene, cam: CameraModel, near: float, tile: int, proj: dict, mode: int):
    """Enqueue the binning of one frame (no host synchronisation: the counts stay
    on the device).  Returns (offsets, entries[capacity], counts (2,) int64 on the
    device: visible voxels, instances; capacity, (tiles_x, tiles_y))."""
    lib = _lib.load()
    dev = ds.device
    tx = -(-cam.width // tile)
    ty = -(-cam.height // tile)
    n_tiles = tx * ty
    offsets = torch.empty(n_tiles + 1, dtype=torch.int64, device=dev)
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    span = proj["span_ref"] if mode == 0 else proj["span_fit"]
    cap = _CAPACITY.get((str(dev), mode), 1 << 20)
    sc, cs = ds.c_struct(), cam.c_struct(rolling=False)
    entries = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    wsb = lib.salf_raster_bin_workspace_bytes(max(ds.n, 1), cap, n_tiles)
    ws = _WS.get(dev, wsb)
    _lib.check(lib.salf_raster_bin(_lib.ref(sc), _lib.ref(cs), float(near), int(tile), int(mode),
                                   proj["zkey"].data_ptr(), span.data_ptr(), None, ws.data_ptr(),
                                   ws.numel(), cap, offsets.data_ptr(), entries.data_ptr(),
                                   counts.data_ptr(), _lib.stream_ptr()), "cull_and_bin")
    return offsets, entries, counts, cap, (tx, ty)


class _Counts:
    """Pinned host copy of a frame's bin counts, read once the stream reaches it
    (an event wait after the frame's kernels are enqueued: the GPU never idles)."""

    def __init__(self, counts: torch.Tensor):
        self.host = torch.empty(2, dtype=torch.int64, pin_memory=True)
        self.host.copy_(counts, non_blocking=True)
        self.event = torch.cuda.Event()
        self.event.record()

    def n_instances(self) -> int:
        self.event.synchronize()
        return int(self.host[1])


def _grow(dev, mode: int, need: int) -> None:
    _CAPACITY[(str(dev), mode)] = int(need * 1.25) + 1024


def _bin_sync(ds: DeviceScene, cam: CameraModel, near: float, tile: int, proj: dict, mode: int):
    """_bin, then wait for the count (the host API returns arrays); re-bins once
    with a larger capacity if the lists did not fit."""
    for _ in range(2):
        offsets, entries, counts, cap, txy = _bin(ds, cam, near, tile, proj, mode)
        n = _Counts(counts).n_instances()
        if n <= cap:
            return offsets, entries[:n], n, txy
        _grow(ds.device, mode, n)
    raise RuntimeError("raster binning failed to size its instance capacity")


def project_voxels(flat, cam: CameraModel, near: float = NEAR_PLANE):
    """render_raster.py:97-129 -> (rect_min (M,2), rect_max (M,2), z_center, culled), NumPy."""
    _require_pinhole(cam)
    ds = as_device_scene(flat)
    if ds.n == 0:
        z = np.zeros((0, 2))
        return z, z.copy(), np.zeros(0), np.zeros(0, bool)
    p = _project(ds, cam, near, TILE_SIZE, want_rect=True)
    rect = p["rect"][: ds.n].cpu().numpy()
    return (rect[:, 0:2].copy(), rect[:, 2:4].copy(), p["zc"][: ds.n].cpu().numpy(),
            p["culled"][: ds.n].cpu().numpy().astype(bool))


def cull_and_bin(flat, cam: CameraModel, tile: int = TILE_SIZE, near: float = NEAR_PLANE) -> TileBins:
    """render_raster.py:143-182: the reference CSR, bit-exact (mode 0)."""
    _require_pinhole(cam)
    ds = as_device_scene(flat)
    tx, ty = -(-cam.width // tile), -(-cam.height // tile)
    if ds.n == 0:
        return TileBins(tx, ty, tile, np.zeros(tx * ty + 1, np.int64), np.zeros(0, np.int64))
    p = _project(ds, cam, near, tile)
    offsets, entries, _, _ = _bin_sync(ds, cam, near, tile, p, mode=0)
    return TileBins(tx, ty, tile, offsets.cpu().numpy(), entries.cpu().numpy().astype(np.int64))


def render_bins(flat, cam: CameraModel, tile: int = TILE_SIZE, near: float = NEAR_PLANE) -> TileBins:
    """The tightened per-tile lists `rasterize` composites (mode 1)."""
    _require_pinhole(cam)
    ds = as_device_scene(flat)
    p = _project(ds, cam, near, tile)
    offsets, entries, _, (tx, ty) = _bin_sync(ds, cam, near, tile, p, mode=1)
    return TileBins(tx, ty, tile, offsets.cpu().numpy(), entries.cpu().numpy().astype(np.int64))


TILE_ORDER = os.environ.get("SALF_TILE_ORDER", "1") == "1"
FWD_TILE_ORDER = TILE_ORDER and os.environ.get("SALF_FWD_TILE_ORDER", "1") == "1"


def _opts(background, near, stop_threshold, tile, exact_color) -> _lib.RasterOptsT:
    o = _lib.RasterOptsT()
    o.background[:] = [float(v) for v in np.asarray(background, np.float64).reshape(3)]
    o.near, o.stop_threshold, o.tile = float(near), float(stop_threshold), int(tile)
    o.exact_color = 1 if exact_color else 0
    return o


def rasterize(flat, cam: CameraModel, *, background=(0.0, 0.0, 0.0), tile: int = TILE_SIZE,
              near: float = NEAR_PLANE, stop_threshold: float = STOP_THRESHOLD,
              max_pairs: int = 4_000_000, exact_color: bool = False,
              return_state: bool = False, events: list | None = None):
    """Per-pixel exact-intersection compositing over depth-sorted tile bins.

    `max_pairs` is accepted for signature compatibility (the reference's host
    batching knob); the GPU path has no pair batching.  `exact_color=True`
    evaluates the colour field in fp64 (parity mode)."""
    del max_pairs
    _require_pinhole(cam)
    if tile < 1 or tile > 16:
        raise ValueError("tile size must be in [1, 16]")
    lib = _lib.load()
    ds = as_device_scene(flat)
    dev = ds.device
    h, w = cam.height, cam.width
    rgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    op = torch.empty((h, w), dtype=torch.float32, device=dev)
    depth = torch.empty((h, w), dtype=torch.float32, device=dev)
    saved = torch.empty((h * w, _lib.SAVED_STRIDE), dtype=torch.float64, device=dev) \
        if return_state else None
    with _lib.nvtx("raster_project"):
        p = _project(ds, cam, near, tile)
    opts = _opts(background, near, stop_threshold, tile, exact_color)
    sc, cs = ds.c_struct(), cam.c_struct(rolling=False)
    for attempt in range(2):
        with _lib.nvtx("raster_bin"):
            offsets, entries, counts, cap, _ = _bin(ds, cam, near, tile, p, mode=1)
        # hit words for the backward (default mode): which list entries each pixel includes
        hitbits = torch.empty(lib.salf_raster_hitbits_words(cap, offsets.numel() - 1), dtype=torch.int32,
                              device=dev) if (return_state and not exact_color) else None
        order = None
        if FWD_TILE_ORDER:  # longest tile lists first (no ragged last wave); the backward reuses the order
            nt = offsets.numel() - 1
            order = torch.empty(nt, dtype=torch.int32, device=dev)
            tws = _WS.get(dev, lib.salf_raster_tile_order_workspace_bytes(nt), slot="tile_order")
            _lib.check(lib.salf_raster_tile_order(offsets.data_ptr(), nt, order.data_ptr(), tws.data_ptr(),
                                                  tws.numel(), _lib.stream_ptr()), "rasterize")
        ev = _timed(events, "raster_composite")
        with _lib.nvtx("raster_composite"):
            _lib.check(lib.salf_raster_composite(_lib.ref(sc), _lib.ref(cs), _lib.ref(opts),
                                                 offsets.data_ptr(), entries.data_ptr(),
                                                 rgb.data_ptr(), op.data_ptr(), depth.data_ptr(),
                                                 _lib.ptr(saved), p["vrange"].data_ptr(), _lib.ptr(order),
                                                 _lib.ptr(hitbits), _lib.stream_ptr()),
                       "rasterize")
        if ev is not None:
            ev[2].record()
        # capacity check after the composite is enqueued: the host waits for the
        # binning only, the GPU keeps compositing
        n_inst = _Counts(counts).n_instances()
        if n_inst <= cap:
            break
        if events is not None:
            events.pop()
        _grow(dev, 1, n_inst)
    else:
        raise RuntimeError("raster binning failed to size its instance capacity")
    fb = Framebuffer(rgb, op, depth)
    if return_state:
        st = RasterState(ds, cam, opts, offsets, entries[:n_inst], saved, n_inst, p["vrange"], hitbits=hitbits)
        if order is not None:
            st.tile_order = order
        return fb, st
    return fb


def rasterize_scene(scene: Scene, cam: CameraModel, t_stamp: float = 0.0, *,
                    background=(0.0, 0.0, 0.0), tile: int = TILE_SIZE,
                    near: float = NEAR_PLANE) -> Framebuffer:
    """render_raster.py:304-308: the scene flattened at t.  The static set stays
    resident between calls (device.static_device_scene); only the posed actor
    voxels are uploaded (device.composed_device_scene)."""
    from .device import composed_device_scene
    _require_pinhole(cam)
    _lib.load()  # no GPU / library: fail here, before any device allocation (no CPU fallback)
    return rasterize(composed_device_scene(scene, t_stamp), cam, background=background, tile=tile, near=near)


def rasterize_backward(state: RasterState, d_color, d_depth, grad: torch.Tensor | None = None,
                       as_dict: bool = True, events: list | None = None, deterministic: bool = False):
    """Per-voxel gradients of a rasterized frame.

    The reference has no raster backward; the gradient is the one
    `backward_records` (reference backward.py:35-101) assigns to the frame's
    hit pairs taken in tile-list order (DESIGN.md §raster backward).
    d_color (H, W, 3) and d_depth (H, W); returns {param: array} like
    backward_records' 'static' entry, or the raw (M, 27) f64 buffer.
    `d_depth=None`: no depth loss (the kernel drops the depth term; same
    values as zero depth seeds).
    `deterministic=True`: ordered per-voxel reduction instead of atomics,
    bitwise identical across runs."""
    lib = _lib.load()
    ds = state.scene
    dev = ds.device
    h, w = state.cam.height, state.cam.width
    dc = _lib.as_f64(d_color, dev).reshape(h * w * 3)
    dd = _lib.as_f64(d_depth, dev).reshape(h * w) if d_depth is not None else None  # None: no depth loss
    if grad is None:
        grad = torch.zeros((max(ds.n, 1), _lib.GRAD_STRIDE), dtype=torch.float64, device=dev)
    if state.n_instances:
        sc, cs = ds.c_struct(), state.cam.c_struct(rolling=False)
        if TILE_ORDER and state.tile_order is None:
            # longest tile lists first (no ragged last wave); normally the forward computed it already.
            # (With one CTA per tile the forward measured faster row-major; with two half-tile CTAs
            # per tile, heavy-first is 1% faster there too.)
            nt = state.offsets.numel() - 1
            state.tile_order = torch.empty(nt, dtype=torch.int32, device=dev)
            tws = _WS.get(dev, lib.salf_raster_tile_order_workspace_bytes(nt), slot="tile_order")
            _lib.check(lib.salf_raster_tile_order(state.offsets.data_ptr(), nt, state.tile_order.data_ptr(),
                                                  tws.data_ptr(), tws.numel(), _lib.stream_ptr()),
                       "rasterize_backward")
        ev = _timed(events, "raster_backward")
        rng = _lib.nvtx("raster_backward")
        rng.__enter__()
        if deterministic:
            wsb = lib.salf_raster_backward_det_workspace_bytes(state.n_instances, max(ds.n, 1))
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            _lib.check(lib.salf_raster_backward_deterministic(
                _lib.ref(sc), _lib.ref(cs), _lib.ref(state.opts), state.offsets.data_ptr(),
                state.entries.data_ptr(), state.n_instances, state.saved.data_ptr(), dc.data_ptr(), _lib.ptr(dd),
                grad.data_ptr(), _lib.ptr(state.vrange), _lib.ptr(state.tile_order), _lib.ptr(state.hitbits),
                ws.data_ptr(), wsb, _lib.stream_ptr()), "rasterize_backward")
        else:
            _lib.check(lib.salf_raster_backward(_lib.ref(sc), _lib.ref(cs), _lib.ref(state.opts),
                                                state.offsets.data_ptr(), state.entries.data_ptr(),
                                                state.saved.data_ptr(), dc.data_ptr(), _lib.ptr(dd),
                                                grad.data_ptr(), _lib.ptr(state.vrange), _lib.ptr(state.tile_order),
                                                _lib.ptr(state.hitbits), _lib.stream_ptr()), "rasterize_backward")
        rng.__exit__(None, None, None)
        if ev is not None:
            ev[2].record()
    if as_dict:
        return grads_to_dict(grad[: ds.n])
    return grad
