"""Drop-in backend for the reference package (`salf`, reference pkg/src/salf).

`install(salf)` re-binds the reference's hot-path functions -- in every loaded
`salf.*` module that imported them by name -- to libsalf_b200, keeping the
reference's signatures, its own dataclasses (`Framebuffer`, `TileBins`,
`RenderRecords`, `OctreeBuffer`, `SceneOctrees`, `RayBatch`) and NumPy float64
outputs.  The reference's callers then run unchanged on the GPU:
`workflows.render` / `lidar_sweep` / `evaluate_scene`, `trainer.train_loop`,
`bench.run_bench` and the reference's own hot-path tests
(tests/test_dropin_reference.py runs them).  SURVEY §8(b) lists the boundary.

Re-bound (reference file:line of the function replaced):
  render_raster.project_voxels :97, cull_and_bin :143, rasterize :201,
    rasterize_scene :304
  render_ray.build_scene_octrees :44, integrate_rays :161,
    render_rays_image :275, render_lidar_ranges :297
  octree.build_octree :54, query_batch :136, query :169, march_batch :276,
    march :298
  backward.backward_records :35
  sensors.gen_camera_rays :129, camera_rays :185, gen_lidar_rays :193

What stays on the device between calls (the reference rebuilds nothing
either, its arrays are the scene): per voxel set, the geometry (centres,
edges, rotations) and its octree, keyed by the identity of the set's
`level` / `ijk` / `rotation` arrays -- densification (densify.py) builds new
arrays, so a new set is uploaded then.  The field parameters are re-sent on
every call because the reference's optimizer updates them in place
(optim.py:35-62); that is one (M, 28) fp32 copy, not a rebuild.

`RenderRecords` from `integrate_rays` carry every per-segment field the
reference defines (render_ray.py:51-83): the hit lists come from the fp64
marcher (bit-exact), the fields from `salf_shade_segments`, and t_before /
included / the per-ray sums from the reference's own log-space composite
(render_ray.py:86-114) evaluated in fp64 on the device.  The fused kernel's
replay state rides along as `records._b200`, so `backward_records` on those
records runs `salf_ray_backward` (or the actor merge) on the device.

precision="fp64" (default) uses the parity kernels (fp64 colour, reference
operation order); precision="mixed" uses the certified mixed-precision
kernels the benchmarks time."""

from __future__ import annotations

import collections
import sys
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import backward as BW
from . import octree as OT
from . import render_raster as RR
from . import render_ray as RY
from . import sensors as SN
from .device import DeviceScene
from .scene import Actor, FlatVoxels, Scene, SceneBounds, SparseVoxelSet

HOT = {
    "render_raster": ("project_voxels", "cull_and_bin", "rasterize", "rasterize_scene"),
    "render_ray": ("build_scene_octrees", "integrate_rays", "render_rays_image", "render_lidar_ranges"),
    "octree": ("build_octree", "query_batch", "query", "march_batch", "march"),
    "backward": ("backward_records",),
    "sensors": ("gen_camera_rays", "camera_rays", "gen_lidar_rays"),
}

_ALPHA_CLAMP = 1.0 - 1e-12  # scene.py:32


# -- reference objects -> this package's objects (arrays shared, not copied) --

def _bounds(b) -> SceneBounds:
    return SceneBounds(np.asarray(b.aabb_min, np.float64), np.asarray(b.aabb_max, np.float64),
                       float(b.base_edge), int(b.max_levels))


def _vset(v) -> SparseVoxelSet:
    s = SparseVoxelSet(_bounds(v.bounds), getattr(v, "budget", 2_500_000))
    s.level, s.ijk = v.level, v.ijk
    s.w_s, s.w_c, s.w_sh, s.log_a, s.log_b = v.w_s, v.w_c, v.w_sh, v.log_a, v.log_b
    s.rotation = v.rotation
    return s


def _camera(cam) -> SN.CameraModel:
    return SN.CameraModel(kind=cam.kind, width=int(cam.width), height=int(cam.height), fx=float(cam.fx),
                          fy=float(cam.fy), cx=float(cam.cx), cy=float(cam.cy),
                          distortion=tuple(float(k) for k in cam.distortion), position=cam.position,
                          quaternion=cam.quaternion, readout_duration=float(cam.readout_duration),
                          linear_velocity=cam.linear_velocity, angular_velocity=cam.angular_velocity)


def _lidar(lid) -> SN.LidarModel:
    return SN.LidarModel(beam_elevations=np.asarray(lid.beam_elevations, np.float64),
                         azimuth_start=float(lid.azimuth_start), azimuth_end=float(lid.azimuth_end),
                         steps=int(lid.steps), scan_period=float(lid.scan_period), position=lid.position,
                         quaternion=lid.quaternion, linear_velocity=lid.linear_velocity,
                         angular_velocity=lid.angular_velocity)


def _flat(flat) -> FlatVoxels:
    return FlatVoxels(flat.centers, flat.edges, flat.rotations, flat.w_s, flat.w_c, flat.w_sh, flat.log_a,
                      flat.log_b, flat.density_mode)


def _np(t) -> np.ndarray:
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@dataclass
class _SetEntry:
    keep: tuple  # the arrays whose identity keys this entry (kept alive so ids stay unique)
    ds: DeviceScene
    tree: OT.OctreeBuffer | None = None


class Backend:
    """The GPU implementation behind the reference's API (see the module docstring)."""

    def __init__(self, salf=None, precision: str = "fp64", device=None):
        if precision not in ("fp64", "mixed"):
            raise ValueError("precision must be 'fp64' or 'mixed'")
        if salf is None:
            import salf  # noqa: F811  (the reference package)
        self.salf = salf
        self.exact = precision == "fp64"
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        _lib.load()  # fail loudly without the CUDA library / a GPU: there is no CPU fallback
        self._sets: dict = {}
        self._flats: dict = {}
        self.orig: dict = {}
        self.calls = collections.Counter()  # re-bound calls served (tests check the backend ran)
        self._mods = {name: sys.modules[f"{salf.__name__}.{name}"] for name in HOT
                      if f"{salf.__name__}.{name}" in sys.modules or self._import(name)}

    def _import(self, name):
        __import__(f"{self.salf.__name__}.{name}")
        return True

    # -- device-resident voxel sets ------------------------------------------

    def _set_entry(self, v, density_mode: str) -> _SetEntry:
        """Geometry + octree of a reference SparseVoxelSet, uploaded once; the
        parameters refreshed from the (possibly updated) host arrays."""
        key = (id(v.level), id(v.ijk), id(v.rotation), density_mode)
        e = self._sets.get(key)
        if e is None:
            ours = _vset(v)
            flat = FlatVoxels(ours.centers(), ours.edges(), ours.rotation, ours.w_s, ours.w_c, ours.w_sh,
                              ours.log_a, ours.log_b, density_mode)
            e = _SetEntry((v.level, v.ijk, v.rotation), DeviceScene(flat, self.device))
            if len(self._sets) >= 8:  # oldest first: densification retires whole sets
                self._sets.pop(next(iter(self._sets)))
            self._sets[key] = e
        else:
            e.ds.set_params(v.w_s, v.w_c, v.w_sh, v.log_a, v.log_b)
        return e

    def _tree(self, v, density_mode: str = "sdf") -> OT.OctreeBuffer:
        e = self._set_entry(v, density_mode)
        if e.tree is None:
            e.tree = OT.build_octree(_vset(v), device=self.device)
        return e.tree

    def _scene(self, scene) -> Scene:
        """This package's Scene over the reference scene's arrays, with the static
        set's cached DeviceScene attached (render_ray._static_device_scene)."""
        static = _vset(scene.static)
        actors = [Actor(a.actor_id, a.extents, _vset(a.voxels), a.times, a.positions, a.quaternions)
                  for a in scene.actors]
        ours = Scene(bounds=_bounds(scene.bounds), static=static, actors=actors,
                     density_mode=scene.density_mode, inner_aabb=getattr(scene, "inner_aabb", None))
        ours._b200_static = self._set_entry(scene.static, scene.density_mode).ds
        return ours

    def _flat_ds(self, flat) -> DeviceScene:
        key = id(flat)
        e = self._flats.get(key)
        if e is None or e.keep[0] is not flat:
            e = _SetEntry((flat,), DeviceScene(_flat(flat), self.device))
            if len(self._flats) > 4:
                self._flats.pop(next(iter(self._flats)))
            self._flats[key] = e
        return e.ds

    # -- render_raster --------------------------------------------------------

    def project_voxels(self, flat, cam, near=RR.NEAR_PLANE):
        self.salf.render_raster._require_pinhole(cam)
        return RR.project_voxels(self._flat_ds(flat), _camera(cam), near)

    def cull_and_bin(self, flat, cam, tile=RR.TILE_SIZE, near=RR.NEAR_PLANE):
        self.salf.render_raster._require_pinhole(cam)
        b = RR.cull_and_bin(self._flat_ds(flat), _camera(cam), tile, near)
        return self.salf.render_raster.TileBins(tiles_x=b.tiles_x, tiles_y=b.tiles_y, tile=b.tile,
                                                offsets=b.offsets.astype(np.int64),
                                                entries=b.entries.astype(np.int64))

    def _raster(self, ds, cam, background, **kw):
        """RR.rasterize -> the reference Framebuffer.  fp64 mode finalises the
        pixels from the kernel's fp64 accumulators (render_raster.py:295-301)
        instead of the fp32 image planes."""
        cm = _camera(cam)
        if not self.exact:
            fb = RR.rasterize(ds, cm, background=background, **kw)
            return self.salf.render_raster.Framebuffer(color=_np(fb.color).astype(np.float64),
                                                       opacity=_np(fb.opacity).astype(np.float64),
                                                       depth=_np(fb.depth).astype(np.float64))
        fb, st = RR.rasterize(ds, cm, background=background, exact_color=True, return_state=True, **kw)
        sv = st.saved.view(cm.height, cm.width, _lib.SAVED_STRIDE)
        bg = torch.as_tensor(np.asarray(background, np.float64).reshape(3), device=sv.device)
        T = sv[..., 5]
        acc_w, acc_wt = sv[..., 3], sv[..., 4]
        ok = acc_w > RY.DEPTH_WEIGHT_MIN
        depth = torch.where(ok, acc_wt / torch.where(ok, acc_w, torch.ones_like(acc_w)),
                            torch.full_like(acc_w, float("nan")))
        return self.salf.render_raster.Framebuffer(color=_np(sv[..., 0:3] + T[..., None] * bg),
                                                   opacity=_np(1.0 - T), depth=_np(depth))

    def rasterize(self, flat, cam, *, background=(0.0, 0.0, 0.0), tile=RR.TILE_SIZE, near=RR.NEAR_PLANE,
                  stop_threshold=RR.STOP_THRESHOLD, max_pairs=4_000_000):
        self.salf.render_raster._require_pinhole(cam)
        return self._raster(self._flat_ds(flat), cam, background, tile=tile, near=near,
                            stop_threshold=stop_threshold, max_pairs=max_pairs)

    def rasterize_scene(self, scene, cam, t_stamp=0.0, *, background=(0.0, 0.0, 0.0), tile=RR.TILE_SIZE,
                        near=RR.NEAR_PLANE):
        self.salf.render_raster._require_pinhole(cam)
        if any(a.voxels.n for a in scene.actors):  # actors move with t: flatten like the reference
            ds = DeviceScene(_flat(self.salf.render_raster.flatten_scene(scene, t_stamp)), self.device)
        else:
            ds = self._set_entry(scene.static, scene.density_mode).ds
        return self._raster(ds, cam, background, tile=tile, near=near)

    # -- octree -----------------------------------------------------------------

    def _ref_buffer(self, tree: OT.OctreeBuffer):
        out = self.salf.octree.OctreeBuffer(nodes_id=tree.nodes_id.astype(np.int64),
                                            nodes_leaf=tree.nodes_leaf.astype(np.int8),
                                            root_min=np.asarray(tree.root_min, np.float64).copy(),
                                            root_edge=float(tree.root_edge), max_depth=int(tree.max_depth))
        out._b200 = tree
        return out

    def _our_tree(self, buf) -> OT.OctreeBuffer:
        t = getattr(buf, "_b200", None)
        if t is not None:
            return t
        ids = np.asarray(buf.nodes_id, np.int64)
        leaf = np.asarray(buf.nodes_leaf)
        words = np.where(leaf == 0, ids, np.where(leaf == 1, -ids - 2, -1)).astype(np.int32)
        t = OT.OctreeBuffer(torch.as_tensor(words, device=self.device), np.asarray(buf.root_min, np.float64),
                            float(buf.root_edge), int(buf.max_depth))
        buf._b200 = t
        return t

    def build_octree(self, voxels, bounds=None):
        if bounds is not None and bounds is not voxels.bounds:
            return self._ref_buffer(OT.build_octree(_vset(voxels), _bounds(bounds), device=self.device))
        return self._ref_buffer(self._tree(voxels))

    def query_batch(self, buffer, p):
        return OT.query_batch(self._our_tree(buffer), p)

    def query(self, buffer, p):
        return int(self.query_batch(buffer, np.asarray(p, np.float64)[None, :])[1][0])

    def march_batch(self, buffer, origins, dirs, t_max=np.inf):
        return OT.march_batch(self._our_tree(buffer), origins, dirs, t_max)

    def march(self, buffer, origin, direction, t_max=np.inf):
        return OT.march(self._our_tree(buffer), origin, direction, t_max)

    # -- render_ray -------------------------------------------------------------

    def build_scene_octrees(self, scene):
        static = self._ref_buffer(self._tree(scene.static, scene.density_mode))
        actors = [self._ref_buffer(self._tree(a.voxels, scene.density_mode)) for a in scene.actors]
        return self.salf.render_ray.SceneOctrees(static=static, actors=actors)

    def _octrees(self, scene, octrees) -> RY.SceneOctrees:
        trees, dss = [], []
        for a, buf in zip(scene.actors, getattr(octrees, "actors", [])):
            if a.voxels.n:
                trees.append(self._our_tree(buf))
                dss.append(self._set_entry(a.voxels, scene.density_mode).ds)
            else:
                trees.append(None)
                dss.append(None)
        static = octrees.static if hasattr(octrees, "static") else octrees
        return RY.SceneOctrees(static=self._our_tree(static), actors=trees, actor_scenes=dss)

    def integrate_rays(self, scene, octrees, origins, dirs, t_stamps=None, *, t_max=np.inf,
                       background=(0.0, 0.0, 0.0), stop_threshold=RY.STOP_THRESHOLD):
        """render_ray.py:161-239, the full RenderRecords (module docstring)."""
        lib = _lib.load()
        origins = np.atleast_2d(np.asarray(origins, np.float64))
        dirs = np.atleast_2d(np.asarray(dirs, np.float64))
        n = origins.shape[0]
        ts = np.zeros(n) if t_stamps is None else np.broadcast_to(np.asarray(t_stamps, np.float64), (n,))
        bg = np.asarray(background, np.float64)
        ours = self._scene(scene)
        octs = self._octrees(scene, octrees)
        dev = self.device
        o = torch.as_tensor(origins, device=dev)
        d = torch.as_tensor(dirs, device=dev)
        finite = bool(np.any(np.isfinite(np.asarray(t_max, np.float64))))
        # the fused kernel (and the device backward) cover the renderers' t_max = inf; a finite
        # t_max gets the full records only, and backward_records then runs the reference's
        fused = None if finite else RY.integrate_rays(ours, octs, o, d, ts, background=bg,
                                                      stop_threshold=stop_threshold, exact_color=self.exact)
        live = any(a.voxels.n for a in ours.actors)
        if finite and live:
            raise NotImplementedError("finite t_max with live actors")
        ds = ours._b200_static
        # per-segment records: the static hit lists (reference early stop only without actors)
        ray, vid, t0, t1 = OT.march_segments(octs.static, o, d, t_max, ds, stop_threshold, not live)
        recs, rays = [], []
        if ray.numel():
            rec = torch.empty((ray.numel(), 24), dtype=torch.float64, device=dev)
            # (the gathered inputs are named: a temporary's memory could be reused before the launch reads it)
            so, sd = o[ray].contiguous(), d[ray].contiguous()
            sv, s0, s1 = vid.contiguous(), t0.contiguous(), t1.contiguous()
            _lib.check(lib.salf_shade_segments(_lib.ref(ds.c_struct()), ray.numel(), so.data_ptr(), sd.data_ptr(),
                                               sv.data_ptr(), s0.data_ptr(), s1.data_ptr(), -1, 0,
                                               int(self.exact), rec.data_ptr(), _lib.stream_ptr()),
                       "integrate_rays")
            recs.append(rec)
            rays.append(ray)
        offs = {}
        if live:
            start, ex_rec, offsets, _ = RY._actor_segments(ours, octs, o, d, ts, dev, self.exact)
            cnt = start[1:] - start[:-1]
            if int(start[-1]):
                recs.append(ex_rec[: int(start[-1])])
                rays.append(torch.repeat_interleave(torch.arange(n, device=dev), cnt))
            offs = {ai: goff for ai, (_, goff, _) in enumerate(offsets)}
        return self._records(recs, rays, n, bg, stop_threshold, ours.density_mode, offs, fused)

    def _records(self, recs, rays, n, bg, stop_threshold, density_mode, offs, fused):
        dev = self.device
        if recs:
            rec = torch.cat(recs)
            ray = torch.cat(rays)
            order = torch.arange(ray.numel(), device=dev)
            for key in (rec[:, 21], rec[:, 20], rec[:, 0], ray.double()):  # lexsort((vid, owner, t0, ray)) :210
                order = order[torch.sort(key[order], stable=True).indices]
            rec, ray = rec[order], ray[order]
        else:
            rec = torch.zeros((0, 24), dtype=torch.float64, device=dev)
            ray = torch.zeros(0, dtype=torch.int64, device=dev)
        owner = rec[:, 20].to(torch.int32)
        gvid = rec[:, 21].to(torch.int64)
        vid = gvid.clone()
        for ai, goff in offs.items():  # actor records carry global ids: back to per-owner indices
            sel = owner == ai
            vid[sel] -= goff
        t0, t1 = rec[:, 0], rec[:, 1]
        alpha, color = rec[:, 10], rec[:, 12:15]
        # the reference's composite (render_ray.py:86-114), fp64
        a = alpha.clamp(0.0, _ALPHA_CLAMP)
        s = torch.log1p(-a)
        csum = torch.cumsum(s, 0)
        counts = torch.bincount(ray, minlength=n) if ray.numel() else torch.zeros(n, dtype=torch.int64, device=dev)
        starts = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        starts[1:] = torch.cumsum(counts, 0)
        prefix = torch.cat([torch.zeros(1, dtype=torch.float64, device=dev), csum])
        base = torch.repeat_interleave(prefix[starts[:-1]], counts)
        t_before = torch.exp((csum - s) - base)
        included = t_before > 1.0 - stop_threshold
        w = torch.where(included, t_before * a, torch.zeros_like(a))
        t_mid = 0.5 * (t0 + t1)
        out_color = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        out_color.index_add_(0, ray, w[:, None] * color)
        log_tf = torch.zeros(n, dtype=torch.float64, device=dev).index_add_(
            0, ray, torch.where(included, s, torch.zeros_like(s)))
        t_final = torch.exp(log_tf)
        out_color += t_final[:, None] * torch.as_tensor(bg, device=dev)
        wsum = torch.zeros(n, dtype=torch.float64, device=dev).index_add_(0, ray, w)
        dnum = torch.zeros(n, dtype=torch.float64, device=dev).index_add_(0, ray, w * t_mid)
        depth = torch.where(wsum > RY.DEPTH_WEIGHT_MIN, dnum / torch.where(wsum > 0, wsum, torch.ones_like(wsum)),
                            torch.full_like(wsum, float("nan")))
        R = self.salf.render_ray.RenderRecords
        out = R(n_rays=n, ray=_np(ray), owner=_np(owner), vid=_np(vid), t0=_np(t0), t1=_np(t1),
                x=_np(rec[:, 4:7]), omega=_np(rec[:, 17:20]), s_field=_np(rec[:, 7]), sigma=_np(rec[:, 9]),
                alpha=_np(alpha), color=_np(color), t_before=_np(t_before), included=_np(included),
                out_color=_np(out_color), opacity=_np(1.0 - t_final), depth=_np(depth), weight_sum=_np(wsum),
                t_final=_np(t_final), background=bg, density_mode=density_mode, group_start=_np(starts))
        if fused is not None:
            out._b200 = fused
        return out

    def _batch(self, batch) -> SN.RayBatch:
        dev = self.device
        return SN.RayBatch(torch.as_tensor(np.asarray(batch.origins, np.float64), device=dev),
                           torch.as_tensor(np.asarray(batch.dirs, np.float64), device=dev),
                           torch.as_tensor(np.asarray(batch.t_stamps, np.float64), device=dev),
                           torch.as_tensor(np.asarray(batch.keys, np.int64), device=dev),
                           torch.as_tensor(np.asarray(batch.valid, bool), device=dev), tuple(batch.shape))

    def _fused64(self, scene, octrees, o, d, ts, background, stop_threshold):
        """fp64 per-ray outputs of the fused kernel, finalised from its fp64
        accumulators like the reference's _composite (render_ray.py:106-113)."""
        rec = RY.integrate_rays(self._scene(scene), self._octrees(scene, octrees),
                                torch.as_tensor(np.asarray(o, np.float64), device=self.device),
                                torch.as_tensor(np.asarray(d, np.float64), device=self.device),
                                np.asarray(ts, np.float64), background=background, stop_threshold=stop_threshold,
                                exact_color=True)
        sv = rec.saved
        T = sv[:, 5]
        bg = torch.as_tensor(np.asarray(background, np.float64).reshape(3), device=sv.device)
        ok = sv[:, 3] > RY.DEPTH_WEIGHT_MIN
        depth = torch.where(ok, sv[:, 4] / torch.where(ok, sv[:, 3], torch.ones_like(T)),
                            torch.full_like(T, float("nan")))
        return _np(sv[:, 0:3] + T[:, None] * bg), _np(1.0 - T), _np(depth)

    def render_rays_image(self, scene, octrees, batch, *, background=(0.0, 0.0, 0.0), chunk=65536,
                          stop_threshold=RY.STOP_THRESHOLD):
        if self.exact:  # render_ray.py:275-294 on the fp64 accumulators
            h, w = batch.shape
            color = np.zeros((h * w, 3))
            color[:] = np.asarray(background, np.float64)
            opacity = np.zeros(h * w)
            depth = np.full(h * w, np.nan)
            sel = np.flatnonzero(batch.valid)
            if sel.size:
                c, op, dp = self._fused64(scene, octrees, batch.origins[sel], batch.dirs[sel],
                                          batch.t_stamps[sel], background, stop_threshold)
                flat = batch.keys[sel, 0] * w + batch.keys[sel, 1]
                color[flat], opacity[flat], depth[flat] = c, op, dp
            return color.reshape(h, w, 3), opacity.reshape(h, w), depth.reshape(h, w)
        c, op, dp = RY.render_rays_image(self._scene(scene), self._octrees(scene, octrees), self._batch(batch),
                                         background=background, chunk=chunk, stop_threshold=stop_threshold)
        return _np(c).astype(np.float64), _np(op).astype(np.float64), _np(dp).astype(np.float64)

    def render_lidar_ranges(self, scene, octrees, batch, *, chunk=65536):
        if self.exact or any(a.voxels.n for a in scene.actors):  # the fused LiDAR kernel is fp32, static-only
            _, _, dp = self._fused64(scene, octrees, batch.origins, batch.dirs, batch.t_stamps, (0.0, 0.0, 0.0),
                                     RY.STOP_THRESHOLD)
            return dp.reshape(batch.shape)
        return _np(RY.render_lidar_ranges(self._scene(scene), self._octrees(scene, octrees), self._batch(batch),
                                          chunk=chunk)).astype(np.float64)

    # -- backward ---------------------------------------------------------------

    def backward_records(self, records, scene, d_color, d_depth):
        fused = getattr(records, "_b200", None)
        if fused is None:  # records this backend did not produce: the reference's own function
            return self.orig["backward"]["backward_records"](records, scene, d_color, d_depth)
        g = BW.backward_records(fused, self._scene(scene), np.asarray(d_color, np.float64),
                                np.asarray(d_depth, np.float64))
        return {k: {p: np.asarray(v, np.float64) for p, v in gd.items()} for k, gd in g.items()}

    # -- sensors ----------------------------------------------------------------

    def _ref_batch(self, b):
        return self.salf.sensors.RayBatch(origins=_np(b.origins).astype(np.float64),
                                          dirs=_np(b.dirs).astype(np.float64),
                                          t_stamps=_np(b.t_stamps).astype(np.float64),
                                          keys=_np(b.keys).astype(np.int64), valid=_np(b.valid).astype(bool),
                                          shape=tuple(b.shape))

    def gen_camera_rays(self, cam, t0=0.0):
        return self._ref_batch(SN.gen_camera_rays(_camera(cam), t0, device=self.device))

    def camera_rays(self, cam, t0=0.0):
        return self._ref_batch(SN.camera_rays(_camera(cam), t0, device=self.device))

    def gen_lidar_rays(self, lidar, t0=0.0):
        return self._ref_batch(SN.gen_lidar_rays(_lidar(lidar), t0, device=self.device))

    # -- (un)installation ---------------------------------------------------------

    def _wrapped(self, name):
        fn = getattr(self, name)

        def call(*args, **kwargs):
            self.calls[name] += 1
            return fn(*args, **kwargs)

        call.__name__ = call.__qualname__ = name
        call.__doc__ = fn.__doc__
        call._b200_backend = self
        return call

    def install(self) -> "Backend":
        pkg = self.salf.__name__
        for mod_name, names in HOT.items():
            mod = self._mods[mod_name]
            self.orig[mod_name] = {n: getattr(mod, n) for n in names}
        wrappers = {n: self._wrapped(n) for names in HOT.values() for n in names}
        for mname, m in list(sys.modules.items()):
            if m is None or not (mname == pkg or mname.startswith(pkg + ".")):
                continue
            for mod_name, names in HOT.items():
                for n in names:
                    if getattr(m, n, None) is self.orig[mod_name][n]:
                        setattr(m, n, wrappers[n])
        return self

    def uninstall(self) -> None:
        pkg = self.salf.__name__
        for mname, m in list(sys.modules.items()):
            if m is None or not (mname == pkg or mname.startswith(pkg + ".")):
                continue
            for mod_name, names in HOT.items():
                for n in names:
                    if getattr(getattr(m, n, None), "_b200_backend", None) is self:
                        setattr(m, n, self.orig[mod_name][n])


def install(salf=None, precision: str = "fp64", device=None) -> Backend:
    """Route the reference package's hot path through libsalf_b200 (module docstring).
    Import every salf module whose names should be re-bound before calling this
    (modules imported later bind the re-bound functions anyway)."""
    if salf is None:
        import salf  # noqa: F811
    for sub in ("render_raster", "render_ray", "octree", "backward", "sensors", "losses", "trainer",
                "workflows", "bench", "densify"):
        try:
            __import__(f"{salf.__name__}.{sub}")
        except ImportError:
            pass
    return Backend(salf, precision, device).install()
