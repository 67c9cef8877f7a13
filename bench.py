"""Benchmark of the SaLF render hot path (BASELINE.json metric: camera FPS at
1920x1080 and LiDAR rays/s at 1/2/4/8 B200 vs the CPU reference).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (`value`, N = 1): C2 -- one 1920x1080 pinhole camera rasterized
forward + backward (colour L1 loss) on the 1M-voxel synthetic scene S1M
(BASELINE.json configs[1]).  N > 1 runs under torchrun, one rank per GPU:
rank r renders camera r of the C5 rig (8 C2-style cameras at yaw 45 deg x r,
distinct views), forward + backward, and the per-voxel gradient buffer is
all-reduced over NCCL (weak scaling: `value` = all ranks' frames/s).  Beside
it, at every N:

* `c5`: the C5 training step (8 cameras + 2 LiDARs, BASELINE configs[4])
  SHARDED over the N ranks by parallel.split_work/assign (row bands, ray
  blocks), global L1 seeds, backward, NCCL gradient all-reduce, device Adam
  (strong scaling: steps/s of the whole rig);
* `lidar`: one C3 sweep per rank (configs[2]), rays/s, with its HBM roofline;

and on rank 0 at N = 1: the C1 frame (configs[0]) on the GPU next to the
reference algorithm over the whole frame on the host cores (not
extrapolated), the C3 sweep on the host cores (whole sweep), the C2 CPU
baseline (sampled tiles, extrapolated, labelled), the surface regime and
C4.  `--impl reference` times the reference on the host cores on the same C2
workload: the UNMODIFIED reference package installed in baseline/_ref
(tools/install_reference.sh; it travels to the GPU box), kind "reference"; if
it is missing, the oracle port (oracle/salf_oracle.py), kind "port".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "camera FPS @1920x1080 (raster fwd+bwd, S1M) and LiDAR rays/s (128-beam)"
UNIT = "frames/s"
WORKLOAD = "C2: S1M init-regime scene (1,023,816 voxels), 1920x1080 pinhole raster forward+backward"


def config_dict(regime: str, world: int, extra: dict | None = None) -> dict:
    """The workload description both arms print (same keys, same values)."""
    c = {"workload": WORKLOAD, "regime": regime, "resolution": [1920, 1080], "voxels": 1023816,
         "loss": "colour L1 (losses.py:22-31), no depth seeds",
         "multi_gpu": "rank r renders C5-rig camera r (yaw 45 deg x r), fwd+bwd, NCCL grad all-reduce"
                      if world > 1 else "single GPU",
         "l2": "flushed (256 MB write) between timed steps"}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------------------
# CPU baselines: the reference algorithm (oracle port) on the host cores.
# Workers are spawned with OMP_NUM_THREADS=1; frame-level
# work (projection, pixel rays, octree) is done once per worker at start-up.

_W = {}
REF_PKG = ROOT / "baseline" / "_ref"  # the UNMODIFIED reference (tools/install_reference.sh); travels to the box


def ref_available() -> bool:
    return (REF_PKG / "salf" / "render_raster.py").is_file()


def _ref_scene(sc):
    """The reference's Scene over this package's scene arrays (no copies)."""
    import salf.scene as RS
    b = RS.SceneBounds(sc.bounds.aabb_min, sc.bounds.aabb_max, sc.bounds.base_edge, sc.bounds.max_levels)
    v = RS.SparseVoxelSet(b, budget=max(sc.static.n + 10, 10))
    src = sc.static
    v.level, v.ijk, v.w_s, v.w_c, v.w_sh = src.level, src.ijk, src.w_s, src.w_c, src.w_sh
    v.log_a, v.log_b, v.rotation = src.log_a, src.log_b, src.rotation
    return RS.Scene(bounds=b, static=v, density_mode=sc.density_mode)


def _ref_cam(c):
    import salf.sensors as RS
    return RS.CameraModel(kind=c.kind, width=c.width, height=c.height, fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy,
                          position=c.position, quaternion=c.quaternion)


def _cpu_init_ref(kind, regime):
    """Worker state for the REFERENCE package's own functions (kind "reference")."""
    sys.path.insert(0, str(REF_PKG))
    import salf.render_raster as RR
    import salf.render_ray as RY
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200.scenes import get_scene
    name = {"c1": "S20k", "c2": "S1M", "c3": "S1M"}[kind]
    sc = _ref_scene(get_scene(name, regime if kind != "c1" else "init"))
    _W.update(ref=True, scene=sc)
    if kind in ("c1", "c2"):
        _W["cam"] = _ref_cam(configs.c1_camera() if kind == "c1" else configs.c2_camera())
        _W["flat"] = RR.flatten_scene(sc)
        if kind == "c2":  # tile membership once per worker (render_raster.py:97-176 on the whole frame)
            rmin, rmax, _, culled = RR.project_voxels(_W["flat"], _W["cam"])
            with np.errstate(invalid="ignore"):
                u0 = np.maximum(np.ceil(rmin[:, 0] - 0.5), 0.0)
                u1 = np.minimum(np.floor(rmax[:, 0] - 0.5), _W["cam"].width - 1)
                v0 = np.maximum(np.ceil(rmin[:, 1] - 0.5), 0.0)
                v1 = np.minimum(np.floor(rmax[:, 1] - 0.5), _W["cam"].height - 1)
            ok = ~culled & (u0 <= u1) & (v0 <= v1)
            _W["span"] = (np.where(ok, u0 // 16, 1), np.where(ok, v0 // 16, 1), np.where(ok, u1 // 16, 0),
                          np.where(ok, v1 // 16, 0))
    else:
        _W["oct"] = RY.build_scene_octrees(sc)
        lid = configs.c3_lidar()
        import salf.sensors as RSn
        b = RSn.gen_lidar_rays(RSn.LidarModel(beam_elevations=lid.beam_elevations, azimuth_start=lid.azimuth_start,
                                              azimuth_end=lid.azimuth_end, steps=lid.steps,
                                              scan_period=lid.scan_period, position=lid.position,
                                              quaternion=lid.quaternion, linear_velocity=lid.linear_velocity,
                                              angular_velocity=lid.angular_velocity))
        _W["o"], _W["d"], _W["t"] = b.origins, b.dirs, b.t_stamps


def _ref_c2_tiles(tiles):
    """The reference on one 16x16 C2 tile, forward AND backward: `rasterize`
    (render_raster.py:201-301) of the tile (camera principal point shifted, the
    voxels whose span covers the tile), then the raster gradient as SURVEY §8c
    defines it -- the tile's hit pairs from the reference's `_pair_fields`
    and field evaluators, `_composite` (render_ray.py:86-114) and
    `backward_records` (backward.py:35-101).  Returns seconds."""
    import dataclasses
    from types import SimpleNamespace
    import salf.backward as RB
    import salf.render_raster as RR
    import salf.render_ray as RY
    import salf.scene as RS
    flat, cam = _W["flat"], _W["cam"]
    total = 0.0
    for t in tiles:
        tx, ty = t % 120, t // 120
        sx0, sy0, sx1, sy1 = _W["span"]
        sel = np.flatnonzero((sx0 <= tx) & (tx <= sx1) & (sy0 <= ty) & (ty <= sy1))
        sub = RR.FlatVoxels(centers=flat.centers[sel], edges=flat.edges[sel], rotations=flat.rotations[sel],
                            w_s=flat.w_s[sel], w_c=flat.w_c[sel], w_sh=flat.w_sh[sel], log_a=flat.log_a[sel],
                            log_b=flat.log_b[sel], density_mode=flat.density_mode)
        tcam = dataclasses.replace(cam, width=16, height=16, cx=cam.cx - 16 * tx, cy=cam.cy - 16 * ty)
        t0 = time.perf_counter()
        RR.rasterize(sub, tcam)
        bins = RR.cull_and_bin(sub, tcam)
        ent = bins.entries[bins.offsets[0]:bins.offsets[1]]
        dirs = RR.gen_camera_rays(tcam).dirs
        t_near = RR.NEAR_PLANE / (dirs @ tcam.rotation_matrix())[:, 2]
        pp, vv = np.repeat(np.arange(256), ent.size), np.tile(ent, 256)
        with np.errstate(over="ignore", invalid="ignore"):
            o, d, t_in, t_out = RR._pair_fields(sub, np.broadcast_to(tcam.position, (pp.size, 3)), dirs[pp], vv)
            t0p = np.maximum(np.maximum(t_in, t_near[pp]), 0.0)
            hit = t_out > t0p + 1e-12
            pp, vv, o, d, t0p, t1p = pp[hit], vv[hit], o[hit], d[hit], t0p[hit], t_out[hit]
            tm = 0.5 * (t0p + t1p)
            x = (o + tm[:, None] * d) / (0.5 * sub.edges[vv])[:, None]
            s_f = RS.eval_sdf(x, sub.w_s[vv])
            sig = RS.sdf_to_density(s_f, np.exp(sub.log_a[vv]), np.exp(sub.log_b[vv]))
            alpha = RS.segment_opacity(sig, t1p - t0p)
            color = RS.eval_color(x, d, sub.w_c[vv], sub.w_sh[vv])
        bg = np.zeros(3)
        (tb, inc, _w, oc, op, dep, ws, tf, gs) = RY._composite(pp, alpha, color, tm, 256, bg, RR.STOP_THRESHOLD)
        rec = RY.RenderRecords(n_rays=256, ray=pp, owner=np.full(pp.size, -1, np.int32), vid=vv, t0=t0p, t1=t1p,
                               x=x, omega=d, s_field=s_f, sigma=sig, alpha=alpha, color=color, t_before=tb,
                               included=inc, out_color=oc, opacity=op, depth=dep, weight_sum=ws, t_final=tf,
                               background=bg, density_mode=sub.density_mode, group_start=gs)
        static = SimpleNamespace(w_s=sub.w_s, w_c=sub.w_c, w_sh=sub.w_sh, log_a=sub.log_a, log_b=sub.log_b)
        RB.backward_records(rec, SimpleNamespace(static=static, actors=[], density_mode=sub.density_mode),
                            np.full((256, 3), 1e-6), np.zeros(256))
        total += time.perf_counter() - t0
    return total


def _ref_c1_band(rows):
    """The reference's rasterize of tile rows [r0, r1) of the C1 frame (a band camera)."""
    import dataclasses
    import salf.render_raster as RR
    cam = _W["cam"]
    r0, r1 = rows
    band = dataclasses.replace(cam, height=16 * (r1 - r0), cy=cam.cy - 16 * r0)
    t0 = time.perf_counter()
    fb = RR.rasterize(_W["flat"], band)
    return time.perf_counter() - t0, fb.color


def _ref_c3_block(lohi):
    """The reference's integrate_rays depth (render_lidar_ranges' body, render_ray.py:297-306) of a ray block."""
    import salf.render_ray as RY
    lo, hi = lohi
    t0 = time.perf_counter()
    rec = RY.integrate_rays(_W["scene"], _W["oct"], _W["o"][lo:hi], _W["d"][lo:hi], _W["t"][lo:hi])
    return time.perf_counter() - t0, rec.depth


def _pin_threads():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def _cpu_init(kind, regime):
    from oracle import salf_oracle as O
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200.scenes import get_scene
    name = {"c1": "S20k", "c2": "S1M", "c3": "S1M"}[kind]
    sc = get_scene(name, regime if kind != "c1" else "init")
    b, v = sc.bounds, sc.static
    vox = O.Voxels.from_grid(b.aabb_min, b.aabb_max, b.base_edge, v.level, v.ijk, v.w_s, v.w_c,
                             v.w_sh, v.log_a, v.log_b)
    _W["vox"] = vox
    if kind in ("c1", "c2"):
        c = configs.c1_camera() if kind == "c1" else configs.c2_camera()
        cam = O.Camera("pinhole", c.width, c.height, c.fx, c.fy, c.cx, c.cy, position=c.position,
                       quaternion=c.quaternion)
        _W["cam"] = cam
        _W["proj"] = O.project_voxels(vox, cam)
        _W["rays"] = O.pixel_rays(cam)
    else:
        _W["tree"] = O.build_octree(vox)
        lid = configs.c3_lidar()
        r = O.lidar_rays(O.Lidar(lid.beam_elevations, lid.azimuth_start, lid.azimuth_end, lid.steps,
                                 lid.scan_period, lid.position, lid.quaternion, lid.linear_velocity,
                                 lid.angular_velocity))
        _W["o"], _W["d"] = r["origins"], r["dirs"]


def _cpu_ready(_):
    return "vox" in _W


def _c2_tiles(tiles):
    """Reference fwd + bwd (raster records -> composite -> backward_records) of
    the given 16x16 tiles of the C2 frame; returns seconds (projection excluded:
    once per worker, like a row-band worker of the reference)."""
    from oracle import salf_oracle as O
    vox, cam = _W["vox"], _W["cam"]
    t0 = time.perf_counter()
    rec = O.raster_records(vox, cam, tiles=tiles, proj=_W["proj"], pix_rays=_W["rays"])
    dc = np.full((rec["n_rays"], 3), 1e-6)
    O.backward_records(rec, vox, dc, np.zeros(rec["n_rays"]))
    return time.perf_counter() - t0


def _c1_band(rows):
    """Reference rasterize (render_raster.py:201-301) of tile rows [r0, r1) of the C1 frame."""
    from oracle import salf_oracle as O
    t0 = time.perf_counter()
    fb = O.rasterize(_W["vox"], _W["cam"], rows=rows, proj=_W["proj"], pix_rays=_W["rays"])
    return time.perf_counter() - t0, fb["color"][rows[0] * 16:rows[1] * 16]


def _c3_block(lohi):
    """Reference render_lidar_ranges (render_ray.py:297-306) of a block of the C3 sweep."""
    from oracle import salf_oracle as O
    lo, hi = lohi
    t0 = time.perf_counter()
    rec = O.integrate_rays(_W["vox"], _W["tree"], _W["o"][lo:hi], _W["d"][lo:hi])
    return time.perf_counter() - t0, rec["depth"]


class CpuPool:
    """Spawned workers (OMP_NUM_THREADS=1) holding one workload's scene state."""

    def __init__(self, kind, regime="init", workers=None):
        import multiprocessing as mp
        from paper_2507_18713_b200.scenes import get_scene
        self.workers = workers or min(len(os.sched_getaffinity(0)), 64)
        get_scene({"c1": "S20k", "c2": "S1M", "c3": "S1M"}[kind], regime if kind != "c1" else "init")
        _pin_threads()  # inherited by the spawned workers before they import numpy
        # the reference package itself when it is installed (baseline/_ref), else the oracle port
        self.kind = "reference" if ref_available() else "port"
        t0 = time.perf_counter()
        self.pool = ProcessPoolExecutor(self.workers, mp_context=mp.get_context("spawn"),
                                        initializer=_cpu_init_ref if self.kind == "reference" else _cpu_init,
                                        initargs=(kind, regime))
        list(self.pool.map(_cpu_ready, range(self.workers)))
        self.init_s = time.perf_counter() - t0

    def close(self):
        self.pool.shutdown()


def c2_tiles_sample(seed, k):
    """k tiles stratified over the 68 tile rows (the per-tile cost depends
    strongly on the row: sky, horizon, road)."""
    rng = np.random.default_rng(seed)
    return [int(min(67, (b + rng.random()) * 68 / k)) * 120 + int(rng.integers(0, 120)) for b in range(k)]


def c2_cpu_step(pool: CpuPool, seed: int):
    """One bounded C2 sample: `workers` tiles in parallel, one per worker.
    Extrapolated frame time on these cores = (8160 / k) x sum(tile times) / workers."""
    tiles = c2_tiles_sample(seed, pool.workers)
    t0 = time.perf_counter()
    secs = list(pool.pool.map(_ref_c2_tiles if pool.kind == "reference" else _c2_tiles, [[t] for t in tiles]))
    wall = time.perf_counter() - t0
    frame_s = 8160 / len(tiles) * float(np.sum(secs)) / pool.workers
    return 1.0 / frame_s, wall, float(np.mean(secs))


def c1_cpu_frame(pool: CpuPool):
    """The whole C1 frame (256 x 256, 16 tile rows) in row bands over the workers."""
    bands = [(r, r + 1) for r in range(16)]
    t0 = time.perf_counter()
    out = list(pool.pool.map(_ref_c1_band if pool.kind == "reference" else _c1_band, bands))
    wall = time.perf_counter() - t0
    img = np.concatenate([c for _, c in out], axis=0)
    return wall, img


def c3_cpu_sweep(pool: CpuPool, n_rays=230400):
    """The whole C3 sweep in ray blocks over the workers."""
    cuts = np.linspace(0, n_rays, 4 * pool.workers + 1).round().astype(int)
    t0 = time.perf_counter()
    out = list(pool.pool.map(_ref_c3_block if pool.kind == "reference" else _c3_block, list(zip(cuts[:-1], cuts[1:]))))
    wall = time.perf_counter() - t0
    return wall, np.concatenate([d for _, d in out])


def run_reference(args, rank):
    """The reference arm: the reference algorithm on the host cores, same C2
    workload; each step is one bounded sample (workers tiles)."""
    if rank != 0:
        return
    pool = CpuPool("c2", args.regime)
    for w in range(args.warmup):
        c2_cpu_step(pool, 1000 + w)
    vals, walls = [], []
    for k in range(args.steps):
        v, wall, _ = c2_cpu_step(pool, k)
        vals.append(v)
        walls.append(wall)
    pool.close()
    value = float(np.mean(vals))
    sample = (f"{pool.workers} random 16x16 tiles of 8160 per step (one per worker, stratified over tile rows), "
              f"forward + backward, projection once per worker; frame time = 8160/{pool.workers} x sum(tile s) "
              f"/ {pool.workers} workers (extrapolated)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(walls)),
        "frames_per_step": pool.workers / 8160, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference pipeline scene S1M, bytes pinned by sha256)",
        "config": config_dict(args.regime, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": pool.workers, "kind": pool.kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "ms_per_step is the wall time of one sample step (a fraction frames_per_step of a frame); "
                "value is the extrapolated whole-frame rate on these cores",
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------
# GPU arm

class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
            return
        # NVML start-up takes ~0.1-0.3 s: wait for the first sample so the timed region is covered
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 3.0 and not Path(self.f.name).read_text().strip():
            time.sleep(0.01)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 8]
        mx = [float(r[2]) for r in rows if len(r) > 8]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows if len(r) > 8 for j in range(4)
                          if r[5 + j].strip().lower() == "active"})
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": float(np.median(load)) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def _dist_init(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "ours":
            # SALF_BENCH_BACKEND=gloo: functional check of the multi-rank path with
            # several ranks sharing one GPU (timings meaningless); default NCCL
            local = local % max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local)
            if os.environ.get("SALF_BENCH_BACKEND", "nccl") == "gloo":
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


# SURVEY §8(d) algorithmic (compulsory) bytes -- the roofline numerators
def bytes_raster_fwd(m, m_vis, hw):
    return 16 * m + 112 * m_vis + 20 * hw


def bytes_raster_bwd(m, m_vis, hw):
    return 16 * m + 220 * m_vis + 32 * hw


def bytes_lidar_fwd(r, u, n_nodes):
    return 24 * r + 12 * r + 128 * u + 4 * n_nodes


def traffic_model_raster(n_inst, m_vis, hw, n_tiles):
    """What THIS implementation must move per launch (its layout), for comparison
    with the ncu DRAM bytes: entry lists, 160-B records, CSR offsets, the f32
    image planes, the 64-B/pixel fp64 saved state, fp64 dL/dC, the (M_vis, 27)
    fp64 gradient rows."""
    rec = 32 + 16 + 112
    fwd = 4 * n_inst + rec * m_vis + 8 * (n_tiles + 1) + 20 * hw + 64 * hw
    bwd = 4 * n_inst + rec * m_vis + 8 * (n_tiles + 1) + 64 * hw + 24 * hw + 216 * m_vis
    return fwd, bwd


# flop models for the secondary ALU roofline (FP32; stated in DESIGN.md §6)
FLOP_PAIR = 24.0        # one ray-vs-voxel slab test
FLOP_SEG_FWD = 120.0    # fields + opacity + colour + compositing of one included segment
FLOP_SEG_BWD = 204.0    # the same fields (120) + the reverse chain and 27 gradient FMAs (84)


def _alu_peak(dev, fp32: bool) -> float:
    """Measured FP64 (DFMA) or FP32 (FFMA) throughput (TFLOP/s) of this GPU: best of 4 launches."""
    import torch
    from paper_2507_18713_b200 import _lib
    lib = _lib.load()
    scratch = torch.zeros(148 * 16, dtype=torch.float64, device=dev)
    grid, iters = 148 * 16, (16000 if fp32 else 4000)
    fn = lib.salf_fp32_peak if fp32 else lib.salf_fp64_peak
    best = 0.0
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(fn(scratch.data_ptr(), grid, iters, _lib.stream_ptr()))
        b.record()
        torch.cuda.synchronize()
        flops = grid * 256 * 64 * iters * 2.0
        best = max(best, flops / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def _json_file(rel):
    p = ROOT / rel
    return json.loads(p.read_text()) if p.exists() else None


def _timeit(fn, n=10, warm=3):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2507_18713_b200 import _lib, configs
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.backward import l1_color_seed
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.parallel import allreduce_grad_
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import gen_lidar_rays

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    scene = get_scene("S1M", args.regime)
    ds = DeviceScene.from_scene(scene, device=dev)
    # N = 1: the C2 camera; N > 1: rank r renders C5-rig camera r (distinct views)
    cam = configs.c2_camera(45.0 * (rank % 8) if world > 1 else 0.0)
    h, w = cam.height, cam.width
    g = torch.Generator().manual_seed(rank)
    gt_host = (0.3 + 0.4 * torch.rand((h, w, 3), generator=g)).pin_memory()
    gt_dev = gt_host.to(dev)
    grad = torch.zeros((ds.n, _lib.GRAD_STRIDE), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    out_host = torch.empty((h, w, 3), dtype=torch.float32).pin_memory()
    loss_host = torch.empty(1, dtype=torch.float64).pin_memory()

    def step(gt, events=None):
        fb, st = RR.rasterize(ds, cam, return_state=True, events=events)
        dc, lsum = l1_color_seed(fb.color, gt)  # losses.py:22-31, one fused kernel
        grad.zero_()
        RR.rasterize_backward(st, dc, None, grad, as_dict=False, events=events)
        if world > 1:
            allreduce_grad_(grad)  # f64 transport of the rows any rank touched
        return st

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        st = step(gt_dev)
    barrier()

    # kernel launches of one step (CUPTI via torch.profiler; outside the timed region)
    launches = ours = None
    kernel_names = None
    try:
        if args.no_profile:
            raise RuntimeError("--no-profile")
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(gt_dev)
            torch.cuda.synchronize()
        kern = [e for e in prof.events() if e.device_type.name == "CUDA"
                and not e.name.lower().startswith(("memcpy", "memset"))]
        launches = len(kern)
        mine = [e.name for e in kern if "salf" in e.name or "k_" in e.name]
        ours = len(mine)
        kernel_names = sorted({n.split("(")[0].split("<")[0].replace("void ", "") for n in mine})
    except Exception as ex:  # profiler unavailable: leave the count unset
        print(f"[bench] launch count unavailable: {ex}", file=sys.stderr)

    # ---- device-timed steps, inputs resident, L2 flushed between steps ----
    clocks = Clocks(local)
    barrier()
    times, kev = [], []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev = []
        a.record()
        step(gt_dev, events=ev)
        b.record()
        times.append((a, b))
        kev.append(ev)
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = [a.elapsed_time(b) for a, b in times]
    kms = {}
    for ev in kev:
        for name, s, e in ev:
            kms.setdefault(name, []).append(s.elapsed_time(e))
    step_ms = float(np.sum(ms)) / args.steps
    t_max = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    step_ms_max = float(t_max.item())
    value = world * 1e3 / step_ms_max

    # ---- end to end through the public API: pinned H2D of the target, D2H of frame + loss ----
    # Copies run on a side stream and overlap compute: step k+1's target is
    # uploaded during step k's backward, step k's frame is read back while its
    # backward runs.  Every byte still crosses PCIe inside the timed region.
    cs = torch.cuda.current_stream(dev)
    xs = torch.cuda.Stream(dev)
    gt_bufs = [torch.empty_like(gt_dev), torch.empty_like(gt_dev)]
    loss_dev = torch.zeros(1, dtype=torch.float64, device=dev)

    def e2e_pass(n_steps):
        up = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        xs.wait_stream(cs)
        with torch.cuda.stream(xs):
            gt_bufs[0].copy_(gt_host, non_blocking=True)
            up[0].record(xs)
        for k in range(n_steps):
            cur = gt_bufs[k % 2]
            cs.wait_event(up[k % 2])
            fb, st = RR.rasterize(ds, cam, return_state=True)
            dc, lsum = l1_color_seed(fb.color, cur)
            loss_dev.copy_((lsum / dc.numel()).reshape(1))
            used[k % 2].record(cs)
            xs.wait_event(used[k % 2])
            with torch.cuda.stream(xs):
                fb.color.record_stream(xs)
                loss_dev.record_stream(xs)
                out_host.copy_(fb.color, non_blocking=True)
                loss_host.copy_(loss_dev, non_blocking=True)
                if k + 1 < n_steps:
                    if k >= 1:
                        xs.wait_event(used[(k + 1) % 2])
                    gt_bufs[(k + 1) % 2].copy_(gt_host, non_blocking=True)
                    up[(k + 1) % 2].record(xs)
            grad.zero_()
            RR.rasterize_backward(st, dc, None, grad, as_dict=False)
            if world > 1:
                allreduce_grad_(grad)
        cs.wait_stream(xs)
        b.record(cs)
        return a, b

    e2e_pass(max(args.warmup, 3))
    barrier()
    a, b = e2e_pass(args.steps)
    barrier()
    te = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * 1e3 / float(te.item())

    # ---- roofline of the dominant kernel (SURVEY §8d bytes) ----
    peaks = _json_file("MEASURED_PEAKS.json") or {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    n_inst = st.n_instances
    m_vis = int(torch.unique(st.entries).numel()) if n_inst else 0
    hw = h * w
    n_tiles = st.offsets.numel() - 1
    k_fwd = float(np.mean(kms.get("raster_composite", [np.nan])))
    k_bwd = float(np.mean(kms.get("raster_backward", [np.nan])))
    fwd_b, bwd_b = bytes_raster_fwd(ds.n, m_vis, hw), bytes_raster_bwd(ds.n, m_vis, hw)
    fwd_t, bwd_t = traffic_model_raster(n_inst, m_vis, hw, n_tiles)
    dom, dom_ms, dom_b, dom_t = ("raster_backward", k_bwd, bwd_b, bwd_t) if k_bwd >= k_fwd else \
        ("raster_composite", k_fwd, fwd_b, fwd_t)
    achieved = dom_b / (dom_ms * 1e-3) / 1e9
    traffic = (_json_file("profiles/traffic.json") or {}).get(dom)

    # secondary ALU rooflines: P pair tests and S_inc included segments (read
    # from the frame's saved state) against a live FP32 FFMA probe
    sv = st.saved
    pairs = float(sv[:, 6].sum().item())  # list entries each pixel visited = pair tests
    s_inc = float(sv[:, 7].sum().item())
    fp32_peak = _alu_peak(dev, fp32=True)
    f_fwd = FLOP_PAIR * pairs + FLOP_SEG_FWD * s_inc
    f_bwd = FLOP_PAIR * pairs + FLOP_SEG_BWD * s_inc

    def alu(kernel, flops, kms_):
        ach = flops / (kms_ * 1e-3) / 1e12
        return {"bound": "fp32", "kernel": kernel, "unit": "TFLOP/s", "achieved": ach, "peak": fp32_peak,
                "frac": ach / fp32_peak, "flops": flops, "kernel_ms": kms_}

    roofline_alu = {
        "raster_backward": {**alu("raster_backward", f_bwd, k_bwd),
                            "formula": f"{FLOP_PAIR:.0f} P + {FLOP_SEG_BWD:.0f} S_inc (DESIGN.md §6)"},
        "raster_composite": {**alu("raster_composite", f_fwd, k_fwd),
                             "formula": f"{FLOP_PAIR:.0f} P + {FLOP_SEG_FWD:.0f} S_inc (SURVEY §8d)"},
        "pair_tests": pairs, "included_segments": s_inc,
        "peak_source": "live FFMA probe (salf_fp32_peak)", "fp64_peak": _alu_peak(dev, fp32=False),
        "ncu": _json_file("profiles/ncu_metrics.json"),
    }

    # ---- C3 LiDAR: one sweep per rank (sensor-sharded, no exchange) ----
    oc = RY.build_scene_octrees(scene)
    lid = configs.c3_lidar()
    lb = gen_lidar_rays(lid, device=dev)
    # the sweep as render_lidar_ranges renders it (render_ray.py:297-306: inference, no backward state)
    for _ in range(max(args.warmup, 3)):
        RY.render_lidar(ds, oc, lb, need_state=False)
    barrier()
    la, lb_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    la.record()
    for _ in range(args.steps):
        RY.render_lidar(ds, oc, lb, need_state=False)
    lb_ev.record()
    barrier()
    t_l = torch.tensor([la.elapsed_time(lb_ev) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_l, op=dist.ReduceOp.MAX)
    lidar_ms = float(t_l.item())
    lidar = {"metric": "LiDAR rays/s (128 beams x 1800 steps, S1M init)", "rays_per_s": world * lb.n / (lidar_ms * 1e-3),
             "sweeps_per_s": world * 1e3 / lidar_ms, "ms_per_sweep": lidar_ms, "n_gpus": world,
             "scaling": "weak", "sharding": "one LiDAR sweep per rank, no exchange",
             "what": "render_lidar_ranges (inference; the training path with backward state is inside c5)"}

    # ---- C5: the rig training step sharded over the ranks (strong scaling) ----
    c5 = c5_step(args, world, rank, dev, scene, ds, oc, barrier)

    if rank != 0:
        return

    if not args.no_extras:
        # LiDAR HBM roofline: U = distinct voxels touched by the sweep's segments
        ret = RY.render_lidar(ds, oc, lb)
        ray, vid, _, _ = RY.segments(ds, oc, lb.origins, lb.dirs)
        u = int(torch.unique(vid).numel())
        del ray, vid
        n_nodes = int(oc.static.n_nodes)
        lb_bytes = bytes_lidar_fwd(lb.n, u, n_nodes)
        la_ach = lb_bytes / (lidar_ms * 1e-3) / 1e9
        lidar["roofline"] = {"bound": "hbm", "kernel": "ray_forward (LiDAR)", "achieved": la_ach, "peak": peak,
                             "unit": "GB/s", "frac": la_ach / peak, "algorithmic_bytes": lb_bytes,
                             "touched_voxels": u, "octree_nodes": n_nodes, "rays": lb.n,
                             "segments": int(ret.saved[:, 6].sum().item()),
                             "formula": "36 R + 128 U + 4 N_nodes (SURVEY §8d)",
                             "traffic": (_json_file("profiles/traffic.json") or {}).get("ray_forward")}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (reference pipeline scene S1M, bytes pinned by sha256; random target image)",
        "config": config_dict(args.regime, world, {"render_instances": n_inst, "visible_voxels": m_vis}),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(gt_host.nbytes),
                "d2h_bytes_per_step": int(out_host.nbytes + loss_host.nbytes)},
        "gpu_launches": ours if ours is not None else launches,
        "gpu_launches_all": launches,
        "kernels": kernel_names,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes": dom_b,
                     "formula": "16 M + 220 M_vis + 32 H W (SURVEY §8d, raster backward)"
                     if dom == "raster_backward" else "16 M + 112 M_vis + 20 H W (SURVEY §8d, raster forward)",
                     "traffic_model": dom_t, "kernel_ms": dom_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650"},
        "roofline_alu": roofline_alu,
        "lidar": lidar,
        "c5": c5,
        "kernels_ms": {k: float(np.mean(v)) for k, v in kms.items()},
        "clocks": clk,
    }
    if world == 1 and not args.no_extras:
        line["extras"] = extras(ds, oc, args)
    if world == 1 and not args.no_cpu:
        line.update(cpu_baselines(args, ds, dev, lidar_ms, value))
    print(json.dumps(line), flush=True)


def c5_step(args, world, rank, dev, scene, ds, oc, barrier):
    """C5: 8 cameras + 2 LiDARs sharded over the ranks (split_work -> assign:
    pinhole row bands and LiDAR ray blocks, LPT-balanced), global L1 seeds
    (counts all-reduced), raster + ray backward into the (M, 27) buffer, NCCL
    all-reduce of the touched rows (f64), device Adam.  Strong scaling."""
    import torch
    import torch.distributed as dist
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200.optim import TrainableScene
    from paper_2507_18713_b200.parallel import assign, split_work
    from paper_2507_18713_b200.train_step import rig_step
    ts = TrainableScene(scene, device=dev)
    cams, lidars = configs.c5_rig()
    sensors = cams + lidars
    g = torch.Generator().manual_seed(5)
    targets = [torch.rand((c.height, c.width, 3), generator=g, dtype=torch.float64).to(dev) for c in cams] + \
              [(1.0 + 20.0 * torch.rand(l.beam_elevations.shape[0] * l.steps, generator=g,
                                        dtype=torch.float64)).to(dev) for l in lidars]
    items = assign(split_work(sensors, world), world)[rank]
    gbuf = ts.zero_grad()

    def one():
        gbuf.zero_()
        rig_step(ts.ds, oc, sensors, targets, items, gbuf)
        ts.adam_step(gbuf)

    n = max(2, min(args.steps, 5))
    for _ in range(2):
        one()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        one()
    b.record()
    barrier()
    t = torch.tensor([a.elapsed_time(b) / n], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    del ts, gbuf, targets
    return {"metric": "C5 rig training steps/s (8 x 1920x1080 cameras + 2 x 128x1800 LiDARs, S1M)",
            "steps_per_s": 1e3 / ms, "ms_per_step": ms, "camera_frames_per_s": 8e3 / ms,
            "lidar_rays_per_s": 2 * 230400 * 1e3 / ms, "n_gpus": world, "scaling": "strong",
            "items_this_rank": len(items), "steps": n,
            "includes": "forward, global L1 seeds, raster + ray backward, grad all-reduce, device Adam + refresh"}


def extras(ds, oc, args):
    """Secondary configurations on rank 0: C2 forward only, surface regime, C4, intensity/ray-drop."""
    import torch
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import camera_rays, gen_lidar_rays

    out = {}
    cam = configs.c2_camera()
    out["c2_forward_fps"] = 1e3 / _timeit(lambda: RR.rasterize(ds, cam))
    lidar = configs.c3_lidar()
    lb = gen_lidar_rays(lidar)
    rng = np.random.default_rng(0)
    feat = torch.as_tensor(rng.uniform(-1, 1, (ds.n, 8)).astype(np.float32), device=ds.device)
    head = rng.uniform(-0.5, 0.5, (2, 13)).astype(np.float32)
    ms = _timeit(lambda: RY.render_lidar(ds, oc, lb, features=feat, head=head))
    out["c3_lidar_intensity_raydrop"] = {"sweeps_per_s": 1e3 / ms, "rays_per_s": lb.n / (ms * 1e-3), "ms": ms}
    ms = _timeit(lambda: RY.render_lidar(ds, oc, gen_lidar_rays(lidar), need_state=False))
    out["c3_lidar_with_raygen"] = {"sweeps_per_s": 1e3 / ms, "ms": ms}
    del feat

    # BASELINE.md §3 surface regime: bake (a = 50, b = 0.02) + the reference prune (densify.py:39-46)
    def regime_block(name, note):
        sc = get_scene("S1M", name)
        dss = DeviceScene.from_scene(sc)
        ocs = RY.build_scene_octrees(sc)
        dcs = torch.full((1080, 1920, 3), 1e-7, dtype=torch.float64, device=dss.device)

        def fb_step():
            fb, st = RR.rasterize(dss, cam, return_state=True)
            RR.rasterize_backward(st, dcs, None, as_dict=False)

        ms_l = _timeit(lambda: RY.render_lidar(dss, ocs, lb, need_state=False))
        return {"voxels": dss.n, "c2_forward_fps": 1e3 / _timeit(lambda: RR.rasterize(dss, cam)),
                "c2_fwd_bwd_fps": 1e3 / _timeit(fb_step, n=5),
                "c3_lidar_sweeps_per_s": 1e3 / ms_l, "c3_lidar_rays_per_s": lb.n / (ms_l * 1e-3),
                "note": note}

    out["surface_regime"] = regime_block(
        "surface", "BASELINE.md §3: S1M fields baked from the analytic primitives (a = 50, b = 0.02, "
                   "SH DC = logit(albedo)/C0), pruned by center_opacity < 0.005 (densify.py:39-46)")
    out["surface_dense_regime"] = regime_block(
        "surface-dense", "trained-like: S1M inner region densified to level 7 near the analytic surfaces, "
                         "fields baked a = 400, b = 0.004 (scenes.make_dense_surface_scene)")
    s2 = get_scene("S2M", "init")
    ds2 = DeviceScene.from_scene(s2)
    oc2 = RY.build_scene_octrees(s2)
    c4 = configs.c4_camera()

    def c4_frame():
        b = camera_rays(c4)
        return RY.integrate_rays(ds2, oc2, b.origins, b.dirs, valid=b.valid, check_unit=False, check=False,
                                 need_state=False)  # render_rays_image semantics (no backward)

    out["c4_fisheye_rs_fps_S2M"] = 1e3 / _timeit(c4_frame, n=5)
    del ds2, oc2

    # dynamic actors: two moving, yawing cars (~12k voxels each) on S1M; the C3
    # sweep through integrate_rays' merge path (static march without early stop + actor frames on
    # the device + merged composite, render_ray.py:161-239) and the C2 frame with the actors
    # flattened at t (render_raster.py:63-89)
    from paper_2507_18713_b200.scenes import with_moving_actors
    sa = with_moving_actors(get_scene("S1M", "init"))
    oca = RY.build_scene_octrees(sa)
    lbt = gen_lidar_rays(lidar)  # per-ray time stamps over the scan period

    def lidar_actors():
        return RY.integrate_rays(sa, oca, lbt.origins, lbt.dirs, lbt.t_stamps, check_unit=False, check=False)

    ms_a = _timeit(lidar_actors, n=5)
    ms_r = _timeit(lambda: RR.rasterize_scene(sa, cam, 0.05), n=5)
    out["actors"] = {"actors": len(sa.actors), "actor_voxels": int(sum(a.voxels.n for a in sa.actors)),
                     "c3_lidar_sweeps_per_s": 1e3 / ms_a, "c3_lidar_ms": ms_a,
                     "c2_raster_forward_fps_incl_flatten_upload": 1e3 / ms_r,
                     "note": "S1M init + 2 moving cars; LiDAR via the merge path (no early stop with live "
                             "actors, render_ray.py:175); raster: static set resident, the posed actor voxels "
                             "(host NumPy poses, render_raster.py:70-82) uploaded per frame"}
    return out


def cpu_baselines(args, ds, dev, lidar_ms, value):
    """The reference algorithm on this box's cores (OMP_NUM_THREADS=1 workers):
    C2 sampled (extrapolated, labelled), C1 whole frame and C3 whole sweep
    (not extrapolated), each next to the GPU number of the same workload."""
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.scenes import get_scene
    out = {}
    pool = CpuPool("c2", args.regime)
    vals = []
    walls = []
    for k in range(2):
        v, wall, tile_s = c2_cpu_step(pool, 7 + k)
        vals.append(v)
        walls.append(wall)
    pool.close()
    v = float(np.mean(vals))
    out["cpu_baseline"] = {
        "value": v, "unit": UNIT, "cores": pool.workers, "kind": pool.kind,
        "sample": f"2 x {pool.workers} random 16x16 tiles of the 8160 (one per worker, stratified over tile rows), "
                  f"fwd + bwd, projection once per worker, {float(np.sum(walls)):.1f} s wall; frame time = "
                  f"8160/k x sum(tile s) / {pool.workers} workers (EXTRAPOLATED)",
        "gpu_over_cpu": value / v}
    # C1: the whole 256^2 frame on S20k, row bands over the cores, vs the GPU
    import torch
    pool = CpuPool("c1")
    wall, img = c1_cpu_frame(pool)
    pool.close()
    c1cam = configs.c1_camera()
    from paper_2507_18713_b200.device import DeviceScene
    ds20 = DeviceScene.from_scene(get_scene("S20k", "init"), device=dev)
    gpu_ms = _timeit(lambda: RR.rasterize(ds20, c1cam), n=20)
    gimg = RR.rasterize(ds20, c1cam).color.double().cpu().numpy()
    out["c1"] = {"workload": "C1: S20k (19,992 voxels), 256x256 pinhole raster forward (BASELINE configs[0])",
                 "gpu_fps": 1e3 / gpu_ms, "cpu_fps": 1.0 / wall, "cpu_cores": pool.workers,
                 "cpu_kind": pool.kind, "cpu_s_per_frame": wall, "gpu_over_cpu": (1e3 / gpu_ms) * wall,
                 "max_abs_diff_gpu_vs_cpu": float(np.abs(gimg - img).max()),
                 "note": "whole frame on both sides, not extrapolated (16 tile-row bands over the workers)"}
    del ds20
    # C3: the whole sweep on the cores vs the GPU sweep
    pool = CpuPool("c3")
    wall, dep = c3_cpu_sweep(pool)
    pool.close()
    out["cpu_baseline_lidar"] = {
        "workload": "C3: 128 x 1800 LiDAR sweep on S1M (BASELINE configs[2])",
        "value": 230400 / wall, "unit": "rays/s", "cores": pool.workers, "kind": pool.kind,
        "sample": "the whole sweep (230,400 rays) in ray blocks over the workers, not extrapolated",
        "gpu_rays_per_s": 230400 / (lidar_ms * 1e-3), "gpu_over_cpu": (230400 / (lidar_ms * 1e-3)) / (230400 / wall),
        "returns": int(np.isfinite(dep).sum())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--regime", choices=["init", "surface"], default="init")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the CUPTI launch count (under ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = _dist_init(args)
    try:
        if args.impl == "reference":
            run_reference(args, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
