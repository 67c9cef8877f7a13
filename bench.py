"""Benchmark: C2 -- 1920x1080 pinhole raster forward + backward on the 1M-voxel
synthetic scene (S1M), one frame per rank per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: each rank renders its own C5-rig
camera (yaw = 45 deg x rank) forward + backward and the per-voxel gradient
buffer is all-reduced over NCCL (the training step's one exchange).  `value`
is whole-job frames/s; rank 0 prints one JSON line.  `--impl reference` times
the reference's CPU algorithm (the oracle port, oracle/salf_oracle.py) on the
host cores on a bounded sample of the same workload.
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


# ------------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on a bounded tile sample

_W = {}


def _cpu_init(regime):
    from oracle import salf_oracle as O
    from paper_2507_18713_b200.scenes import get_scene
    sc = get_scene("S1M", regime)
    b, v = sc.bounds, sc.static
    _W["vox"] = O.Voxels.from_grid(b.aabb_min, b.aabb_max, b.base_edge, v.level, v.ijk, v.w_s, v.w_c,
                                   v.w_sh, v.log_a, v.log_b)


def _cpu_tile(args):
    """Reference forward (rasterize) + backward (raster records -> backward_records)
    of ONE 16x16 tile of the C2 frame; returns seconds."""
    from oracle import salf_oracle as O
    from paper_2507_18713_b200 import configs
    tx, ty = args
    c = configs.c2_camera()
    cam = O.Camera("pinhole", c.width, c.height, c.fx, c.fy, c.cx, c.cy, position=c.position,
                   quaternion=c.quaternion)
    vox = _W["vox"]
    t0 = time.perf_counter()
    win = (tx, ty, tx, ty)
    fb = O.rasterize(vox, cam, window=win)
    rec = O.raster_records(vox, cam, window=win)
    dc = np.zeros((rec["n_rays"], 3))
    dc[:] = 1e-6
    O.backward_records(rec, vox, dc, np.zeros(rec["n_rays"]))
    del fb
    return time.perf_counter() - t0


def _cpu_ready(_):
    return "vox" in _W


def _sample_tiles(k, seed):
    """k tiles stratified over the 68 tile rows (one per row band, random row
    inside the band and random column): the per-tile cost depends strongly on
    the row (sky, horizon, road), so stratifying cuts the estimate's variance."""
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(0, 120)), int(min(67, (b + rng.random()) * 68 / k))) for b in range(k)]


class CpuBaseline:
    def __init__(self, regime="init", workers=None):
        n = workers or min(len(os.sched_getaffinity(0)), 64)
        self.workers = n
        from paper_2507_18713_b200.scenes import get_scene
        get_scene("S1M", regime)  # build the cached container once, before the workers start
        import multiprocessing as mp
        self.pool = ProcessPoolExecutor(n, mp_context=mp.get_context("spawn"), initializer=_cpu_init,
                                        initargs=(regime,))
        list(self.pool.map(_cpu_ready, range(n)))  # every worker has loaded the scene

    def sample(self, seed):
        """One bounded sample: `workers` tiles in parallel -> extrapolated frames/s."""
        tiles = _sample_tiles(self.workers, seed)
        t0 = time.perf_counter()
        secs = list(self.pool.map(_cpu_tile, tiles))
        wall = time.perf_counter() - t0
        tiles_per_s = len(tiles) / wall
        return tiles_per_s / (120 * 68), dict(wall_s=wall, tile_s_mean=float(np.mean(secs)))

    def close(self):
        self.pool.shutdown()


def run_reference(args, rank):
    if rank != 0:
        return
    base = CpuBaseline("init")
    for w in range(args.warmup):
        base.sample(1000 + w)
    vals, info = [], []
    for k in range(args.steps):
        v, i = base.sample(k)
        vals.append(v)
        info.append(i)
    base.close()
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference pipeline scene S1M, bytes pinned by sha256)",
        "config": {"workload": WORKLOAD, "resolution": [1920, 1080], "voxels": 1023816,
                   "sample": "one 16x16 tile per worker per step, extrapolated to 8160 tiles"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": base.workers, "kind": "port",
                         "sample": f"{base.workers} tiles of 8160 per step, stratified over tile rows "
                                   "(fwd+bwd), extrapolated linearly to the full frame"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": {"tile_s_mean": float(np.mean([i["tile_s_mean"] for i in info]))},
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
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

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


def _algorithmic_bytes(n_inst, m_vis, hw, n_tiles, depth_seeds=False):
    """Compulsory HBM bytes per launch; the backward
    reads dL/dC (24 B/pixel) and, with depth seeds, dL/dD (8 B/pixel)."""
    rec = 32 + 16 + 112  # geo + ab + prm per visible voxel
    fwd = 4 * n_inst + rec * m_vis + 8 * (n_tiles + 1) + 20 * hw + 64 * hw
    seeds = (32 if depth_seeds else 24) * hw
    bwd = 4 * n_inst + rec * m_vis + 8 * (n_tiles + 1) + 64 * hw + seeds + 216 * m_vis
    return fwd, bwd


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


def _ncu_metrics():
    """Per-kernel ncu metrics of the committed capture (profiles/), if present:
    the roofline above is HBM; these kernels are FP64-pipe / latency bound."""
    p = ROOT / "profiles" / "ncu_metrics.json"
    return json.loads(p.read_text()) if p.exists() else None


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2507_18713_b200 import _lib, configs
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200.backward import l1_color_seed
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    scene = get_scene("S1M", args.regime)
    ds = DeviceScene.from_scene(scene, device=dev)
    # every rank renders the C2 view: identical per-rank work, so the N-GPU
    # number measures the data-parallel step (weak scaling), not pose imbalance
    cam = configs.c2_camera()
    h, w = cam.height, cam.width
    g = torch.Generator().manual_seed(rank)
    gt_host = (0.3 + 0.4 * torch.rand((h, w, 3), generator=g)).pin_memory()
    gt_dev = gt_host.to(dev)
    dd = None  # colour L1 loss only (losses.py:22-31): no depth seeds, the backward drops the depth term
    grad = torch.zeros((ds.n, _lib.GRAD_STRIDE), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    out_host = torch.empty((h, w, 3), dtype=torch.float32).pin_memory()
    loss_host = torch.empty(1, dtype=torch.float64).pin_memory()

    from paper_2507_18713_b200.parallel import allreduce_grad_
    SPARSE_ALLREDUCE = os.environ.get("SALF_SPARSE_ALLREDUCE", "1") == "1"

    def allreduce_grad(buf):
        # fp32 transport of the rows any rank touched (parallel.allreduce_grad_)
        allreduce_grad_(buf, sparse=SPARSE_ALLREDUCE)

    def step(gt, events=None, e2e=False):
        fb, st = RR.rasterize(ds, cam, return_state=True, events=events)
        dc, lsum = l1_color_seed(fb.color, gt)  # losses.py:22-31, one fused kernel
        grad.zero_()
        RR.rasterize_backward(st, dc, dd, grad, as_dict=False, events=events)
        if world > 1:
            allreduce_grad(grad)
        if e2e:
            loss_host.copy_((lsum / dc.numel()).reshape(1), non_blocking=True)
            out_host.copy_(fb.color, non_blocking=True)
        return st

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        st = step(gt_dev)
    barrier()

    # kernel launches of one step (CUPTI via torch.profiler; outside the timed region)
    launches = None
    ours = None
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
        ours = sum(1 for e in kern if "salf" in e.name or "k_" in e.name or "cub" in e.name.lower())
    except Exception as ex:  # profiler unavailable: leave the count unset
        ours = None
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
            RR.rasterize_backward(st, dc, dd, grad, as_dict=False)
            if world > 1:
                allreduce_grad(grad)
        cs.wait_stream(xs)
        b.record(cs)
        return a, b

    # untimed warm-up of the end-to-end pipeline (pinned copies, side stream,
    # allocator blocks held by record_stream), then the timed pass
    e2e_pass(max(args.warmup, 3))
    barrier()
    a, b = e2e_pass(args.steps)
    barrier()
    e2e_ms = a.elapsed_time(b) / args.steps
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * 1e3 / float(te.item())

    # ---- the LiDAR half of the metric at N GPUs: each rank sweeps its own
    # 128 x 1800 C3 LiDAR (sensor-sharded, no exchange), device-timed, max over ranks ----
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.sensors import gen_lidar_rays
    oc = RY.build_scene_octrees(scene)
    lid = configs.c3_lidar()
    lb = gen_lidar_rays(lid)
    for _ in range(max(args.warmup, 3)):
        RY.render_lidar(ds, oc, lb)
    barrier()
    la, lb_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    la.record()
    for _ in range(args.steps):
        RY.render_lidar(ds, oc, lb)
    lb_ev.record()
    barrier()
    t_l = torch.tensor([la.elapsed_time(lb_ev) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_l, op=dist.ReduceOp.MAX)
    lidar_ms = float(t_l.item())
    del oc

    if rank != 0:
        return

    # ---- roofline of the dominant kernel ----
    peaks = {}
    pp = ROOT / "MEASURED_PEAKS.json"
    if pp.exists():
        peaks = json.loads(pp.read_text())
    peak = float(peaks.get("hbm_gbs", 6650.0))
    n_inst = st.n_instances
    m_vis = int(torch.unique(st.entries).numel()) if n_inst else 0
    fwd_b, bwd_b = _algorithmic_bytes(n_inst, m_vis, h * w, (st.offsets.numel() - 1))
    k_fwd = float(np.mean(kms.get("raster_composite", [np.nan])))
    k_bwd = float(np.mean(kms.get("raster_backward", [np.nan])))
    dom, dom_ms, dom_b = ("raster_backward", k_bwd, bwd_b) if k_bwd >= k_fwd else \
        ("raster_composite", k_fwd, fwd_b)
    achieved = dom_b / (dom_ms * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(dom)

    # secondary (ALU) roofline of the forward composite: SURVEY §8d's
    # F = 24 P + 120 S_inc flop (P = pair tests, S_inc = included segments,
    # both read from the frame's saved state) against a live FP32 FFMA peak
    # probe -- the default path shades in fp32 (fp64 only for the per-pair
    # closest-approach parameter and the log-transmittance sum)
    sv = st.saved
    pairs = float(sv[:, 6].sum().item())
    s_inc = float(sv[:, 7].sum().item())
    flops = 24.0 * pairs + 120.0 * s_inc
    fp32_peak = _alu_peak(dev, fp32=True)
    alu = {"bound": "fp32", "kernel": "raster_composite", "unit": "TFLOP/s",
           "achieved": flops / (k_fwd * 1e-3) / 1e12, "peak": fp32_peak,
           "frac": flops / (k_fwd * 1e-3) / 1e12 / fp32_peak, "flops": flops,
           "pair_tests": pairs, "included_segments": s_inc,
           "formula": "24 P + 120 S_inc (SURVEY 8d)", "peak_source": "live FFMA probe (salf_fp32_peak)",
           "fp64_peak": _alu_peak(dev, fp32=False)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (reference pipeline scene S1M, bytes pinned by sha256; random target image)",
        "config": {"workload": WORKLOAD, "regime": args.regime, "resolution": [w, h],
                   "voxels": ds.n, "parallelism": f"data-parallel x{world} (C2 view per rank), grad all-reduce "
                   f"({os.environ.get('SALF_BENCH_BACKEND', 'nccl').upper()}, fp32 transport"
                   + (", rows any rank touched)" if SPARSE_ALLREDUCE else ")"),
                   "l2": "flushed (256 MB write) between timed steps", "render_instances": n_inst,
                   "visible_voxels": m_vis},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(gt_host.nbytes),
                "d2h_bytes_per_step": int(out_host.nbytes + loss_host.nbytes)},
        "gpu_launches": ours if ours is not None else launches,
        "gpu_launches_all": launches,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes": dom_b, "kernel_ms": dom_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650"},
        "roofline_alu": alu,
        "lidar": {"metric": "LiDAR rays/s (128-beam, 1800 steps, S1M init)", "rays_per_s": world * lb.n / (lidar_ms * 1e-3),
                  "sweeps_per_s": world * 1e3 / lidar_ms, "ms_per_sweep": lidar_ms, "n_gpus": world,
                  "scaling": "weak", "sharding": "one LiDAR sweep per rank, no exchange"},
        "kernels_ms": {k: float(np.mean(v)) for k, v in kms.items()},
        "ncu": _ncu_metrics(),
        "clocks": clk,
    }
    if not args.no_extras and world == 1:
        line["extras"] = extras(ds, args)
    if not args.no_cpu and world == 1:
        base = CpuBaseline(args.regime)
        v, info = base.sample(7)
        base.close()
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": base.workers, "kind": "port",
                                "sample": f"{base.workers} 16x16 tiles of 8160 stratified over tile rows (fwd+bwd), "
                                          f"{info['wall_s']:.1f} s wall, extrapolated to the frame"}
    print(json.dumps(line), flush=True)


def extras(ds, args):
    """Secondary configurations on rank 0: C2 forward only, C3 LiDAR, C4 fisheye, surface regime."""
    import torch
    from paper_2507_18713_b200 import configs
    from paper_2507_18713_b200 import render_raster as RR
    from paper_2507_18713_b200 import render_ray as RY
    from paper_2507_18713_b200.device import DeviceScene
    from paper_2507_18713_b200.scenes import get_scene
    from paper_2507_18713_b200.sensors import camera_rays, gen_lidar_rays

    def timeit(fn, n=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    out = {}
    cam = configs.c2_camera()
    out["c2_forward_fps"] = 1e3 / timeit(lambda: RR.rasterize(ds, cam))
    scene = get_scene("S1M", args.regime)
    oc = RY.build_scene_octrees(scene)
    lidar = configs.c3_lidar()
    lb = gen_lidar_rays(lidar)

    def c3(dsx, ocx, **kw):
        ms = timeit(lambda: RY.render_lidar(dsx, ocx, lb, **kw))
        ms_gen = timeit(lambda: RY.render_lidar(dsx, ocx, gen_lidar_rays(lidar), **kw))
        ret = RY.render_lidar(dsx, ocx, lb, **kw)
        return {"rays_per_s": lb.n / (ms * 1e-3), "sweeps_per_s": 1e3 / ms, "ms": ms,
                "ms_with_raygen": ms_gen, "rays": lb.n,
                "segments": int(ret.saved[:, 6].sum().item()),
                "returns": int(torch.isfinite(ret.depth).sum().item()),
                "status_max": int(ret.status.max().item())}

    out["c3_lidar"] = c3(ds, oc)
    rng = np.random.default_rng(0)
    feat = torch.as_tensor(rng.uniform(-1, 1, (ds.n, 8)).astype(np.float32), device=ds.device)
    head = rng.uniform(-0.5, 0.5, (2, 13)).astype(np.float32)
    out["c3_lidar_intensity_raydrop"] = c3(ds, oc, features=feat, head=head)
    del feat
    s2 = get_scene("S2M", "init")
    ds2 = DeviceScene.from_scene(s2)
    oc2 = RY.build_scene_octrees(s2)
    c4 = configs.c4_camera()

    def c4_frame():
        b = camera_rays(c4)
        return RY.integrate_rays(ds2, oc2, b.origins, b.dirs, valid=b.valid, check_unit=False)

    out["c4_fisheye_rs_fps_S2M"] = 1e3 / timeit(c4_frame, n=5)
    del ds2, oc2
    sur = get_scene("S1M", "surface-dense")
    dss = DeviceScene.from_scene(sur)
    ocs = RY.build_scene_octrees(sur)
    dcs = torch.full((1080, 1920, 3), 1e-7, dtype=torch.float64, device=dss.device)
    dds = None  # colour-only loss

    def fb_step():
        fb, st = RR.rasterize(dss, cam, return_state=True)
        RR.rasterize_backward(st, dcs, dds, as_dict=False)

    # C5: the 8-camera + 2-LiDAR rig training step on one GPU (all sensors on
    # this rank): forward, global L1 seeds, backward, then device Adam
    from paper_2507_18713_b200.optim import TrainableScene
    from paper_2507_18713_b200.parallel import split_work
    from paper_2507_18713_b200.train_step import rig_step
    ts = TrainableScene(scene)
    cams, lidars = configs.c5_rig()
    sensors = cams + lidars
    g = torch.Generator().manual_seed(5)
    targets = [torch.rand((c.height, c.width, 3), generator=g, dtype=torch.float64).to(ts.ds.device)
               for c in cams] + [(1.0 + 20.0 * torch.rand(l.beam_elevations.shape[0] * l.steps, generator=g,
                                                            dtype=torch.float64)).to(ts.ds.device) for l in lidars]
    items = split_work(sensors, 1)
    gbuf = ts.zero_grad()

    def c5_step():
        gbuf.zero_()
        rig_step(ts.ds, oc, sensors, targets, items, gbuf)
        ts.adam_step(gbuf)

    ms5 = timeit(c5_step, n=3)
    out["c5_train_step"] = {"ms": ms5, "steps_per_s": 1e3 / ms5, "sensors": "8 x 1920x1080 pinhole + 2 x 128x1800 LiDAR",
                            "includes": "forward, L1 seeds, raster + ray backward, device Adam, scene refresh"}
    del ts, gbuf, targets
    # §8f rows beyond the hot path: densify round, salf.v1 device load, secondary effects
    import time
    from paper_2507_18713_b200.densify import DensifyConfig
    from paper_2507_18713_b200.device import load_device_scene
    from paper_2507_18713_b200.octree import build_octree_from_device
    from paper_2507_18713_b200.scenes import DATA
    ts = TrainableScene(scene)
    gacc = torch.rand(ts.n, dtype=torch.float64, device=ts.ds.device, generator=torch.Generator(
        device=ts.ds.device).manual_seed(1))

    def dens():
        t2 = TrainableScene.__new__(TrainableScene)
        t2.__dict__.update(ts.__dict__)
        t2.densify(gacc, DensifyConfig(budget=ts.n + 40 * 20000))
        build_octree_from_device(t2.level8, t2.ijk, scene.bounds)

    out["densify_round_S1M"] = {"ms": timeit(dens, n=3), "splits": 20000,
                                "includes": "flags, ranking, gather + 8-child expansion, moment remap, "
                                            "device scene rebuild, device octree build"}
    del ts, gacc
    sp = DATA / "S1M_init"
    if (sp / "voxels.bin").exists():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        load_device_scene(sp)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        from paper_2507_18713_b200.scene import load_scene
        sc_h, _ = load_scene(sp)
        DeviceScene.from_scene(sc_h)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out["scene_load_S1M"] = {"device_decode_s": t1 - t0, "host_load_plus_upload_s": t2 - t1,
                                 "bytes": (sp / "voxels.bin").stat().st_size}
    sph = [RY.InjectedSphere([2.0, 0.0, 0.8], 0.6, "mirror"), RY.InjectedSphere([4.0, 1.5, 0.6], 0.5, "glass"),
           RY.InjectedSphere([3.0, -1.5, 0.5], 0.4, "opaque", albedo=[0.8, 0.2, 0.1])]
    cb = camera_rays(cam)
    out["effects_c2_camera_S1M"] = {
        "fps": 1e3 / timeit(lambda: RY.trace_effects(ds, oc, cb.origins, cb.dirs, None, sph, [0.3, -0.5, 0.8],
                                                     max_bounces=2), n=3),
        "rays": cb.n, "spheres": "mirror, glass, opaque; 2 bounces; sun shadows"}
    out["surface_dense_regime"] = {
        "voxels": dss.n,
        "c2_forward_fps": 1e3 / timeit(lambda: RR.rasterize(dss, cam)),
        "c2_fwd_bwd_fps": 1e3 / timeit(fb_step, n=5),
        "c3_lidar": c3(dss, ocs),
        "note": "trained-like scene: S1M inner region densified to level 7 near the analytic "
                "surfaces (scenes.make_dense_surface_scene), fields baked a=400, b=0.004"}
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
