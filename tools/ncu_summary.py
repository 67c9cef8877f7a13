"""Summarise an ncu --set full report into profiles/: per-kernel duration,
DRAM traffic, L2/L1 hit rates, occupancy, pipe utilisation, top stalls.
Usage: python tools/ncu_summary.py <report.ncu-rep> <out.md> [traffic.json]"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def _hbm_gbs():
    from pathlib import Path
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6550.0


HBM_GBS = _hbm_gbs()


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, out_md, traffic_json=None):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    scale = {"ms": 1e6, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "ns": 1.0, "nsecond": 1.0,
             "s": 1e9, "second": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}
    per = defaultdict(list)
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        vals = {}
        for w in want:
            if w in col:
                try:
                    vals[w] = float(r[col[w]].replace(",", "")) * scale.get(units[col[w]], 1.0)
                except ValueError:
                    pass
        per[name].append(vals)
    lines = [f"# ncu summary of `{rep.split('/')[-1]}`", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(tools/ncu_target.py: C2 raster fwd+bwd and C3 LiDAR on S1M init). "
             "Per-launch means over the captured launches.", ""]
    traffic = {}
    metrics = {}
    for name, lst in per.items():
        avg = {k: sum(v[k] for v in lst if k in v) / max(1, sum(1 for v in lst if k in v)) for k in want}
        dur_ms = avg["gpu__time_duration.sum"] / 1e6
        rd, wr = avg["dram__bytes_read.sum"], avg["dram__bytes_write.sum"]
        key = {"k_composite": "raster_composite", "k_composite_fast": "raster_composite",
               "k_composite_redo": "raster_composite_redo", "k_backward": "raster_backward",
               "k_backward_fast": "raster_backward", "k_backward_hits": "raster_backward",
               "k_ray_forward": "ray_forward",
               "k_ray_forward_fast": "ray_forward", "k_ray_backward": "ray_backward"}.get(
            name.split("<")[0].replace("salf::", ""), name)
        traffic[key] = rd + wr
        metrics[key] = {"duration_ms": dur_ms, "dram_bytes": rd + wr,
                        "l2_hit_pct": avg["lts__t_sector_hit_rate.pct"],
                        "l1_hit_pct": avg["l1tex__t_sector_hit_rate.pct"],
                        "occupancy_pct": avg["sm__warps_active.avg.pct_of_peak_sustained_active"],
                        "registers": avg["launch__registers_per_thread"],
                        "issue_active_pct": avg["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                        "fp64_pipe_pct": avg["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]}
        lines += [f"## {name} ({len(lst)} launches)", "",
                  f"* duration {dur_ms:.3f} ms; DRAM read {rd / 1e6:.1f} MB + write {wr / 1e6:.1f} MB "
                  f"= {(rd + wr) / dur_ms / 1e6:.1f} GB/s ({100 * (rd + wr) / dur_ms / 1e6 / HBM_GBS:.2f}% of the "
                  f"measured {HBM_GBS:.0f} GB/s)",
                  f"* L2 hit {avg['lts__t_sector_hit_rate.pct']:.1f}%, L1 hit {avg['l1tex__t_sector_hit_rate.pct']:.1f}%",
                  f"* registers/thread {avg['launch__registers_per_thread']:.0f}, achieved occupancy "
                  f"{avg['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f}%",
                  f"* issue active {avg['smsp__issue_active.avg.pct_of_peak_sustained_active']:.1f}%, "
                  f"FP64 pipe {avg['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:.1f}%, "
                  f"ALU {avg['sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active']:.1f}%, "
                  f"FMA {avg['sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active']:.1f}%, "
                  f"LSU {avg['sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']:.1f}%",
                  f"* active threads per warp instruction {avg['smsp__thread_inst_executed_per_inst_executed.ratio']:.1f}",
                  ""]
        # stall breakdown from the source page
        src = ncu_csv(rep, "--page", "source", "--kernel-name", name.split("<")[0].split("::")[-1],
                      "--launch-count", "1")
        if len(src) > 2:
            h = src[1]
            body = [r for r in src[2:] if r and r[0].startswith("0x")]
            st = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
            tot = {h[i]: sum(float(r[i] or 0) for r in body) for i in st}
            allv = sum(tot.values()) or 1.0
            top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
            lines += ["* stall samples: " + ", ".join(f"{k[6:]} {100 * v / allv:.0f}%" for k, v in top), ""]
    open(out_md, "w").write("\n".join(lines) + "\n")
    if traffic_json:
        json.dump(traffic, open(traffic_json, "w"), indent=1, sort_keys=True)
        json.dump(metrics, open(traffic_json.replace("traffic", "ncu_metrics"), "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
