"""Per-source-line hot spots of one kernel in an ncu report (needs -lineinfo).
Usage: python tools/ncu_lines.py <report.ncu-rep> <kernel regex> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, kern, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    samples, insts = defaultdict(int), defaultdict(int)
    src = {}
    f, line, hdr = "?", None, None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            f = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            hdr = {h: i for i, h in enumerate(row)}
            continue
        if hdr is None or len(row) < 6:
            continue
        if row[0]:
            line = (f, int(row[0]))
            src[line] = row[1].strip()[:90]
            continue
        if line is None:
            continue
        try:
            samples[line] += int(row[4])
            insts[line] += int(row[7])
        except ValueError:
            pass
    tot = sum(samples.values()) or 1
    itot = sum(insts.values()) or 1
    print(f"total samples {tot}, warp instructions {itot}")
    for k, v in sorted(samples.items(), key=lambda kv: -kv[1])[:int(top)]:
        print(f"{100 * v / tot:5.1f}% smp {100 * insts[k] / itot:5.1f}% ins  {k[0]}:{k[1]}  {src.get(k, '')}")


if __name__ == "__main__":
    main(*sys.argv[1:])
