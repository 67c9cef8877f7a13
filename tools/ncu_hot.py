"""Per-instruction view of one kernel in an ncu report (source page, SASS):
executed-instruction mix by opcode and the hottest stall sites.
usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
# one launch only: stop at the next header if several kernels matched
tot = 0
ops = Counter()
stall = Counter()
recs = []
for i, r in enumerate(rows):
    if r.get("Address") == "Address":
        break
    src = r["Source"].strip()
    n = int(r["Instructions Executed"] or 0)
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    tok = src.split()
    op = tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "")
    op = op.split(".")[0]
    ops[op] += n
    stall[op] += s
    tot += n
    recs.append((n, s, i, src))
print(f"total warp instructions executed: {tot:,}")
ts = sum(stall.values())
print("opcode mix (share of executed, share of stall samples):")
for op, n in ops.most_common(25):
    print(f"  {op:10s} {100 * n / tot:5.1f}%  {100 * stall[op] / max(ts, 1):5.1f}%")
print(f"top {top} stall sites:")
for n, s, i, src in sorted(recs, key=lambda x: -x[1])[:top]:
    print(f"  #{i:5d} exec {n:>12,} stall {s:>6} {src[:70]}")
