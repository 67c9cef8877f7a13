"""Per-kernel times of one C2 frame from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file F`): the launches
between two consecutive k_project launches, in order.
usage: python tools/launch_frame.py LAUNCHES.csv [which-frame-from-end]"""
import csv
import sys


def frame(fn, back=2):
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    hdr = rows[0]
    i_n, i_v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ks = [(r[i_n], float(r[i_v])) for r in rows[1:]]
    idx = [i for i, (n, _) in enumerate(ks) if n.split("(")[0].split("<")[0].endswith("k_project")]
    a, b = idx[-back - 1], idx[-back]
    return ks[a:b]


if __name__ == "__main__":
    ks = frame(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
    for n, v in ks:
        print(f"{v / 1e3:9.1f} us  {n[:90]}")
    print(f"{sum(v for _, v in ks) / 1e6:9.3f} ms total, {len(ks)} launches")
