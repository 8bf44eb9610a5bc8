"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: count, total and mean time.  Usage: python profiles/launch_summary.py X.csv"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        k = r[ki].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
        tot += v
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:5d} {t:9.1f} us {t / c:8.1f} us/launch {100 * t / tot:5.1f} %  {k}")
    print(f"total {tot:.1f} us over {sum(c for c, _ in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
