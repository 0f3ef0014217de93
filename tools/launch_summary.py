"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total and mean time, share.

    python tools/launch_summary.py launches.csv
"""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        name = r[ki].replace("(int)", "").replace("(bool)", "").replace("fhtb::", "")
        name = name.split("(")[0] if "<" not in name else name[:name.index(">") + 1]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    return agg


if __name__ == "__main__":
    agg = load(sys.argv[1])
    tot = sum(t for _, t in agg.values())
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-60s %5d launches %10.1f us total %9.1f us avg %5.1f%%" % (name[:60], n, t, t / n, 100 * t / tot))
    print("total %.1f us" % tot)
