"""Per-kernel limiter evidence from an ncu --set full details CSV (one row per
captured launch): duration, DRAM / L1-TEX / SM throughput, issue activity,
occupancy.  Written to profiles/far_kernel_bounds.json for bench.py.

    python tools/kernel_bounds.py details.csv [out.json]
"""
import csv
import json
import sys

WANT = {"Duration": "duration", "DRAM Throughput": "dram_pct", "L1/TEX Cache Throughput": "l1tex_pct",
        "Compute (SM) Throughput": "sm_pct", "Issue Slots Busy": "issue_pct",
        "Registers Per Thread": "registers", "Achieved Occupancy": "occupancy_pct",
        "Eligible Warps Per Scheduler": "eligible_warps"}


def main(path, out):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = {}
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in WANT:
            continue
        d = launches.setdefault(r[ii], {"kernel": r[ki].split("(")[0].replace("void ", "")})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "Duration":
            v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
            d["duration_us"] = v
        else:
            d[WANT[r[mi]]] = v
    res = {"source": path, "launches": list(launches.values())}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/far_kernel_bounds.json")
