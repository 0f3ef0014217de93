"""Far-field DRAM traffic per vector from an ncu CSV of
dram__bytes_read.sum / dram__bytes_write.sum over one far-field application
(tools/prof_apply.py --flags far --batch B), written to profiles/traffic.json.

    python tools/traffic.py dram.csv BATCH MODEL_BYTES_PER_VECTOR [out.json]
"""
import csv
import json
import sys


def main(path, batch, model, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = 0.0
    per = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[mi].startswith("dram__bytes"):
            continue
        name = r[ki]
        if "fhtb::" not in name or "table" in name or "twiddle" in name:
            continue
        v = float(r[vi].replace(",", ""))
        tot += v
        short = name.replace("fhtb::", "").replace("(int)", "").replace("(bool)", "").split("(")[0]
        per[short] = per.get(short, 0.0) + v
    res = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every far-field kernel of one "
                     "cfg2 far-field call (%d vectors), %s" % (batch, path),
           "far_field_dram_bytes_per_vector": tot / batch,
           "model_bytes_per_vector": model,
           "ratio_to_model": tot / batch / model,
           "per_kernel_bytes_per_vector": {k: v / batch for k, v in sorted(per.items(), key=lambda kv: -kv[1])}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), float(sys.argv[3]),
         sys.argv[4] if len(sys.argv) > 4 else "profiles/traffic.json")
