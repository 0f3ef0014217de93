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
    def family(k):
        if "far_pass1" in k:
            return "far_pass1"
        if "far_rowsum_fin" in k:
            return "far_rowsum_fin"
        if "far_rowsum" in k:
            return "far_rowsum"
        if "far_rowdot" in k:
            return "far_rowdot"
        if "far_reduce" in k:
            return "far_reduce"
        if "colgen" in k:
            return "far_narrow_cols"
        if "far_pass2" in k:
            args = k[k.index("<") + 1:k.index(">")].replace(" ", "").split(",") if "<" in k else []
            return "far_narrow_cols" if len(args) > 2 and args[2] == "2" else "far_pass2"
        return "other"

    fam = {}
    for k, v in per.items():
        fam[family(k)] = fam.get(family(k), 0.0) + v / batch
    res = {"per_family_dram_bytes_per_vector": fam,
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every far-field kernel of one "
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
