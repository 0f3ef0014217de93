"""Copy the outputs of tools/session_final.sh (gpurun_out/r2/) into
profiles/round2/ and refresh profiles/traffic.json, far_kernel_bounds.json
and near_kernel_bounds.json from them.

    python tools/collect_round2.py
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "r2")
DST = os.path.join(ROOT, "profiles", "round2")
os.makedirs(DST, exist_ok=True)
for f in ("bench_cfg2.json", "bench_sweep_g1.json", "bench_single24_g1.json", "bench_reference.json",
          "launches_bench.csv", "dram_far.csv", "r2_far_details.csv", "r2_far_raw.csv", "r2_far_lines.txt",
          "r2_near_details.csv", "r2_near_raw.csv"):
    p = os.path.join(SRC, f)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(DST, f))
bench = json.loads(open(os.path.join(SRC, "bench_cfg2.json")).read().strip().splitlines()[-1])
model = bench["roofline"]["far_field"]["model_bytes_per_vector"]
py = sys.executable
subprocess.run([py, os.path.join(ROOT, "tools", "traffic.py"), os.path.join(DST, "dram_far.csv"), "8", str(model),
                os.path.join(ROOT, "profiles", "traffic.json")], check=True, stdout=subprocess.DEVNULL)
subprocess.run([py, os.path.join(ROOT, "tools", "kernel_bounds.py"), os.path.join(DST, "r2_far_details.csv"),
                os.path.join(ROOT, "profiles", "far_kernel_bounds.json")], check=True, stdout=subprocess.DEVNULL)
subprocess.run([py, os.path.join(ROOT, "tools", "kernel_bounds.py"), os.path.join(DST, "r2_near_details.csv"),
                os.path.join(ROOT, "profiles", "near_kernel_bounds.json")], check=True, stdout=subprocess.DEVNULL)
out = subprocess.run([py, os.path.join(ROOT, "tools", "launch_summary.py"), os.path.join(DST, "launches_bench.csv")],
                     check=True, capture_output=True, text=True).stdout
open(os.path.join(DST, "launches_bench_summary.txt"), "w").write(out)
print(out)
print(open(os.path.join(ROOT, "profiles", "traffic.json")).read())
