#!/bin/bash
# ncu --set full of the pass-2 kernel family (full and narrow-column forms) on
# a small cfg2 far-field application; the details / raw / source pages are
# exported to CSV on the box (the .ncu-rep itself can exceed the 64 MiB
# gpurun_out limit).  usage: tools/ncu_narrow.sh [kernel-regex] [count] [tag]
cd "$(dirname "$0")/.."
K=${1:-far_pass2}; C=${2:-4}; TAG=${3:-r2_pass2}
mkdir -p gpurun_out
python tools/prof_apply.py --batch 6 > gpurun_out/prof_plain.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -c $C -f \
  -o /tmp/$TAG python tools/prof_apply.py --batch 6 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_source.csv 2>/dev/null
ls -la /tmp/$TAG.ncu-rep gpurun_out/
