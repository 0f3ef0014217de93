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
# hot source lines per captured kernel (stall samples / executed instructions per line)
for kn in "far_pass2_kernel<2048, 16, 0" "far_pass2_kernel<512" "far_pass2_kernel<2048, 16, 2" "far_pass1" "far_rowsum_kernel" "far_rowsum2_kernel<256" "far_rowsum2_kernel<1024"; do
  echo "== $kn"; python tools/ncu_lines.py /tmp/$TAG.ncu-rep "$kn" 45
done > gpurun_out/${TAG}_lines.txt 2>&1
ls -la /tmp/$TAG.ncu-rep gpurun_out/
