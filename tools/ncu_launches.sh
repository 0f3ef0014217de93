#!/bin/bash
# per-launch durations of one small cfg2 far-field application (ncu, serialised, cold)
cd "$(dirname "$0")/.."
B=${1:-6}
python tools/prof_apply.py --batch $B > gpurun_out/prof_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:far_ --csv --log-file gpurun_out/launches_b$B.csv python tools/prof_apply.py --batch $B > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc=$?"
