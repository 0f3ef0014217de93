#!/bin/bash
# Round-2 record: bench lines, launch list, DRAM traffic, ncu --set full of the far and near kernels.
cd "$(dirname "$0")/.."
O=gpurun_out/r2; mkdir -p $O
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench rc=$?"
python bench.py --workload sweep --gpus 1 --steps 3 --warmup 3 > $O/bench_sweep_g1.json 2> $O/bench_sweep.err; echo "sweep rc=$?"
python bench.py --workload single24 --gpus 1 --steps 3 --warmup 3 > $O/bench_single24_g1.json 2> $O/bench_single.err; echo "single rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
# launch list of the bench command (cfg2 steps only)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-tasks --no-e2e > $O/ncu_bench.log 2>&1; echo "launch list rc=$?"
# DRAM traffic of one far-field application (8 vectors)
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/dram_far.csv \
  python tools/prof_apply.py --batch 8 > $O/ncu_dram.log 2>&1; echo "dram rc=$?"
# full sets
bash tools/ncu_narrow.sh "far_pass2|far_pass1|far_rowsum" 9 r2_far > $O/ncu_far_full.log 2>&1
mv gpurun_out/r2_far_* $O/ 2>/dev/null
timeout 1200 ncu --set full --clock-control none -k regex:near_kernel -c 1 -f -o /tmp/r2_near python tools/prof_apply.py --flags near --batch 64 > $O/ncu_near.log 2>&1
ncu -i /tmp/r2_near.ncu-rep --page details --csv > $O/r2_near_details.csv
ncu -i /tmp/r2_near.ncu-rep --page raw --csv > $O/r2_near_raw.csv
ls -la $O
