set -x
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
for pr in 11 12; do FHTB_FAR_PRUNE_ROWS=$pr python tools/time_apply.py --reps 5; done > gpurun_out/ab_prune_rows.jsonl 2>&1
python bench.py --workload sweep --gpus 1 --steps 3 --warmup 1 > gpurun_out/bench_sweep_g1.json 2> gpurun_out/bench_sweep_g1.err; echo "sweep rc=$?"
python bench.py --workload single24 --gpus 1 --steps 3 --warmup 1 > gpurun_out/bench_single24_g1.json 2> gpurun_out/bench_single24_g1.err; echo "single rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
bash tools/sanitize.sh; echo "sanitize done"
