for v in 0 1; do FHTB_FAR_ROWSUM=$v python tools/time_apply.py --reps 5; done > gpurun_out/ab_rowsum.jsonl 2>&1
cat gpurun_out/ab_rowsum.jsonl
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log
python bench.py --no-tasks --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_quick.json
