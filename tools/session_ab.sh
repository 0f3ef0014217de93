# A/B of the fused narrow-row forms (far_rowsum 0 / 1 / 2) on the cfg2 far field,
# then the GPU tests under the requested setting (default: library default)
for v in 0 1 2; do FHTB_FAR_ROWSUM=$v python tools/time_apply.py --reps 5; done > gpurun_out/ab_rowsum.jsonl 2>&1
cut -c1-200 gpurun_out/ab_rowsum.jsonl
FHTB_FAR_ROWSUM=${1:-2} python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log
FHTB_FAR_ROWSUM=${1:-2} bash tools/ncu_launches.sh 6
