base=$((4 + (1<<4) + (3<<20)))
for r in 1 2; do for v in $((base + (1<<19))) $base; do FHTB_FAR_VARIANT=$v python tools/time_apply.py --reps 5 | cut -c1-110; done; done
