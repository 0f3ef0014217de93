for r in 1 2; do for v in 9 8; do FHTB_FAR_MIN_COLS=$v python tools/time_apply.py --reps 5 | cut -c1-110; done; done
