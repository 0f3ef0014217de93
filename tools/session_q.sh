for eps in 1e-3 1e-8 1e-12; do
for v in "0 4" "1 4" "2 1" "2 4"; do set -- $v; FHTB_FAR_ROWSUM=$1 FHTB_FAR_ROWSUM_MIN_PAIRS=$2 python tools/time_apply.py --reps 5 --eps $eps | cut -c1-170; done
done
