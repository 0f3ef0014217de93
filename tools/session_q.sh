# far-field variant sweep (FHTB_FAR_VARIANT bit fields, fhtb_far.cu) on the cfg2 far field
base=$((4 + (1<<4) + (3<<20)))
for v in $base $((4 + (1<<4) + (1<<20))) $((4 + (1<<4) + (2<<20))) $((4 + (1<<4) + (4<<20))) $((4 + (2<<4) + (3<<20))) $((4 + (3<<4) + (3<<20))) $((4 + (4<<4) + (3<<20))) $((1 + (1<<4) + (3<<20))) $((5 + (1<<4) + (3<<20))); do
  FHTB_FAR_VARIANT=$v python tools/time_apply.py --reps 5 | cut -c1-120
done
