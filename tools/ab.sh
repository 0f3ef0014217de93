#!/bin/bash
# Alternate tools/time_apply.py between library builds, R rounds each:
#   tools/ab.sh R lib1 lib2 ... -- [time_apply args]     (lib "tree" = in-tree build)
R=$1; shift
libs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done
[ "$1" == "--" ] && shift
for r in $(seq 1 $R); do
  for l in "${libs[@]}"; do
    if [ "$l" == "tree" ]; then lib=""; else lib="$l"; fi
    FHTB_LIB=$lib timeout 300 python tools/time_apply.py "$@" | sed "s|^{|{\"lib\": \"$l\", |"
  done
done
