#!/bin/bash
# usage: tools/sweep.sh "ENV1=a ENV2=b" "ENV1=c" ... -- [time_apply args]
# runs tools/time_apply.py once per environment setting (separate processes,
# so grids are rebuilt with the options), one JSON line each
cfgs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do cfgs+=("$1"); shift; done
[ "$1" == "--" ] && shift
for c in "${cfgs[@]}"; do
  env $c timeout 300 python tools/time_apply.py "$@" || echo "{\"env\": \"$c\", \"failed\": true}"
done
