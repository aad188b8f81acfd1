#!/bin/bash
# ncu launch-list A/B of env knobs (serialised per-kernel durations, so
# concurrent side-stream work does not confound the comparison):
# scripts/gpu_ncu_ab.sh <tag> <config> <kernel-regex> "ENV=.." ...
TAG=$1; CFG=$2; RE=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
i=0
for e in "$@"; do
  env $e timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file $OUT/l_$i.csv python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > $OUT/l_$i.log 2>&1
  echo "[$e]"; python tools/ncu_summary.py launches $OUT/l_$i.csv | grep -E "$RE|launches,"
  i=$((i+1))
done
