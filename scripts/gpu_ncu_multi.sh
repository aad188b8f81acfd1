#!/bin/bash
# ncu --set full of the first C launches matching a regex (after S skipped)
# usage: scripts/gpu_ncu_multi.sh <tag> <config> <kernel-regex> <skip> <count>
TAG=$1; CFG=$2; KRE=$3; SKIP=${4:-0}; CNT=${5:-6}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
$CMD > $OUT/plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s $SKIP -c $CNT -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
