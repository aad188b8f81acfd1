#!/bin/bash
# one ncu --set full capture + source/details export
# usage: scripts/gpu_ncu1.sh <tag> <config> <kernel-regex> <skip>
TAG=$1; CFG=$2; KRE=$3; SKIP=${4:-3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
$CMD > $OUT/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KRE" -s $SKIP -c 1 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/prof.ncu-rep --page source --csv > $OUT/source.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
