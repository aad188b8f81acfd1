#!/bin/bash
# ncu launch list (device time per kernel) for the given configs
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in "$@"; do
  CMD="python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
  $CMD > $OUT/plain_$c.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $CMD > $OUT/ncu_$c.log 2>&1
  echo "$c rc=$?"; python -c "
import json; d=json.loads(open('$OUT/plain_$c.log').read().strip().splitlines()[-1]); print('$c', 'ms/sweep', d['ms_per_step'], d['sweep_roofline'])"
  python tools/ncu_summary.py launches $OUT/launches_$c.csv | head -22
done
