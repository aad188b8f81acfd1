#!/bin/bash
# A/B of env knobs on one config: scripts/gpu_env_ab.sh <tag> <config> "ENV=.. ENV2=.." ...
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 10 > $OUT/ab_$i.json 2>$OUT/ab_$i.err
  python -c "
import json; d=json.load(open('$OUT/ab_$i.json')); k=d['kernels']; print('[$e]', 'ms/sweep', d['ms_per_step'], {n: round(v.get('ms_per_step', 0), 3) for n, v in k.items()})" || tail -3 $OUT/ab_$i.err
  i=$((i+1))
done
