#!/bin/bash
# bench lines (3xTF32 and 1xTF32) + launch list + one ncu --set full capture
# usage: scripts/gpu_prof.sh <tag> <config> <kernel-regex> [skip]
TAG=$1; CFG=$2; KRE=$3; SKIP=${4:-3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 10 > $OUT/bench_3x.json 2>$OUT/bench.err; echo "bench3x rc=$?"
FCTN_TF32=1x timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 10 > $OUT/bench_1x.json 2>>$OUT/bench.err; echo "bench1x rc=$?"
CMD="python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
$CMD > $OUT/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
for f in $OUT/bench_3x.json $OUT/bench_1x.json; do python -c "
import json; d=json.load(open('$f')); print('$f', 'ms/sweep', d['ms_per_step'], 'frac', d['sweep_roofline']['frac']); [print('  ',k,v) for k,v in d['kernels'].items()]"; done
