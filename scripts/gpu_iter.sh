#!/bin/bash
# Fast iteration on the GPU box: GPU tests + one bench line per listed config.
# usage: scripts/gpu_iter.sh <tag> [configs...]
TAG=${1:-iter}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
tail -15 $OUT/pytest_gpu.log
for c in "$@"; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$?"; cat $OUT/bench_$c.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], 'ms/sweep', d['ms_per_step'], 'frac', d['sweep_roofline']['frac']); [print('  ',k,v) for k,v in d['kernels'].items()]" 2>/dev/null || tail -5 $OUT/bench_$c.err
done
