#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the ncu launch list of
# the same bench command, one `ncu --set full` capture of the top kernel.
# usage: scripts/gpu_evidence.sh <tag> <kernel-regex> [bench args...]
set -u
TAG=${1:-r01}; KRE=${2:-k_stream}; shift 2 || true
ARGS="$@"
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
python bench.py $ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $OUT/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $OUT/ncu_launch.log 2>&1
echo "launch-list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o $OUT/prof \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $OUT/ncu_full.log 2>&1
echo "ncu-full rc=$?"
tail -3 $OUT/pytest_gpu.log
