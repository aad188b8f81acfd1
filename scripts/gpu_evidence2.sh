#!/bin/bash
# Round evidence for c4 (headline) and c5: bench lines, launch lists, ncu --set full of the top kernels.
# usage: scripts/gpu_evidence2.sh <tag>
TAG=${1:-ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
python bench.py --config c5 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?"
for c in c4 c5; do
  CMD="python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
  timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/launches_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1
  echo "launches $c rc=$?"
done
full() {  # tag config regex skip
  CMD="python bench.py --config $2 --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$3" -s $4 -c 1 -o $OUT/full_$1 $CMD > $OUT/ncu_full_$1.log 2>&1
  echo "full $1 rc=$?"
  ncu -i $OUT/full_$1.ncu-rep --page raw --csv > $OUT/full_$1_raw.csv 2>/dev/null
}
full c4_zpass c4 "k_stream_tsp" 2
full c4_compose c4 "k_compose_tma" 2
full c5_join c5 "k_join_tc" 2
full c5_stream c5 "k_stream_ts<" 2
full c5_compose c5 "k_compose_t" 1
