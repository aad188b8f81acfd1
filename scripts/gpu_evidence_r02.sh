#!/bin/bash
# Round-2 evidence: bench lines c1..c5 (c4 = the default line with e2e and the
# reference CPU baseline), the reference arm, launch lists for c4 / c5 and
# ncu --set full captures of the top kernels.  usage: scripts/gpu_evidence_r02.sh <tag>
TAG=${1:-ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 rc=$?"
for c in c5 c3 c2 c1; do python bench.py --config $c --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"; done
python bench.py --impl reference > $OUT/reference_arm.json 2> $OUT/reference_arm.err; echo "reference rc=$?"
for c in c4 c5 c3; do
  CMD="python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
  timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/launches_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1
  echo "launches $c rc=$?"
  python tools/ncu_summary.py launches $OUT/launches_$c.csv > $OUT/launches_$c.txt 2>&1
done
full() {  # tag config regex skip
  CMD="python bench.py --config $2 --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$3" -s $4 -c 1 -o $OUT/full_$1 $CMD > $OUT/ncu_full_$1.log 2>&1
  echo "full $1 rc=$?"
  python tools/ncu_summary.py full $OUT/full_$1.ncu-rep > $OUT/full_$1.txt 2>&1
}
full c4_zpass c4 "k_stream_tsp" 2
full c4_compose c4 "k_compose_tma" 2
full c4_chol c4 "k_chol" 6
full c5_join c5 "k_join_tc" 4
full c5_stream c5 "k_stream_tsw" 2
full c5_compose c5 "k_compose" 1
full c3_stream c3 "k_stream_dmma" 4
