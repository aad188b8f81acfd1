#!/bin/bash
# ncu --set full (source-level stall sampling) of the c4 Cholesky and DFT kernels + a c4 launch list
TAG=${1:-cholprof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
for spec in "chol:k_chol:6" "dftinv:k_dft_inv:6" "dftfwd:k_dft_fwd:6"; do
  IFS=: read tag rx skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 -o $OUT/full_$tag $CMD > $OUT/ncu_full_$tag.log 2>&1
  echo "full $tag rc=$?"
  python tools/ncu_summary.py full $OUT/full_$tag.ncu-rep > $OUT/full_$tag.txt 2>&1
  ncu -i $OUT/full_$tag.ncu-rep --page source --csv > $OUT/src_$tag.csv 2>/dev/null
  python tools/ncu_stalls.py $OUT/src_$tag.csv 40 > $OUT/stalls_$tag.txt 2>&1
done
CMD="python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launch_c4.log 2>&1
python tools/ncu_summary.py launches $OUT/launches_c4.csv > $OUT/launches_c4.txt 2>&1
head -30 $OUT/launches_c4.txt
