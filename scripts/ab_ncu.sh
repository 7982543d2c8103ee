#!/bin/bash
# Per-kernel durations of one training step for base (build/base) and the working tree, under ncu.
OUT=${OUT:-gpurun_out/abncu}
RE=${RE:-'k_(preprocess|blend|loss|grad_record|adam|merge)|Onesweep|k_emit'}
mkdir -p $OUT
for mode in base new; do
  if [ $mode = base ]; then export DGS_LIB=$PWD/build/base/libdgs_b200.so; else unset DGS_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k "regex:$RE" --csv \
     --log-file $OUT/l_$mode.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCHARGS:---no-deterministic} --graph off > /dev/null 2>&1
  echo "== $mode"; python scripts/launch_table.py $OUT/l_$mode.csv | tail -${TAILN:-40}
done
