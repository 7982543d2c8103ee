#!/bin/bash
# Per-kernel durations of one training step with and without an env switch (ENVSW), under ncu.
OUT=${OUT:-gpurun_out/abncu}
RE=${RE:-'k_(preprocess|blend|loss|grad_record|adam|merge)|Onesweep|k_emit'}
mkdir -p $OUT
for mode in off on; do
  if [ $mode = on ]; then EX="env $ENVSW"; else EX=""; fi
  timeout 600 $EX ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
     --clock-control none -k "regex:$RE" --csv \
     --log-file $OUT/l_$mode.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCHARGS:---no-deterministic} --graph off > /dev/null 2>&1
  echo "== $ENVSW $mode"; python scripts/launch_table.py $OUT/l_$mode.csv | tail -${TAILN:-40}
done
