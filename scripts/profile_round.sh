#!/bin/bash
# One GPU call: bench line, kernel launch list, ncu --set full of the hot
# kernels of one training step (after the target render).  Outputs -> $OUT.
set -x
OUT=${OUT:-gpurun_out/r1}
mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; tail -c 4000 $OUT/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none \
    -k "regex:k_(preprocess|blend_fwd|blend_bwd|grad_record|adam_stream4|loss|emit_pairs)|Onesweep" -s 8 -c 12 \
    -o $OUT/full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu.log 2>&1
ls -la $OUT
