#!/bin/bash
# One GPU call: bench line, kernel launch list of one training step, ncu --set full of the hot kernels.
# Outputs -> $OUT (default gpurun_out/prof).  Summarise with scripts/summarize_profile.py.
set -x
OUT=${OUT:-gpurun_out/prof}
mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; tail -c 3000 $OUT/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# skip the 31 matching launches of the target render and the warm-up step (whose first binning also sizes the pair buffers); capture the 15 of the timed step
timeout 1800 ncu --set full --import-source on --clock-control none \
    -k "regex:k_(preprocess|blend_fwd|blend_bwd_rec|grad_record|adam_stream4|loss|emit_pairs|merge)|Onesweep" \
    -s 31 -c 15 -o $OUT/full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu.log 2>&1
ls -la $OUT
