#!/bin/bash
# One GPU call: parity tests, a bench line, the kernel launch list, and an ncu
# --set full capture of the hot kernels of the first training step.
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; tail -c 3000 $OUT/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none \
    -k "regex:k_(preprocess|blend_fwd|blend_bwd|project_bwd_adam|loss|merge)" -s 2 -c 6 \
    -o $OUT/prof_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu.log 2>&1
ls -la $OUT
