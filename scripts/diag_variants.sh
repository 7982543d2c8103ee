#!/bin/bash
# Time the C3 step under each value of an environment knob: VAR=DGS_BWD_MINB VALS="2 3 4 6"
OUT=${OUT:-gpurun_out/var}; mkdir -p $OUT
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/b_$v.json 2>/dev/null
  python -c "import json,sys;d=json.load(open('$OUT/b_$v.json'));print('$VAR=$v', round(d['ms_per_step'],3), d['stages_ms_per_step'])"
done
