#!/bin/bash
# A/B one env switch on the default bench: OUT=gpurun_out/<name> VAR=DGS_X [STEPS=20]
OUT=${OUT:-gpurun_out/ab}
mkdir -p $OUT
for mode in new legacy; do
  if [ $mode = legacy ]; then export $VAR=1; else unset $VAR; fi
  timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > $OUT/bench_$mode.json 2> $OUT/bench_$mode.err
  python -c "import json;d=json.load(open('$OUT/bench_$mode.json'));print('$mode', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items()})" || tail -5 $OUT/bench_$mode.err
done
