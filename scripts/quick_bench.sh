#!/bin/bash
# One bench run, summary line: OUT=gpurun_out/<name> [STEPS=20]
OUT=${OUT:-gpurun_out/qb}
mkdir -p $OUT
timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items()})" || tail -5 $OUT/bench.err
