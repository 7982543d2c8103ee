#!/bin/bash
# Bench under several values of one env switch, alternating twice: OUT=gpurun_out/<name> VAR=DGS_X VALS="0 1" [STEPS=20]
OUT=${OUT:-gpurun_out/abenv}
mkdir -p $OUT
for i in 1 2; do
  for v in $VALS; do
    export $VAR=$v
    timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > $OUT/b_${v}_$i.json 2> $OUT/b_${v}_$i.err
    python -c "import json;d=json.load(open('$OUT/b_${v}_$i.json'));s=d['step_stats']['per_view_avg'];print('$VAR=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items() if k.startswith('blend')}, 'subrounds', s['subrounds_bwd'], 'small', s['small_subrounds_bwd'])" || tail -5 $OUT/b_${v}_$i.err
  done
done
