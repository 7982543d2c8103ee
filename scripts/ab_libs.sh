#!/bin/bash
# Bench several library builds on one box: LIBS="name=path ..." (path "-" = working tree), OUT=gpurun_out/<name>
OUT=${OUT:-gpurun_out/ablibs}
mkdir -p $OUT
for i in 1 2; do
  for spec in $LIBS; do
    name=${spec%%=*}; path=${spec#*=}
    if [ "$path" = "-" ]; then unset DGS_LIB; else export DGS_LIB=$PWD/$path; fi
    timeout 600 python bench.py --no-cpu-baseline --no-deterministic --steps ${STEPS:-20} > $OUT/b_${name}_$i.json 2> $OUT/b_${name}_$i.err
    python -c "import json;d=json.load(open('$OUT/b_${name}_$i.json'));s=d['step_stats']['per_view_avg'];print('$name', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items() if k.startswith('blend')}, 'evals', s['evals_fwd'], 'ovf', d['step_stats'].get('overflow_steps_timed'))" || tail -5 $OUT/b_${name}_$i.err
  done
done
