#!/bin/bash
# base build (eager) vs working tree eager vs working tree graph, alternating twice on one box
OUT=${OUT:-gpurun_out/abgraph}
mkdir -p $OUT
for i in 1 2; do
  for mode in base eager graph; do
    if [ $mode = base ]; then export DGS_LIB=$PWD/build/base/libdgs_b200.so; G="--graph off"; else unset DGS_LIB; fi
    if [ $mode = eager ]; then G="--graph off"; fi
    if [ $mode = graph ]; then G="--graph on"; fi
    timeout 600 python bench.py --no-cpu-baseline --no-deterministic --steps ${STEPS:-20} $G > $OUT/b_${mode}_$i.json 2> $OUT/b_${mode}_$i.err
    python -c "import json;d=json.load(open('$OUT/b_${mode}_$i.json'));print('$mode', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), (d.get('graph') or {}).get('ms_per_step_eager'), {k: round(v,3) for k,v in d['stages_ms_per_step'].items()})" || tail -3 $OUT/b_${mode}_$i.err
  done
done
