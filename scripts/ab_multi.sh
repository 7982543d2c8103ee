#!/bin/bash
# A/B/... of several prebuilt libraries on one box, alternating twice:
#   LIBS="base:build/base/libdgs_b200.so v2:build/v2/libdgs_b200.so new:" OUT=gpurun_out/x scripts/ab_multi.sh
# (an empty path = the working tree's library)
OUT=${OUT:-gpurun_out/abm}
mkdir -p $OUT
for i in 1 2; do
  for spec in $LIBS; do
    name=${spec%%:*}; lib=${spec#*:}
    if [ -n "$lib" ]; then export DGS_LIB=$PWD/$lib; else unset DGS_LIB; fi
    timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} ${BENCH_ARGS:-} > $OUT/b_${name}_$i.json 2> $OUT/b_${name}_$i.err
    python -c "import json;d=json.load(open('$OUT/b_${name}_$i.json'));print('$name', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items() if v})" || tail -5 $OUT/b_${name}_$i.err
  done
done
