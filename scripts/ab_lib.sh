#!/bin/bash
# A/B the working-tree library against build/base (scripts/build_base.sh) on one box, alternating twice.
OUT=${OUT:-gpurun_out/ablib}
mkdir -p $OUT
for i in 1 2; do
  for mode in base new; do
    if [ $mode = base ]; then export DGS_LIB=$PWD/build/base/libdgs_b200.so; else unset DGS_LIB; fi
    timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > $OUT/b_${mode}_$i.json 2> $OUT/b_${mode}_$i.err
    python -c "import json;d=json.load(open('$OUT/b_${mode}_$i.json'));print('$mode', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items()})" || tail -5 $OUT/b_${mode}_$i.err
  done
done
