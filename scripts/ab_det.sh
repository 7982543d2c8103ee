#!/bin/bash
# A/B of the deterministic=1 step (working tree vs build/base), alternating twice on one box.
OUT=${OUT:-gpurun_out/abdet}
mkdir -p $OUT
for i in 1 2; do
  for mode in base new; do
    if [ $mode = base ]; then export DGS_LIB=$PWD/build/base/libdgs_b200.so; else unset DGS_LIB; fi
    timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > $OUT/b_${mode}_$i.json 2> $OUT/b_${mode}_$i.err
    python -c "import json;d=json.load(open('$OUT/b_${mode}_$i.json'));m=d['deterministic_mode'];print('$mode', round(d['ms_per_step'],3), round(m['ms_per_step'],3), {k: round(v,3) for k,v in (m.get('stages_ms_per_step_eager') or {}).items()})" || tail -5 $OUT/b_${mode}_$i.err
  done
done
