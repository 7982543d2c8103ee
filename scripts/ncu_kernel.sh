#!/bin/bash
# ncu --set full (with source) of selected kernels of one C3 training step.
#   OUT=gpurun_out/x KREGEX='k_blend_bwd' SKIP=0 COUNT=1 scripts/ncu_kernel.sh
OUT=${OUT:-gpurun_out/ncu}
mkdir -p $OUT
KREGEX=${KREGEX:-k_blend_bwd}
timeout ${TMO:-1200} ncu --set full --import-source on --clock-control none -k "regex:${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-1} \
    -o $OUT/full python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${BENCH_ARGS:-} > $OUT/ncu.log 2>&1
ncu -i $OUT/full.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/full.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
for k in $(ncu -i $OUT/full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum 2>/dev/null | awk -F'","' 'NR>2{print $5}' | sed 's/(.*//' | sort -u); do
  ncu -i $OUT/full.ncu-rep --page source --csv --print-source cuda,sass -k "$k" > $OUT/src_$k.csv 2>/dev/null
done
ls -la $OUT
