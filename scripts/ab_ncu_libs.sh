#!/bin/bash
# Per-kernel ncu durations of one step for several library builds: LIBS="name=path ..." (path "-" = working tree)
OUT=${OUT:-gpurun_out/abncul}
RE=${RE:-'k_adam'}
mkdir -p $OUT
for spec in $LIBS; do
  name=${spec%%=*}; path=${spec#*=}
  if [ "$path" = "-" ]; then unset DGS_LIB; else export DGS_LIB=$PWD/$path; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k "regex:$RE" --csv \
     --log-file $OUT/l_$name.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCHARGS:---no-deterministic} --graph off > /dev/null 2>&1
  echo "== $name"; python scripts/launch_table.py $OUT/l_$name.csv | tail -${TAILN:-4}
done
