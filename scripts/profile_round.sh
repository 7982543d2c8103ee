#!/bin/bash
# One GPU call: bench line, kernel launch list of one training step, ncu --set full of the hot kernels.
# Outputs -> $OUT (default gpurun_out/prof).  Summarise with scripts/summarize_profile.py.
set -x
OUT=${OUT:-gpurun_out/prof}
mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; tail -c 3000 $OUT/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-deterministic --graph off > /dev/null 2>&1
# capture the hot kernels of the last (timed) step: skip every matching launch before its preprocess
RE='k_(preprocess|blend_fwd|blend_bwd_rec|grad_record|adam_stream4|loss|emit_pairs|merge)|Onesweep'
read SKIP COUNT < <(python - "$OUT/launches.csv" "$RE" <<'PY'
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i0]; ki, ii = h.index("Kernel Name"), h.index("ID")
seen, names = set(), []
for r in rows[i0 + 1:]:
    if len(r) == len(h) and r[ii] not in seen:
        seen.add(r[ii]); names.append(r[ki])
last = max(i for i, n in enumerate(names) if "k_preprocess" in n)
rx = re.compile(sys.argv[2])
m = [bool(rx.search(n)) for n in names]
print(sum(m[:last]), sum(m[last:]))
PY
)
echo "ncu full: skip $SKIP, capture $COUNT"
timeout 1800 ncu --set full --import-source on --clock-control none -k "regex:$RE" \
    -s $SKIP -c $COUNT -o $OUT/full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-deterministic --graph off > $OUT/ncu.log 2>&1
ls -la $OUT
