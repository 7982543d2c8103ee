#!/bin/bash
# One GPU call: gpu tests + a 20-step bench; summary to stdout.  OUT=gpurun_out/<name>
OUT=${OUT:-gpurun_out/check}
mkdir -p $OUT
(timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log)
timeout 600 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest.log
python - "$OUT/bench.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
except Exception as e:
    print("bench failed", e); sys.exit(0)
print(round(d["ms_per_step"], 3), "ms/step", round(d["value"], 1), "Mpx/s", "e2e", round(d["e2e"]["value"], 1))
print(d["stages_ms_per_step"])
s = d["step_stats"]
print({k: s["per_view_avg"].get(k) for k in ("evals_fwd", "contribs_bwd", "subrounds_bwd", "replay_tiles_bwd")}, s.get("loss_last"))
PY
tail -3 $OUT/bench.err
