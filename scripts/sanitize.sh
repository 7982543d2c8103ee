#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the small golden cases
# ("run compute-sanitizer ... on the small configs").  Logs -> $OUT.
OUT=${OUT:-gpurun_out/san}
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='test_full_train_step_matches_reference or test_partial_backward_gradients or test_partial_render_and_contributor_order'
K='g1_synth or g4_synth'
timeout 1500 $CS --tool memcheck --leak-check full --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "($SEL) and ($K)" > $OUT/memcheck.log 2>&1; echo "memcheck exit $?" >> $OUT/memcheck.log
timeout 1200 $CS --tool memcheck --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_edges.py -q -x > $OUT/memcheck_edges.log 2>&1; echo "memcheck edges exit $?" >> $OUT/memcheck_edges.log
timeout 1800 $CS --tool racecheck --racecheck-report all --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "test_full_train_step_matches_reference and g1_synth" > $OUT/racecheck.log 2>&1; echo "racecheck exit $?" >> $OUT/racecheck.log
timeout 1200 $CS --tool synccheck --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "test_full_train_step_matches_reference and g1_synth" > $OUT/synccheck.log 2>&1; echo "synccheck exit $?" >> $OUT/synccheck.log
for f in $OUT/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|exit|passed|failed" $f | tail -4; done
