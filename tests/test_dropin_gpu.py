"""C++ drop-in (include/dgs_b200/dgs_gpu.hpp) beside the reference itself.

oracle/_ref/dropin_check is compiled in the build container from the
unmodified reference headers plus the drop-in header (oracle/Makefile
`dropin`), so every dgs::gpu entry point runs next to the dgs:: function it
replaces on identical inputs; the binary prints its error figures as JSON and
exits non-zero when any is outside tolerance (tolerances in
oracle/dropin_check.cpp's header).
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_check not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["ok"] is True
    assert rep["orders_mismatch"] == 0 and rep["merge_max_abs"] == 0
    assert rep["merge_backward_max_abs"] == 0 and rep["loss_grad_max_abs"] == 0
