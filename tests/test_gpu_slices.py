"""GPU: the multi-rank manager path (row slices with a 10-row SSIM halo,
exchange buffers, per-slice loss sums) run as virtual slices on one B200 must
produce bit-identical gradients of every partial map, and the same loss, as
the whole-image path.  This covers everything of the N>1 step except the NCCL
transport itself (tests/test_multirank_cpu.py covers the plan across real
processes)."""
import numpy as np
import pytest

from conftest import Golden
from paper_2406_11836_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["g2_synth_kd2_default", "g4_synth_kd3_bg"])
@pytest.mark.parametrize("slices", [2, 3, 5])
def test_virtual_slices_match_whole_image(name, slices):
    g = Golden(name)
    s = g.splats()
    cam = g.camera()
    cfg = engine.train_config(kd_depth=g.args["kd"])
    out = {}
    for S in (1, slices):
        mgr = engine.Manager(s, cfg, engine.render_options(oracle=g.oracle_mode))
        mgr.ctx.set_virtual_slices(S)
        res = mgr.train_step([cam], g["step_target"][None], g.bg)
        maps = [mgr.ctx.dump_grad_maps(k, 0, cam) for k in range(g.subsets())]
        out[S] = (res, maps)
        mgr.close()
    (r1, m1), (rS, mS) = out[1], out[slices]
    assert abs(r1["loss"] - rS["loss"]) <= 1e-12 * max(1.0, abs(r1["loss"]))
    for k in range(g.subsets()):
        np.testing.assert_array_equal(m1[k][0], mS[k][0], err_msg=f"partial {k}")
        np.testing.assert_array_equal(m1[k][1], mS[k][1], err_msg=f"grad map {k}")
