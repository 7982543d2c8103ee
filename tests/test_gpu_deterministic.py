"""GPU: TrainConfig::deterministic = 1 — "fixed-order reductions" (optim.hpp:33;
parallel.hpp:23-55: the reference's per-chunk GradBuffers merged in chunk
order, so a step is bitwise reproducible).

The B200 backward sums every member's 9 pixel-space adjoints as fixed point
in units of 2^-72 (blend_bwd.cu acc_add / to_fixed: two 64-bit words per
value, plain integer atomics): integer addition is associative, so the totals
do not depend on the order the atomics land in, and they are exact up to one
rounding (2^-73) per warp sub-round.

* Two runs of the same training steps are bitwise identical (gradients,
  post-Adam parameters and moments), on a scene large enough for heavy atomic
  contention, both backward paths (record walk and ring replay).
* Gradient parity against the reference without a noise mask, for both modes,
  is tests/test_gpu_parity.py::test_partial_backward_gradients.
"""
import numpy as np
import pytest

from paper_2406_11836_b200 import engine
from test_gpu_parity import PARAM_FIELDS

pytestmark = pytest.mark.gpu


def _run(s, cam, target, det, steps=2, records=True):
    cfg = engine.train_config(kd_depth=1, deterministic=det)
    mgr = engine.Manager(s, cfg, engine.render_options(grad_skip_eps=0.0))
    mgr.ctx.set_backward_records(records)
    for _ in range(steps):
        mgr.train_step([cam], target[None])
    out = [mgr.ctx.store_subset(k, s.sh_coeffs) for k in range(mgr.table.subset_count)]
    g2d = [mgr.ctx.dump_pixel_grads(k) for k in range(mgr.table.subset_count)]
    mgr.close()
    return out, g2d


@pytest.mark.parametrize("records", [True, False], ids=["record-walk", "ring-replay"])
def test_deterministic_steps_bitwise_identical(records):
    s = engine.synth_splats(200_000, seed=11, sh_degree=3)
    cam = engine.ring_camera(640, 360, 3, n_views=64)
    tm = engine.Manager(s, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
    target, _ = tm.render(cam)
    tm.close()
    s = engine.perturb(s, 5)
    a, ga = _run(s, cam, target, 1, records=records)
    b, gb = _run(s, cam, target, 1, records=records)
    for k in range(len(a)):
        for x, y in zip(ga[k], gb[k]):
            np.testing.assert_array_equal(x, y, err_msg=f"pixel-space adjoints, subset {k}")
        for which in range(3):  # params, m, v
            for f in PARAM_FIELDS:
                np.testing.assert_array_equal(getattr(a[k][which], f), getattr(b[k][which], f),
                                              err_msg=f"subset {k} {('p', 'm', 'v')[which]}.{f}")
    assert np.abs(ga[0]).max() > 0
