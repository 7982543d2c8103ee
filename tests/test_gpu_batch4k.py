"""GPU: config C4's step shape — a batch of 4 views at 3840x2160 with a 4-way
KD split (Manager::train_step, manager.hpp:313-386: per-view partials, merge,
loss x 1/B, merge adjoint; worker.hpp:86-127: GradBuffers summed over the
views, one Adam step) — against the unmodified reference run here
(oracle/_ref/ref_dump dump_batch) on a small synthetic scene.

At 4K the composite records take 4.2 GB per (subset, view) slot; the 16 slots
of this step exercise the record capacity guard (records where they fit, the
ring-replay backward where they would not).  Checks: the batch loss, every
subset's summed gradients (unmasked: conftest.grad_ok against the reference
and its exact-accumulation probe, 16 u B otherwise) through the GPU's own
per-subset backward, and the post-Adam parameters."""
import subprocess

import numpy as np
import pytest

from conftest import REF_DUMP, adam_lr_rows, oracle_step_bounds, post_adam_ok
from paper_2406_11836_b200 import engine

pytestmark = pytest.mark.gpu

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")
ARGS = dict(scene="synth", count=600, w=3840, h=2160, n_views=64, seed=31, kd=2, mode="oracle", view=0, perturb=7,
            batch_views="0,16,33,48")


def test_batch4_4k_train_step_matches_reference(tmp_path):
    if not REF_DUMP.exists():
        pytest.skip("oracle/_ref/ref_dump not built (needs /root/reference at build time)")
    argv = [str(REF_DUMP)] + [f"{k}={v}" for k, v in ARGS.items()] + ["dump_batch", "save_scene", "dump_table",
                                                                       f"out={tmp_path}"]
    subprocess.run(argv, check=True, capture_output=True, timeout=900)
    z = {f.stem: np.load(f) for f in tmp_path.glob("*.npy")}
    s = engine.Splats(z["scene_id"], z["scene_mu"], z["scene_log_scale"], z["scene_rotation"],
                      z["scene_opacity_logit"], z["scene_sh"])
    from capi_helpers import camera_from_record
    cams = [camera_from_record(r) for r in z["batch_cameras"]]
    targets = z["batch_targets"]
    B = len(cams)
    assert B == 4 and cams[0].width == 3840 and cams[0].height == 2160
    cfg = engine.train_config(kd_depth=ARGS["kd"], batch_size=B)
    mgr = engine.Manager(s, cfg, engine.render_options(oracle=True))
    res = mgr.train_step(cams, targets)
    # [1]: the reference's loss template in double on its own float images (its float
    # instantiation sums 8.3M terms per view sequentially in float: ~4x off at 4K).  The GPU
    # sums the reference's own float per-pixel terms (bit-exact) in double; the double
    # template also evaluates the SSIM maps in double: 2e-5 relative.
    want_loss = float(z["batch_loss"][1])
    assert abs(res["loss"] - want_loss) <= 2e-5 * abs(want_loss), (res["loss"], want_loss, float(z["batch_loss"][0]))
    off, ids = z["kd_member_off"], z["kd_member_ids"]
    members = [ids[off[k]:off[k + 1]].astype(np.int64) for k in range(len(off) - 1)]
    bounds = oracle_step_bounds(s, members, mgr.table.planes, z["batch_cameras"], targets, True)
    lrs = adam_lr_rows(cfg, s.sh_coeffs)
    for k in range(mgr.table.subset_count):
        p, _, _, step = mgr.ctx.store_subset(k, s.sh_coeffs)
        assert step == 1
        for f in FIELDS:
            want = z[f"k{k}_batch_adam_{f}"]
            ok, e, noisy = post_adam_ok(getattr(p, f).reshape(want.shape), want,
                                        z[f"k{k}_batch_grad_d_{f}"].reshape(want.shape), lrs[f],
                                        bound=bounds[k]["d_" + f])
            assert ok.all(), (k, f, int((~ok).sum()), float(e[~noisy].max()) if (~noisy).any() else 0.0)
    mgr.close()
