"""GPU: device-side repartition (dgs_repartition: snapshot, build_kdtree,
assign_subsets and migration on the B200) against the host path, which is
bit-exact with the reference (tests/test_host_cpu.py pins build_kdtree and
assign_subsets against the reference goldens).  Checked bit for bit: the KD
planes, every subset's member set, and every member's parameters and Adam
moments after migration (manager.hpp:389-482)."""
import numpy as np
import pytest

from conftest import Golden
from paper_2406_11836_b200 import engine

pytestmark = pytest.mark.gpu

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")


def _host_reference(mgr, depth):
    p, m, v, step = mgr.snapshot()
    table = engine.build_kdtree(p.mu, depth)
    members = engine.assign_subsets(table, p, float(mgr.options.truncation_radius))
    return p, m, v, step, table, members


def _check(mgr, ref):
    p, m, v, step, table, members = ref
    np.testing.assert_array_equal(mgr.table.planes, table.planes, err_msg="KD planes")
    assert mgr.table.subset_count == table.subset_count
    row = {int(i): j for j, i in enumerate(p.id)}
    for k in range(table.subset_count):
        gp, gm, gv, gstep = mgr.ctx.store_subset(k, p.sh_coeffs)
        assert gstep == step
        want = np.sort(p.id[members[k]])
        np.testing.assert_array_equal(np.sort(gp.id), want, err_msg=f"subset {k} members")
        sel = np.array([row[int(i)] for i in gp.id], np.int64)
        for src, got in ((p, gp), (m, gm), (v, gv)):
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(got, f), getattr(src, f)[sel], err_msg=f"subset {k} {f}")


@pytest.mark.parametrize("name", ["g2_synth_kd2_default", "g4_synth_kd3_bg"])
def test_device_repartition_after_training_matches_host(name):
    g = Golden(name)
    s = g.splats()
    cfg = engine.train_config(kd_depth=g.args["kd"])
    mgr = engine.Manager(s, cfg, engine.render_options(oracle=g.oracle_mode))
    cam = g.camera()
    for _ in range(2):  # centres move, shared replicas drift apart (sync off)
        mgr.train_step([cam], g["step_target"][None], g.bg)
    ref = _host_reference(mgr, g.args["kd"])
    mgr.repartition(device=True)
    _check(mgr, ref)
    # and the step still runs on the migrated state
    res = mgr.train_step([cam], g["step_target"][None], g.bg)
    assert np.isfinite(res["loss"])
    mgr.close()


def test_device_repartition_changes_depth_at_scale():
    s = engine.synth_splats(200_000, seed=31, sh_degree=3)
    cfg = engine.train_config(kd_depth=1)
    mgr = engine.Manager(s, cfg, engine.render_options())
    mgr.config.kd_depth = 3
    ref = _host_reference(mgr, 3)
    mgr.repartition(device=True)
    assert mgr.table.subset_count == 8
    _check(mgr, ref)
    mgr.close()
