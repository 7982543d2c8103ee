"""GPU: BASELINE.json configs 1 and 2 as parity cases.

* C1 — 100k synthetic splats, one 800x800 view, single subset: one full
  training step (partial render, merge, L1 + D-SSIM, merge adjoint, backward,
  Adam) against the C restatement of the reference (oracle/dgs_oracle.c,
  pinned bit-exact to the reference's own goldens in tests/test_oracle_cpu.py)
  run through the same call sequence (manager.hpp:313-386).
* C2 — 1M splats, 1920x1080, 2-way KD split, oracle options: the per-subset
  partials and the merged image equal the reference's own partial_render,
  merge and render_view on sampled rows (ref_dump dump_rows; the reference's
  merge == monolithic check, test_engine.cpp:171-203, 1e-4 in float).
* The three ways targets reach the step (pageable host, pinned host,
  device-resident) give the same loss.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_binding as ob
from conftest import adam_lr_rows, oracle_gradients, post_adam_ok
from paper_2406_11836_b200 import engine

pytestmark = pytest.mark.gpu

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")


def test_c1_train_step_matches_oracle():
    gt = engine.synth_splats(100_000, seed=11, sh_degree=3)
    cam = engine.ring_camera(800, 800, 0, n_views=64)
    tmgr = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
    target, _ = tmgr.render(cam)
    tmgr.close()
    target = np.ascontiguousarray(target, np.float32)
    s = engine.perturb(gt, 5)
    bg = np.zeros(3, np.float32)
    H, W = cam.height, cam.width

    # GPU: Manager::train_step (K = 1)
    cfg = engine.train_config(kd_depth=0)
    mgr = engine.Manager(s, cfg, engine.render_options(grad_skip_eps=0.0))
    res = mgr.train_step([cam], target[None], bg)
    p, _, _, step = mgr.ctx.store_subset(0, s.sh_coeffs)
    mgr.close()
    assert step == 1

    # oracle: the same sequence on the CPU
    o = ob.opts(False, grad_skip_eps=0.0)
    ocam = ob.cam_of(cam.record())
    sub = ob.Sub()
    sub.n = 0
    sc = ob.Scene(s)
    ct = np.zeros((H, W, 4), np.float32)
    assert ob.lib().orc_partial_render(C.byref(sc.c), C.byref(sub), C.byref(ocam), C.byref(o), ob.p(ct), 0, None,
                                       None) == 0
    order = np.zeros((H, W, 1), np.uint16)
    count = np.zeros((H, W), np.uint16)
    ob.lib().orc_pixel_orders((ob.Sub * 1)(sub), 1, C.byref(ocam), ob.p(order), ob.p(count))
    rgb = np.zeros((H, W, 3), np.float32)
    ob.lib().orc_merge(ob.p(ct), ob.p(order), ob.p(count), 1, W, H, ob.p(bg), ob.p(rgb), None)
    grad = np.zeros_like(rgb)
    means = np.zeros(3, np.float32)
    loss = ob.lib().orc_loss(ob.p(rgb), ob.p(target), W, H, C.c_float(cfg.lambda_ssim), ob.p(grad), ob.p(means))
    assert abs(res["loss"] - loss) <= 1e-4 * max(1.0, abs(loss)), (res["loss"], loss)
    gct = np.zeros((1, H, W, 4), np.float32)
    ob.lib().orc_merge_backward(ob.p(ct), ob.p(order), ob.p(count), 1, W, H, ob.p(grad), ob.p(bg), ob.p(gct))
    gr, garr = ob.empty_grads(s.n, s.sh_coeffs)
    assert ob.lib().orc_partial_backward(C.byref(sc.c), C.byref(sub), C.byref(ocam), C.byref(o), ob.p(gct[0]),
                                         C.byref(gr)) == 0
    want = s.copy()
    rows = 11 + 3 * s.sh_coeffs
    mm = np.zeros((s.n, rows), np.float32)
    vv = np.zeros((s.n, rows), np.float32)
    ob.lib().orc_adam(C.c_int64(s.n), s.sh_coeffs, ob.p(want.mu), ob.p(want.log_scale), ob.p(want.rotation),
                      ob.p(want.opacity_logit), ob.p(want.sh), ob.p(mm), ob.p(vv), C.byref(gr),
                      C.c_double(cfg.lr_position_start), C.c_double(cfg.lr_scale), C.c_double(cfg.lr_rotation),
                      C.c_double(cfg.lr_opacity), C.c_double(cfg.lr_sh_dc), C.c_double(cfg.lr_sh_rest),
                      C.c_double(cfg.adam_beta1), C.c_double(cfg.adam_beta2), C.c_double(cfg.adam_eps),
                      C.c_uint64(1))

    # members by id (the subset stores them in its own order)
    row = {int(i): j for j, i in enumerate(s.id)}
    sel = np.array([row[int(i)] for i in p.id], np.int64)
    lrs = adam_lr_rows(cfg, s.sh_coeffs)
    assert np.abs(garr["d_mu"]).max() > 0
    bound = oracle_gradients(s, np.zeros((0, 5), np.float32), cam.record(), False, gct[0], bound=True,
                             grad_skip_eps=0.0)
    for f in FIELDS:
        got = getattr(p, f)
        ok, e, noisy = post_adam_ok(got, getattr(want, f)[sel], garr["d_" + f][sel], lrs[f],
                                    bound=bound["d_" + f][sel])
        assert ok.all(), (f, float(e[~noisy].max()) if (~noisy).any() else 0.0, int((~ok).sum()))


C2_ROWS = (0, 137, 300, 539, 540, 777, 950, 1079)


def ref_rows(tmp_path, count, width, height, kd, rows, mode="oracle"):
    """The unmodified reference (oracle/_ref/ref_dump dump_rows): render_view,
    every subset's partial_render and their merge on sampled rows."""
    import subprocess
    from conftest import REF_DUMP
    if not REF_DUMP.exists():
        pytest.skip("oracle/_ref/ref_dump not built (needs /root/reference at build time)")
    argv = [str(REF_DUMP), "scene=synth", f"count={count}", f"w={width}", f"h={height}", "n_views=64", "seed=11",
            f"kd={kd}", "view=0", f"mode={mode}", "dump_rows", "rows=" + ",".join(map(str, rows)), f"out={tmp_path}"]
    subprocess.run(argv, check=True, capture_output=True)
    return {f.stem: np.load(f) for f in tmp_path.glob("rows_*.npy")}


def test_c2_kd_split_matches_reference_render(tmp_path):
    """C2 (1M splats, 1920x1080, 2-way KD split, oracle options) against the
    reference itself: every subset's partial (C_k, T_k), the merged image and
    the reference's monolithic render_view on sampled rows, within 1e-4
    (test_engine.cpp:171-203); and the GPU's own split == unsplit render."""
    s = engine.synth_splats(1_000_000, seed=11, sh_degree=3)
    cam = engine.ring_camera(1920, 1080, 0, n_views=64)
    ro = engine.render_options(oracle=True)
    ref = ref_rows(tmp_path, 1_000_000, 1920, 1080, 1, C2_ROWS)
    rows = list(C2_ROWS)
    out = {}
    for depth in (0, 1):
        mgr = engine.Manager(s, engine.train_config(kd_depth=depth), ro)
        if depth == 1:
            assert mgr.table.subset_count == 2
            for k in range(2):
                ct = mgr.ctx.render_partial(k, cam)[rows]
                ec = np.abs(ct[..., :3] - ref[f"rows_k{k}_C"]).max()
                et = np.abs(ct[..., 3] - ref[f"rows_k{k}_T"]).max()
                assert ec <= 1e-4 and et <= 1e-4, (k, float(ec), float(et))
        out[depth] = mgr.render(cam)
        mgr.close()
    (rgb0, t0), (rgb1, t1) = out[0], out[1]
    assert t0.min() < 0.5  # the view sees the scene
    for rgb, t in ((rgb1, t1), (rgb0, t0)):
        assert np.abs(rgb[rows] - ref["rows_merged_C"]).max() <= 1e-4
        assert np.abs(t[rows] - ref["rows_merged_T"]).max() <= 1e-4
        assert np.abs(rgb[rows] - ref["rows_render_C"]).max() <= 1e-4
        assert np.abs(t[rows] - ref["rows_render_T"]).max() <= 1e-4
    assert np.abs(rgb1 - rgb0).max() <= 1e-4, float(np.abs(rgb1 - rgb0).max())
    assert np.abs(t1 - t0).max() <= 1e-4, float(np.abs(t1 - t0).max())


def test_host_target_paths_agree():
    """Pinned host targets (direct H2D) and pageable ones (staged through
    pinned memory by helper threads) give the same step as device-resident
    targets: the forward and the loss are deterministic, so the loss is
    bit-identical."""
    import torch

    s = engine.synth_splats(20_000, seed=3, sh_degree=3)
    cam = engine.ring_camera(320, 180, 2, n_views=64)
    rng = np.random.default_rng(1)
    target = rng.random((1, 180, 320, 3), dtype=np.float32)
    pinned = torch.empty(target.size, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = target.reshape(-1)
    losses = []
    for mode in ("pageable", "pinned", "device"):
        mgr = engine.Manager(s, engine.train_config(kd_depth=1), engine.render_options())
        if mode == "pageable":
            r = mgr.train_step([cam], target)
        elif mode == "pinned":
            r = mgr.train_step([cam], pinned.numpy().reshape(target.shape))
        else:
            tdev = mgr.ctx.upload_targets(target)
            r = mgr.train_step([cam], None, targets_device_ptr=tdev)
        losses.append(r["loss"])
        mgr.close()
    assert losses[0] == losses[1] == losses[2], losses
