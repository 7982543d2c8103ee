"""GPU: edge cases of the training step — a view that culls every splat,
KD leaves with no members, image sizes that are not multiples of the 16-pixel
tile, a single splat, the reference's zero-quaternion error
(math.hpp:36-37 -> std::domain_error), and the two capacity fallbacks: the
exact kernels for pixels whose (t, id) reorder ring overflows, and the
ordered-ring replay for tiles whose composite records overflow."""
import ctypes as C

import numpy as np
import pytest

import oracle_binding as ob
from paper_2406_11836_b200 import engine

pytestmark = pytest.mark.gpu

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")


def _away(cam):
    """The same camera moved 100 units back along its axis: every splat lies behind it."""
    c = engine.Camera.from_record(cam.record())
    c.t_wc[2] = c.t_wc[2] - 100.0
    return c


def test_view_that_culls_everything():
    s = engine.synth_splats(3000, seed=4, sh_degree=3)
    cam = _away(engine.ring_camera(96, 64, 1, n_views=64))
    mgr = engine.Manager(s, engine.train_config(kd_depth=1), engine.render_options())
    rgb, t = mgr.render(cam, bg=(0.25, 0.5, 0.75))
    np.testing.assert_array_equal(t, np.ones_like(t))
    np.testing.assert_array_equal(rgb, np.broadcast_to(np.float32([0.25, 0.5, 0.75]), rgb.shape))
    before = [mgr.ctx.store_subset(k, s.sh_coeffs)[0] for k in range(mgr.table.subset_count)]
    target = np.random.default_rng(0).random((1, 64, 96, 3), dtype=np.float32)
    res = mgr.train_step([cam], target)
    assert np.isfinite(res["loss"]) and res["loss"] > 0
    # no gradient anywhere: the first Adam step leaves every parameter as it was (m = v = 0)
    for k in range(mgr.table.subset_count):
        p, _, _, step = mgr.ctx.store_subset(k, s.sh_coeffs)
        assert step == 1
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(p, f), getattr(before[k], f), err_msg=f)
    mgr.close()


def test_empty_kd_leaves():
    """Three small splats split 8 ways: some KD leaves get no members; the
    merged render still equals the unsplit one and the step runs."""
    s = engine.synth_splats(1_000_000, seed=9, sh_degree=3).take(np.arange(3))
    cam = engine.ring_camera(80, 60, 0, n_views=64)
    ro = engine.render_options(oracle=True)
    out = {}
    for depth in (0, 3):
        mgr = engine.Manager(s, engine.train_config(kd_depth=depth), ro)
        out[depth] = mgr.render(cam)
        if depth == 3:
            sizes = [int(engine.lib().dgs_subset_size(mgr.ctx.handle, k)) for k in range(8)]
            assert min(sizes) == 0, sizes  # the case under test: leaves without members
            res = mgr.train_step([cam], out[0][0][None])
            assert np.isfinite(res["loss"])
        mgr.close()
    (rgb0, t0), (rgb3, t3) = out[0], out[3]
    assert (t0 < 1).any()
    assert np.abs(rgb3 - rgb0).max() <= 1e-4
    assert np.abs(t3 - t0).max() <= 1e-4


@pytest.mark.parametrize("count,wh", [(4000, (257, 131)), (4000, (17, 15)), (1, (64, 48))])
def test_ragged_sizes_and_single_splat_match_oracle(count, wh):
    W, H = wh
    s = engine.synth_splats(10_000, seed=12, sh_degree=3)
    cam = engine.ring_camera(W, H, 3, n_views=64)
    if count == 1:  # the splat nearest the view centre
        s = s.take(np.array([int(np.argmin(np.linalg.norm(s.mu, axis=1)))]))
    else:
        s = s.take(np.arange(count))
    ctx = engine.Context(0)
    ctx.set_table(engine.build_kdtree(s.mu, 0))
    ctx.set_options(engine.render_options(), engine.train_config())
    ctx.load_subset(0, s)
    ct = ctx.render_partial(0, cam)
    ctx.close()
    sc = ob.Scene(s)
    sub = ob.Sub()
    sub.n = 0
    ref = np.zeros((H, W, 4), np.float32)
    assert ob.lib().orc_partial_render(C.byref(sc.c), C.byref(sub), C.byref(ob.cam_of(cam.record())),
                                       C.byref(ob.opts(False)), ob.p(ref), 0, None, None) == 0
    assert (ref[..., 3] < 1).any()
    assert np.abs(ct - ref).max() <= 1e-4


def test_zero_quaternion_raises_domain_error():
    s = engine.synth_splats(500, seed=2, sh_degree=3)
    cam = engine.ring_camera(64, 48, 0, n_views=64)
    s.rotation[:, :] = 0.0
    ctx = engine.Context(0)
    ctx.set_table(engine.build_kdtree(s.mu, 0))
    ctx.set_options(engine.render_options(), engine.train_config())
    ctx.load_subset(0, s)
    with pytest.raises(ArithmeticError, match="quaternion"):
        ctx.render_partial(0, cam)
    ctx.close()


def test_partition_epoch_mismatch_raises():
    """WorkerCore::dispatch(MsgRenderTask) refuses a task from another
    partition epoch (worker.hpp:63, std::runtime_error)."""
    s = engine.synth_splats(800, seed=3, sh_degree=3)
    cam = engine.ring_camera(64, 48, 0, n_views=64)
    target = np.zeros((1, 48, 64, 3), np.float32)
    mgr = engine.Manager(s, engine.train_config(kd_depth=1), engine.render_options())
    mgr.train_step([cam], target)  # epoch 0 everywhere: fine
    mgr.ctx.set_epoch(1)  # the manager moved on; subsets still hold epoch 0
    with pytest.raises(RuntimeError, match="partition epoch mismatch"):
        mgr.train_step([cam], target)
    with pytest.raises(RuntimeError, match="partition epoch mismatch"):
        mgr.ctx.render_partial(0, cam)
    mgr.ctx.set_epoch(0)
    mgr.train_step([cam], target)
    mgr.repartition()  # device repartition: subsets and manager both at epoch 1
    assert mgr.epoch == 1
    mgr.train_step([cam], target)
    mgr.close()


def _ring_overflow_scene(cam, n=64, seed=7):
    """n translucent splats at one distance from the camera centre, clustered
    around the view axis: their ranges share one bucket, so the (t, id) ring
    can emit none of them before the list ends and overflows after 8."""
    rng = np.random.default_rng(seed)
    q = np.asarray(cam.q_wc, np.float64)
    w, x, y, z = q / np.linalg.norm(q)
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    t = np.asarray(cam.t_wc, np.float64)
    o = -R.T @ t
    fwd = R.T @ np.array([0.0, 0.0, 1.0])
    right, up = R.T @ np.array([1.0, 0.0, 0.0]), R.T @ np.array([0.0, 1.0, 0.0])
    s = engine.Splats.empty(n, 16)
    s.id[:] = np.arange(n, dtype=np.uint64)
    for j in range(n):
        d = fwd + 0.004 * (rng.standard_normal() * right + rng.standard_normal() * up)
        s.mu[j] = o + 3.2 * d / np.linalg.norm(d)
    s.log_scale[:] = np.log(0.2 * rng.uniform(0.6, 1.4, (n, 3)))  # anisotropic: rotation gradients are not noise
    s.rotation[:] = rng.standard_normal((n, 4))
    s.opacity_logit[:] = -2.2  # alpha ~ 0.1: no early termination within 64
    s.sh[:, 0, :] = rng.uniform(-1.0, 1.0, (n, 3))
    return s


@pytest.mark.parametrize("n", [64, 300])
def test_ring_overflow_fallbacks_match_oracle(n):
    """Pixels whose reorder ring overflows take the exact fallback kernels
    (forward and backward): the composite and the gradients still match the
    oracle.  n = 300 also fills the fallback's own 256-entry ring, whose walk
    then continues from the last emitted contribution."""
    cam = engine.ring_camera(48, 40, 0, n_views=64)
    s = _ring_overflow_scene(cam, n=n)
    ro, o = engine.render_options(grad_skip_eps=0.0), ob.opts(False, grad_skip_eps=0.0)
    mgr = engine.Manager(s, engine.train_config(kd_depth=0), ro)
    mgr.ctx.set_collect_stats(True)
    target = np.zeros((1, 40, 48, 3), np.float32)
    res = mgr.train_step([cam], target)
    mgr.close()
    assert res["overflow_pixels"] > 0, "the scene did not overflow the ring"

    ctx = engine.Context(0)
    ctx.set_table(engine.build_kdtree(s.mu, 0))
    ctx.set_options(ro, engine.train_config())
    ctx.load_subset(0, s)
    cap = 512
    ct, ids, cnt = ctx.render_partial(0, cam, dbg_cap=cap)
    sc = ob.Scene(s)
    sub = ob.Sub()
    sub.n = 0
    ocam = ob.cam_of(cam.record())
    ref = np.zeros((40, 48, 4), np.float32)
    rids = np.zeros((40 * 48, cap), np.uint32)
    rcnt = np.zeros(40 * 48, np.uint32)
    assert ob.lib().orc_partial_render(C.byref(sc.c), C.byref(sub), C.byref(ocam), C.byref(o), ob.p(ref), cap,
                                       ob.p(rids), ob.p(rcnt)) == 0
    assert rcnt.max() > 8
    assert np.abs(ct - ref).max() <= 1e-4
    np.testing.assert_array_equal(cnt, rcnt)
    for p in np.nonzero(rcnt)[0]:
        np.testing.assert_array_equal(ids[p, :cnt[p]], rids[p, :rcnt[p]], err_msg=f"pixel {p}")
    # backward through the fallback: gradients against the oracle's
    g = (np.random.default_rng(5).standard_normal((40, 48, 4)) * 1e-2).astype(np.float32)
    got = ctx.render_partial_backward(0, cam, g, s.sh_coeffs)
    order = np.argsort(ctx.store_subset(0, s.sh_coeffs)[0].id)  # storage order -> id order
    ctx.close()
    gr, want = ob.empty_grads(s.n, s.sh_coeffs)
    assert ob.lib().orc_partial_backward(C.byref(sc.c), C.byref(sub), C.byref(ocam), C.byref(o), ob.p(g),
                                         C.byref(gr)) == 0
    for f in ("mu", "log_scale", "rotation", "opacity_logit"):
        a = getattr(got, f)[order].astype(np.float64)
        b = want["d_" + f].astype(np.float64)
        floor = 1e-3 * np.abs(b).max()
        err = np.abs(a - b) / np.maximum(np.abs(b), floor)
        assert err.max() <= 1e-3, (f, float(err.max()))


def test_record_capacity_overflow_replays_tile():
    """Pixels with more composited contributions than the record holds
    (kRecCap = 256) mark their tile for the ordered-ring replay in the
    backward; the gradients still match the oracle's."""
    cam = engine.ring_camera(40, 32, 0, n_views=64)
    n = 400
    s = _ring_overflow_scene(cam, n=n, seed=8)
    # spread along the view axis (distinct ranges, so the ring drains) and faint (no termination)
    s.mu[:] = (s.mu + np.linspace(-0.6, 0.6, n)[:, None] * _view_axis(cam)).astype(np.float32)
    s.opacity_logit[:] = -4.6  # alpha ~ 0.01
    # small splats: the order slack (~ D^2 / 2r) stays below the range spacing, so no ring overflow
    s.log_scale[:] = np.log(0.03 * np.random.default_rng(4).uniform(0.6, 1.4, (n, 3))).astype(np.float32)
    ro, o = engine.render_options(grad_skip_eps=0.0), ob.opts(False, grad_skip_eps=0.0)
    mgr = engine.Manager(s, engine.train_config(kd_depth=0), ro)
    mgr.ctx.set_collect_stats(True)
    res = mgr.train_step([cam], np.zeros((1, 32, 40, 3), np.float32))
    mgr.close()
    assert res["overflow_pixels"] == 0
    assert res["replay_tiles_bwd"] > 0, "no tile exceeded the record capacity"
    ctx = engine.Context(0)
    ctx.set_table(engine.build_kdtree(s.mu, 0))
    ctx.set_options(ro, engine.train_config())
    ctx.load_subset(0, s)
    ctx.render_partial(0, cam)
    g = (np.random.default_rng(6).standard_normal((32, 40, 4)) * 1e-2).astype(np.float32)
    got = ctx.render_partial_backward(0, cam, g, s.sh_coeffs)
    order = np.argsort(ctx.store_subset(0, s.sh_coeffs)[0].id)
    ctx.close()
    sc = ob.Scene(s)
    sub = ob.Sub()
    sub.n = 0
    gr, want = ob.empty_grads(s.n, s.sh_coeffs)
    assert ob.lib().orc_partial_backward(C.byref(sc.c), C.byref(sub), C.byref(ob.cam_of(cam.record())), C.byref(o),
                                         ob.p(g), C.byref(gr)) == 0
    for f in ("mu", "log_scale", "rotation", "opacity_logit"):
        a = getattr(got, f)[order].astype(np.float64)
        b = want["d_" + f].astype(np.float64)
        floor = 1e-3 * np.abs(b).max()
        err = np.abs(a - b) / np.maximum(np.abs(b), floor)
        assert err.max() <= 1e-3, (f, float(err.max()))


def _view_axis(cam):
    q = np.asarray(cam.q_wc, np.float64)
    w, x, y, z = q / np.linalg.norm(q)
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    return R.T @ np.array([0.0, 0.0, 1.0])


def test_device_repartition_into_empty_leaves():
    """dgs_repartition to a depth with more leaves than splats: the device
    path still equals the host path (planes, members, migrated p/m/v)."""
    from test_gpu_repartition import _check, _host_reference

    s = engine.synth_splats(1_000_000, seed=9, sh_degree=3).take(np.arange(3))
    cam = engine.ring_camera(48, 40, 0, n_views=64)
    mgr = engine.Manager(s, engine.train_config(kd_depth=0), engine.render_options())
    mgr.train_step([cam], np.zeros((1, 40, 48, 3), np.float32))
    mgr.config.kd_depth = 3
    ref = _host_reference(mgr, 3)
    mgr.repartition(device=True)
    assert mgr.table.subset_count == 8
    sizes = [int(engine.lib().dgs_subset_size(mgr.ctx.handle, k)) for k in range(8)]
    assert min(sizes) == 0, sizes
    _check(mgr, ref)
    res = mgr.train_step([cam], np.zeros((1, 40, 48, 3), np.float32))
    assert np.isfinite(res["loss"])
    mgr.close()
