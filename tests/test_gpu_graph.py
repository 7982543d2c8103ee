"""GPU: train steps as CUDA graph replays (dgs_set_graph_mode).

A captured step has no host round trip: the pair counts stay on the device and
the tile sort runs over each slot's learnt capacity with the tail padded by tile
key 0xffff; the AdamParams are re-read from pinned memory at every replay; the
results land in a pinned tail buffer.  With TrainConfig::deterministic = 1 the
graph steps must equal the eager steps bit for bit (parameters, both Adam
moments, losses, a render afterwards) across several views (one graph each),
with one and two KD subsets and with batch 2 (the view chains on the second
stream join the capture), and with pinned host targets (uploaded outside the
graph on the copy stream, which the graph waits for as an external event; the
host pointer may change between replays).  A replay whose pair counts outgrow the captured
capacity (forced with DGS_GRAPH_CAP_TEST, in a subprocess) must skip its Adam
step, re-run eagerly and still give the eager result."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2406_11836_b200 import engine  # noqa: E402

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")
CASES = {"k1_b1": dict(kd=0, batch=1), "k2_b1": dict(kd=1, batch=1), "k2_b2": dict(kd=1, batch=2),
         "k1_b2_host": dict(kd=0, batch=2, host=True)}


def scene():
    gt = engine.synth_splats(30_000, seed=7, sh_degree=3)
    cams = [engine.ring_camera(320, 240, v, n_views=64) for v in range(0, 64, 16)]
    tm = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
    targets = np.stack([tm.render(cam)[0] for cam in cams])
    tm.close()
    return engine.perturb(gt, 5), cams, targets


def run(sc, c, graph, steps=12):
    import torch

    init, cams, targets = sc
    cfg = engine.train_config(kd_depth=c["kd"], deterministic=1, batch_size=c["batch"])
    mgr = engine.Manager(init, cfg, engine.render_options())
    mgr.ctx.set_graph_mode(graph)
    # device-resident planar targets (the bench's layout): fixed pointers per view
    tdev = torch.from_numpy(targets.transpose(0, 3, 1, 2).copy()).cuda()
    vb = tdev[0].numel() * 4
    # pinned host targets (HWC, the e2e layout): two copies used alternately, so
    # replays see a different host pointer than the one captured
    pins = [torch.from_numpy(targets.copy()).pin_memory() for _ in range(2)] if c.get("host") else None
    losses = []
    for s in range(steps):
        v0 = (s * c["batch"]) % len(cams)
        idx = [(v0 + j) % len(cams) for j in range(c["batch"])]
        if pins is not None:
            assert idx == list(range(idx[0], idx[0] + c["batch"]))
            r = mgr.train_step([cams[i] for i in idx], pins[s % 2].numpy()[idx[0]:idx[0] + c["batch"]])
        elif c["batch"] == 1:
            r = mgr.train_step([cams[idx[0]]], None, targets_device_ptr=tdev.data_ptr() + idx[0] * vb)
        else:  # batches of consecutive views: contiguous device targets
            assert idx == list(range(idx[0], idx[0] + c["batch"]))
            r = mgr.train_step([cams[i] for i in idx], None, targets_device_ptr=tdev.data_ptr() + idx[0] * vb)
        losses.append(r["loss"])
    rgb, _ = mgr.render(cams[0])
    out = {"losses": np.asarray(losses), "rgb": rgb}
    for k in range(mgr.table.subset_count):
        p, m, v, step = mgr.ctx.store_subset(k, init.sh_coeffs)
        out[f"step{k}"] = np.asarray(step)
        for f in FIELDS:
            out[f"p{k}_{f}"], out[f"m{k}_{f}"], out[f"v{k}_{f}"] = getattr(p, f), getattr(m, f), getattr(v, f)
    mgr.close()
    return out


@pytest.fixture(scope="module")
def sc():
    return scene()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_graph_steps_equal_eager(sc, name):
    c = CASES[name]
    g, e = run(sc, c, True), run(sc, c, False)
    for key in g:
        assert np.array_equal(g[key], e[key]), key


@pytest.mark.gpu
def test_state_restore_replays_identically(sc):
    """dgs_state_save / dgs_state_restore: steps after a restore equal the
    steps after the save bit for bit (parameters, moments, step count, losses),
    with the step graphs captured in between still replayed."""
    import torch

    init, cams, targets = sc
    cfg = engine.train_config(kd_depth=1, deterministic=1)
    mgr = engine.Manager(init, cfg, engine.render_options())
    mgr.ctx.set_graph_mode(True)
    tdev = torch.from_numpy(targets.transpose(0, 3, 1, 2).copy()).cuda()
    vb = tdev[0].numel() * 4

    def steps(n):
        return [mgr.train_step([cams[s % len(cams)]], None, targets_device_ptr=tdev.data_ptr() + (s % len(cams)) * vb)
                ["loss"] for s in range(n)]

    def state():
        out = {}
        for k in range(mgr.table.subset_count):
            p, m, v, step = mgr.ctx.store_subset(k, init.sh_coeffs)
            out[(k, "step")] = np.asarray(step)
            for name, sp in (("p", p), ("m", m), ("v", v)):
                for f in FIELDS:
                    out[(k, name, f)] = getattr(sp, f)
        return out

    with pytest.raises(Exception, match="no saved state"):
        mgr.ctx.restore_state()
    steps(2 * len(cams))  # every view captured
    mgr.ctx.save_state()
    a, sa = steps(10), state()
    mgr.ctx.restore_state()
    b, sb = steps(10), state()
    mgr.close()
    assert a == b
    for key in sa:
        assert np.array_equal(sa[key], sb[key]), key


@pytest.mark.gpu
def test_graph_capacity_overflow_reruns_eagerly(sc, tmp_path):
    out = tmp_path / "overflow.npz"
    env = dict(os.environ, DGS_GRAPH_CAP_TEST="1")
    subprocess.run([sys.executable, __file__, str(out)], check=True, env=env, cwd=ROOT, timeout=600)
    g = np.load(out)
    e = run(sc, CASES["k1_b1"], False)
    for key in e:
        assert np.array_equal(g[key], e[key]), key


@pytest.mark.gpu
def test_graph_waits_for_the_host_target_upload(sc, tmp_path):
    """Pinned host targets are uploaded outside the graph; the graph waits for
    the upload through an external event node.  With the upload held back by
    20 ms (DGS_TEST_UPLOAD_DELAY_US, a spin kernel ahead of it on the copy
    stream) a replay that did not wait would blend against the previous
    step's targets; it must still equal the eager steps."""
    out = tmp_path / "delayed.npz"
    env = dict(os.environ, DGS_TEST_UPLOAD_DELAY_US="20000")
    subprocess.run([sys.executable, __file__, str(out), "k1_b2_host"], check=True, env=env, cwd=ROOT, timeout=600)
    g = np.load(out)
    e = run(sc, CASES["k1_b2_host"], False)
    for key in e:
        assert np.array_equal(g[key], e[key]), key


if __name__ == "__main__":
    case = sys.argv[2] if len(sys.argv) > 2 else "k1_b1"
    res = run(scene(), CASES[case], True)
    np.savez(sys.argv[1], **res)
