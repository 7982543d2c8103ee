"""GPU: config.grad_sync (worker.hpp:103-144,
manager.hpp:351-379).  With sync on, every replica of a shared splat applies
Adam to the sum of its replicas' gradients (summed in worker order), so the
replicas stay bit-identical; the post-Adam values follow the reference's
per-subset gradients (the goldens) summed the same way."""
import numpy as np
import pytest

from conftest import Golden, adam_lr_rows, post_adam_ok
from paper_2406_11836_b200 import engine

pytestmark = pytest.mark.gpu

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")


@pytest.mark.parametrize("name", ["g2_synth_kd2_default", "g4_synth_kd3_bg"])
def test_grad_sync_keeps_replicas_identical_and_matches_summed_reference(name):
    g = Golden(name)
    s = g.splats()
    K = g.subsets()
    cfg = engine.train_config(kd_depth=g.args["kd"], grad_sync=1)
    mgr = engine.Manager(s, cfg, engine.render_options(oracle=g.oracle_mode))
    cam = g.camera()
    mgr.train_step([cam], g["step_target"][None], g.bg)
    off, ids = g["kd_member_off"], g["kd_member_ids"]
    members = [ids[off[k]:off[k + 1]].astype(np.int64) for k in range(K)]
    # reference gradients summed over replicas in worker order (float32, manager.hpp:363-371)
    summed = {f: {} for f in FIELDS}
    for k in range(K):
        for f in FIELDS:
            gk = g[f"k{k}_grad_d_{f}"].reshape((len(members[k]),) + getattr(s, f).shape[1:]).astype(np.float32)
            for j, idx in enumerate(members[k]):
                sid = int(s.id[idx])
                summed[f][sid] = gk[j].copy() if sid not in summed[f] else (summed[f][sid] + gk[j]).astype(np.float32)
    lrs = adam_lr_rows(cfg, s.sh_coeffs)
    stored = [mgr.ctx.store_subset(k, s.sh_coeffs) for k in range(K)]
    by_id = {}
    n_shared = 0
    for k, (p, m, v, step) in enumerate(stored):
        assert step == 1
        for i in range(p.n):
            sid = int(p.id[i])
            vals = tuple(np.concatenate([getattr(x, f)[i].ravel() for f in FIELDS]) for x in (p, m, v))
            if sid in by_id:
                n_shared += 1
                for a, b in zip(by_id[sid], vals):
                    np.testing.assert_array_equal(a, b, err_msg=f"replicas of splat {sid} diverged")
            else:
                by_id[sid] = vals
        for f in FIELDS:
            got = getattr(p, f)
            sids = [int(x) for x in p.id]
            p0 = np.stack([getattr(s, f)[int(np.nonzero(s.id == sid)[0][0])] for sid in sids]).astype(np.float64)
            gsum = np.stack([summed[f][sid] for sid in sids]).astype(np.float64)
            lr = np.broadcast_to(np.asarray(lrs[f], np.float64), gsum.shape[1:]) if f == "sh" else lrs[f]
            # first Adam step (optim.hpp:90-97): p - lr * g / (|g| + eps)
            want = p0 - np.asarray(lr, np.float64) * gsum / (np.abs(gsum) + cfg.adam_eps)
            ok, e, noisy = post_adam_ok(got.astype(np.float64), want, gsum, lr)
            assert ok.all(), (k, f, int((~ok).sum()))
    assert n_shared > 0, "the scene has no shared splats: the test would be vacuous"
    mgr.close()
