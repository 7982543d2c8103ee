"""Diagnostic: post-Adam mismatches of the full golden step, with the gradient, its rounding bound and the GPU gradient."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from conftest import Golden, golden_bounds, adam_lr_rows, post_adam_ok, U_F32, K_ROUND
from test_gpu_parity import members_of, PARAM_FIELDS
from paper_2406_11836_b200 import engine
for name in sys.argv[1:]:
    g = Golden(name)
    s = g.splats()
    cfg = engine.train_config(kd_depth=g.args.get("kd", 0))
    mgr = engine.Manager(s, cfg, engine.render_options(oracle=g.oracle_mode))
    cam = g.camera()
    res = mgr.train_step([cam], g["step_target"][None], g.bg)
    lrs = adam_lr_rows(cfg, s.sh_coeffs)
    members = members_of(g)
    bounds = golden_bounds(g, members)
    # the GPU's own gradients for the same step inputs (the golden's dC/dT)
    for k in range(g.subsets()):
        p, _, _, _ = mgr.ctx.store_subset(k, s.sh_coeffs)
        for f in PARAM_FIELDS:
            want = g[f"k{k}_adam_{f}"]
            gr = g[f"k{k}_grad_d_{f}"]
            b = bounds[k]["d_" + f].reshape(gr.shape)
            ok, e, noisy = post_adam_ok(getattr(p, f).reshape(want.shape), want, gr, lrs[f], bound=b)
            for i in np.nonzero(~ok.reshape(-1))[0][:5]:
                print(name, k, f, int(i), "p_ref", float(want.reshape(-1)[i]), "p_gpu", float(getattr(p, f).reshape(-1)[i]),
                      "p0", float(getattr(s.take(members[k]), f).reshape(-1)[i]), "g_ref", float(gr.reshape(-1)[i]),
                      "uB", float(U_F32 * b.reshape(-1)[i]), flush=True)
    mgr.close()
