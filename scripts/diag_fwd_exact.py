"""Diagnostic: how close the GPU forward (partials, merged render, loss gradient) is to the reference goldens."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from conftest import Golden
from test_gpu_parity import members_of, make_ctx
from paper_2406_11836_b200 import engine
for name in sys.argv[1:]:
    g = Golden(name)
    ctx, table, s = make_ctx(g, members_of(g))
    cam = g.camera()
    parts = []
    for k in range(g.subsets()):
        ct = ctx.render_partial(k, cam)
        parts.append(ct)
        C, T = g[f"k{k}_C"], g[f"k{k}_T"]
        print(name, k, "C bit-equal frac", float((ct[..., :3] == C).mean()), "max", float(np.abs(ct[..., :3] - C).max()),
              "T bit-equal frac", float((ct[..., 3] == T).mean()), "max", float(np.abs(ct[..., 3] - T).max()))
    if "step_render" in g:
        rgb, _ = ctx.merge(cam, np.stack(parts), g.bg)
        print(name, "merged bit-equal frac", float((rgb == g["step_render"]).mean()), "max", float(np.abs(rgb - g["step_render"]).max()))
        l, grad, _ = ctx.loss(rgb, g["step_target"])
        print(name, "loss grad bit-equal frac", float((grad == g["step_grad_color"]).mean()), "n diff", int((grad != g["step_grad_color"]).sum()))
    ctx.close()
