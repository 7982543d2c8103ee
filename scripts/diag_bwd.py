import sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import Golden, rel_err
from paper_2406_11836_b200 import engine
from test_gpu_parity import make_ctx, members_of
for name in sys.argv[1:]:
    g = Golden(name)
    ctx, table, s = make_ctx(g, members_of(g))
    cam = g.camera()
    for k in range(g.subsets()):
        grad_ct = np.concatenate([g[f"k{k}_dC"], g[f"k{k}_dT"][..., None]], axis=-1)
        got = ctx.render_partial_backward(k, cam, grad_ct, s.sh_coeffs)
        g2 = ctx.dump_pixel_grads(k)
        src = g[f"k{k}_proj_source"]
        ref = g[f"k{k}_g2d"]
        mine = g2[src]
        for f in range(9):
            e = rel_err(mine[:, f], ref[:, f])
            scale = np.abs(ref[:, f]).max()
            big = np.abs(ref[:, f]) > 1e-3 * scale
            print(name, k, 'g2d', f, 'max rel', e.max(), 'max rel on big', e[big].max() if big.any() else 0, 'scale', scale,
                  'worst idx', e.argmax(), mine[e.argmax(), f], ref[e.argmax(), f])
        for fld in ("d_mu", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
            want = g[f"k{k}_grad_{fld}"]
            a = getattr(got, fld[2:]).reshape(want.shape)
            e = rel_err(a, want)
            scale = np.abs(want).max()
            big = np.abs(want) > 1e-3 * scale
            print(name, k, fld, 'max rel', e.max(), 'on big', e[big].max() if big.any() else 0, 'scale', scale)
