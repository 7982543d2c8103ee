"""Step time and work counters over a long C3 run (same view every step, as in bench.py)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2406_11836_b200 import engine

N, W, H = 10_000_000, 1920, 1080
STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 120
gt = engine.synth_splats(N, seed=11, sh_degree=3)
cam = engine.ring_camera(W, H, 0, n_views=64)
t = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
target, _ = t.render(cam)
t.close()
mgr = engine.Manager(engine.perturb(gt, 5), engine.train_config(kd_depth=0, iterations=30000, deterministic=0),
                     engine.render_options(grad_skip_eps=0.0))
tdev = mgr.ctx.upload_targets(target[None])
for i in range(STEPS):
    stats = i % 10 == 0
    if stats:
        mgr.ctx.set_collect_stats(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = mgr.train_step([cam], None, targets_device_ptr=tdev)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    if stats:
        mgr.ctx.set_collect_stats(False)
        print(f"step {i:4d} {dt:8.2f} ms loss {r['loss']:.5f} pairs {r['pairs']/1e6:.2f}M evals {r['evals_fwd']/1e6:.1f}M "
              f"contribs {r['contribs_bwd']/1e6:.1f}M ovf {r['overflow_pixels']} replay {r['replay_tiles_bwd']} vis {r['visible']}",
              flush=True)
