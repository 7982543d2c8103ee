"""Diagnostic: per-stage times of the C3 step with deterministic = 0 and 1."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2406_11836_b200 import engine
import bench

a = bench.parse()
gt = engine.synth_splats(a.count, seed=11, sh_degree=3)
cam = engine.ring_camera(a.width, a.height, a.view, n_views=64)
init = engine.perturb(gt, 5)
tm = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
target, _ = tm.render(cam)
tm.close()
ro = engine.render_options(grad_skip_eps=0.0)
mgr = engine.Manager(init, engine.train_config(kd_depth=0, iterations=30000, deterministic=0), ro)
ctx = mgr.ctx
tdev = ctx.upload_targets(target[None])
stream = torch.cuda.ExternalStream(ctx.stream())
import os
modes = (1,) if os.environ.get("DIAG_ONLY_DET") else (0, 1, 0)
reps = 2 if os.environ.get("DIAG_ONLY_DET") else 10
for det in modes:
    ctx.set_options(ro, engine.train_config(kd_depth=0, iterations=30000, deterministic=det))
    for _ in range(3):
        mgr.train_step([cam], None, targets_device_ptr=tdev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        mgr.train_step([cam], None, targets_device_ptr=tdev)
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    for _ in range(10):
        mgr.train_step([cam], None, targets_device_ptr=tdev)
    st = ctx.stage_times()
    ctx.set_profiling(False)
    print("det", det, "ms/step", round(e0.elapsed_time(e1) / reps, 3), {k: round(v[0] / 10, 3) for k, v in st.items()},
          flush=True)
