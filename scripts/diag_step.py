"""Diagnostic: per-step wall/GPU time of the C3 step under different host conditions."""
import sys, time, json, math
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2406_11836_b200 import engine
import bench

a = bench.parse()
gt = engine.synth_splats(a.count, seed=11, sh_degree=3)
cam = engine.ring_camera(a.width, a.height, a.view, n_views=64)
init = engine.perturb(gt, 5)
tm = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
t0 = time.time(); target, _ = tm.render(cam); print("target render s", time.time() - t0, flush=True)
tm.close()
mgr = engine.Manager(init, engine.train_config(kd_depth=0, iterations=30000, deterministic=0), engine.render_options(grad_skip_eps=0.0))
ctx = mgr.ctx
tdev = ctx.upload_targets(target[None])
stream = torch.cuda.ExternalStream(ctx.stream())
def run(n, label, host=False):
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); w = time.perf_counter(); hts = []
    for _ in range(n):
        h = time.perf_counter()
        if host: mgr.train_step([cam], target[None])
        else: mgr.train_step([cam], None, targets_device_ptr=tdev)
        hts.append((time.perf_counter() - h) * 1e3)
    e1.record(stream); torch.cuda.synchronize()
    st = ctx.stage_times(); ctx.set_profiling(False)
    print(label, "gpu ms/step", e0.elapsed_time(e1) / n, "wall", (time.perf_counter() - w) * 1e3 / n, "host call ms", np.median(hts),
          {k: round(v[0] / n, 3) for k, v in st.items()}, flush=True)
ctx.set_collect_stats(True)
for i in range(60):
    r = mgr.train_step([cam], None, targets_device_ptr=tdev)
    if i % 3 == 0:
        print(i, {k: r[k] for k in ("loss", "pairs", "evals_fwd", "contribs_fwd", "overflow_pixels", "subrounds_bwd", "tiles_work_fwd")}, flush=True)
ctx.set_collect_stats(False)
run(10, "after 60")
