"""Where does the e2e step (host targets) lose time against the device-resident step?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2406_11836_b200 import engine

N, W, H, STEPS = 10_000_000, 1920, 1080, 20
gt = engine.synth_splats(N, seed=11, sh_degree=3)
cam = engine.ring_camera(W, H, 0, n_views=64)
t = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
target, _ = t.render(cam)
t.close()
mgr = engine.Manager(engine.perturb(gt, 5), engine.train_config(kd_depth=0, iterations=30000, deterministic=0),
                     engine.render_options(grad_skip_eps=0.0))
ctx = mgr.ctx
stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda:0"))
tdev = ctx.upload_targets(target[None])
pinned = torch.empty(target.size, dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = target.reshape(-1)
host_pinned = pinned.numpy().reshape(1, H, W, 3)
host_pageable = np.ascontiguousarray(target[None], np.float32)


def run(label, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    w0 = time.perf_counter()
    for _ in range(STEPS):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{label:28s} events {e0.elapsed_time(e1) / STEPS:.3f} ms  wall {(time.perf_counter() - w0) * 1e3 / STEPS:.3f} ms")


run("device targets", lambda: mgr.train_step([cam], None, targets_device_ptr=tdev))
run("host pinned targets", lambda: mgr.train_step([cam], host_pinned))
run("host pageable targets", lambda: mgr.train_step([cam], host_pageable))
# raw PCIe copy
dst = torch.empty(target.size, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    dst.copy_(pinned, non_blocking=True)
b.record()
torch.cuda.synchronize()
print(f"pinned H2D {target.nbytes / 1e6:.1f} MB: {a.elapsed_time(b) / 10:.3f} ms")
