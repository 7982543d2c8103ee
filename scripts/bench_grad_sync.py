"""config.grad_sync (worker.hpp:103-144, manager.hpp:351-379) on one B200: the C3
workload split into 2 KD subsets on one GPU, ms per training step with
grad_sync = 0 (gradient record + streaming Adam) and 1 (full gradient rows,
shared replicas summed in worker order, dense Adam over G).  CUDA events on
the context stream; prints one JSON line."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2406_11836_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
steps, warm = 10, 3
gt = engine.synth_splats(n, seed=11, sh_degree=3)
cams = [engine.ring_camera(1920, 1080, v, n_views=64) for v in range(0, 64, 8)]
tm = engine.Manager(gt, engine.train_config(kd_depth=0), engine.render_options(oracle=True))
targets = np.stack([tm.render(c)[0] for c in cams])
tm.close()
init = engine.perturb(gt, 5)
tdev = torch.from_numpy(targets.transpose(0, 3, 1, 2).copy()).cuda()
out = {"workload": f"{n / 1e6:g}M synthetic Gaussians, 1920x1080, 2 KD subsets on one GPU, batch 1, 8 ring views"}
for gs in (0, 1):
    mgr = engine.Manager(init, engine.train_config(kd_depth=1, grad_sync=gs, deterministic=0), engine.render_options())
    stream = torch.cuda.ExternalStream(mgr.ctx.stream())
    view_bytes = 3 * 1920 * 1080 * 4
    it = 0
    def step():
        global it
        v = it % len(cams)
        it += 1
        return mgr.train_step([cams[v]], None, targets_device_ptr=tdev.data_ptr() + v * view_bytes)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        r = step()
    e1.record(stream)
    torch.cuda.synchronize()
    out[f"grad_sync_{gs}_ms_per_step"] = e0.elapsed_time(e1) / steps
    out[f"grad_sync_{gs}_loss_last"] = r["loss"]
    mgr.close()
print(json.dumps(out))
