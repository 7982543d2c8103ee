"""Time Manager.repartition on the device vs the host path (C3 scale: 10M
splats, KD depth 0 -> 3 on one GPU).  Prints one JSON line."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: F401  (CUDA context warm-up)
from paper_2406_11836_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
s = engine.synth_splats(n, seed=11, sh_degree=3)
out = {"splats": n, "depth": 3}
for dev in (True, False):
    mgr = engine.Manager(s, engine.train_config(kd_depth=0), engine.render_options())
    mgr.config.kd_depth = 3
    mgr.ctx.sync()
    t = time.perf_counter()
    mgr.repartition(device=dev)
    mgr.ctx.sync()
    out["device_s" if dev else "host_s"] = time.perf_counter() - t
    out["subset_sizes_" + ("device" if dev else "host")] = [int(engine.lib().dgs_subset_size(mgr.ctx.handle, k))
                                                            for k in range(8)]
    mgr.close()
print(json.dumps(out))

# init_from_pointcloud at the same scale (trainer.hpp:24-91): the reference's
# neighbour term is O(N^2) on the CPU (days at 10M); here an exact grid k-NN.
import numpy as np  # noqa: E402

rng = np.random.default_rng(1)
pts = (rng.random((n, 3)) * 2 - 1).astype(np.float32)
ctx = engine.Context(0)
engine.init_from_pointcloud(ctx, pts[:1000], None, 1000, seed=1, sh_degree=3)  # warm-up
t = time.perf_counter()
engine.init_from_pointcloud(ctx, pts, None, n, seed=1, sh_degree=3)
print(json.dumps({"init_from_pointcloud_points": n, "seconds": time.perf_counter() - t}))
ctx.close()
