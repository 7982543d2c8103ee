#!/bin/bash
# Can two ranks share one GPU in an NCCL communicator here?  (functional test of the multi-rank step)
OUT=${OUT:-gpurun_out/tworank}; mkdir -p $OUT
export CUDA_VISIBLE_DEVICES=0
cat > /tmp/tworank.py <<'PY'
import os, sys, json, math
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
from paper_2406_11836_b200 import engine
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
obj = [engine.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
try:
    s = engine.synth_splats(20000, seed=11, sh_degree=3)
    cam = engine.ring_camera(320, 180, 0, n_views=64)
    tm = engine.Manager(s, engine.train_config(kd_depth=0), engine.render_options(oracle=True), device=0)
    target, _ = tm.render(cam); tm.close()
    init = engine.perturb(s, 5)
    cfg = engine.train_config(kd_depth=1)
    mgr = engine.Manager(init, cfg, engine.render_options(), device=0, rank=rank, world=world, nccl_id=obj[0])
    r = mgr.train_step([cam], target[None])
    print(json.dumps({"rank": rank, "loss": r["loss"], "nccl_bytes": r["nccl_bytes"]}), flush=True)
    # single-rank reference of the same step
    if rank == 0:
        ref = engine.Manager(init, cfg, engine.render_options(), device=0)
        rr = ref.train_step([cam], target[None])
        print(json.dumps({"single_rank_loss": rr["loss"]}), flush=True)
except Exception as e:
    print("rank", rank, "error:", repr(e), flush=True)
PY
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 /tmp/tworank.py > $OUT/out.txt 2>&1
tail -20 $OUT/out.txt
