"""One rank's share of the 8-way configs C4 / C5 (BASELINE.json configs[3], [4]) on
one B200: a real KD leaf of the full scene, timed through Manager::train_step.

  python scripts/bench_rank_proxy.py --config c4 [--leaves 0,3] [--steps 5]
  python scripts/bench_rank_proxy.py --config c5

C4: 100M Gaussians, 3840x2160, 8-way KD partition, batch of 4 views per step.
C5: 500M Gaussians, 1920x1080, 8-way KD partition, batch 1.

Scene: synth_scene's distributions (io.hpp:491-537: mu ~ U[-1,1]^3, base scale
1.1 N^-1/3 (0.6 + 0.9u), per-axis x (0.7 + 0.6u), q = normalized N(0,1)^4,
alpha ~ U(0.5, 0.95), SH DC colour ~ U(0.1, 0.9), higher bands 0) drawn with
numpy for all N centres and scales (the libstdc++ stream of dgs_synth_splats is
single-threaded and would need 118 GB of host memory at N = 500M).  The KD
tree (depth 3, exact medians) and the membership test (3 sigma, replicas
included) run over all N; leaf k's members get their remaining parameters.

What runs: a context holding the real 8-leaf table, leaf k with its members
and the seven other leaves empty, so the forward, the per-pixel subspace order,
the merge, the loss, the merge adjoint, the backward and the dense Adam step
are the code a rank of an 8-GPU run executes on its leaf — minus the NCCL
exchange (its payload is reported) and with the merge/loss/merge-adjoint done
over the whole image instead of the rank's 1/8 row slice (reported per stage,
and subtracted in `rank_step_ms_estimate`).  Output: one JSON line per leaf
plus a summary line; the 8-GPU step is bounded below by the slowest leaf.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c4": dict(count=100_000_000, width=3840, height=2160, batch=4, kd=3),
    "c5": dict(count=500_000_000, width=1920, height=1080, batch=1, kd=3),
}


def gen_centres(n, seed):
    rng = np.random.default_rng(seed)
    mu = np.empty((n, 3), np.float32)
    ls = np.empty((n, 3), np.float32)
    spacing = 1.1 * n ** (-1.0 / 3.0)
    step = 25_000_000
    for i in range(0, n, step):
        j = min(n, i + step)
        mu[i:j] = (rng.random((j - i, 3), dtype=np.float32) * 2.0 - 1.0)
        base = spacing * (0.6 + 0.9 * rng.random(j - i))
        ls[i:j] = np.log(base[:, None] * (0.7 + 0.6 * rng.random((j - i, 3)))).astype(np.float32)
    return mu, ls


def leaf_splats(engine, idx, mu, ls, seed):
    rng = np.random.default_rng(seed)
    n = len(idx)
    s = engine.Splats.empty(n, 16)
    s.id[:] = idx.astype(np.uint64)
    s.mu[:] = mu[idx]
    s.log_scale[:] = ls[idx]
    q = rng.standard_normal((n, 4)).astype(np.float32)
    s.rotation[:] = q / np.linalg.norm(q, axis=1, keepdims=True)
    a = 0.5 + 0.45 * rng.random(n)
    s.opacity_logit[:] = np.log(a / (1.0 - a)).astype(np.float32)
    s.sh[:, 0, :] = ((0.1 + 0.8 * rng.random((n, 3)) - 0.5) / 0.28209479177387814).astype(np.float32)
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--leaves", default="all")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--count", type=int, default=0, help="override N (smaller dry runs)")
    a = ap.parse_args()
    cfgd = dict(CONFIGS[a.config])
    if a.count:
        cfgd["count"] = a.count
    N, W, H, B, kd = cfgd["count"], cfgd["width"], cfgd["height"], cfgd["batch"], cfgd["kd"]
    K = 1 << kd

    import torch
    from paper_2406_11836_b200 import engine

    t0 = time.time()
    mu, ls = gen_centres(N, 11)
    t_gen = time.time() - t0
    table = engine.build_kdtree(mu, kd)
    t_kd = time.time() - t0 - t_gen

    class _MuLs:  # assign_subsets reads only mu and log_scale
        def __init__(self, m, l):
            self.mu, self.log_scale, self.n = m, l, m.shape[0]
    members = engine.assign_subsets(table, _MuLs(mu, ls), 3.0)
    t_assign = time.time() - t0 - t_gen - t_kd
    sizes = [len(m) for m in members]
    views = [(8 * i) % 64 for i in range(B)] if B > 1 else [0]
    cams = [engine.ring_camera(W, H, v, n_views=64) for v in views]
    leaves = list(range(K)) if a.leaves == "all" else [int(x) for x in a.leaves.split(",")]
    print(json.dumps({"config": a.config, "gaussians": N, "width": W, "height": H, "batch": B, "kd_subsets": K,
                      "leaf_members": sizes, "replica_overlap": sum(sizes) / N - 1.0,
                      "setup_s": {"generate": t_gen, "kdtree": t_kd, "assign": t_assign}}), flush=True)

    results = []
    for k in leaves:
        ts = time.time()
        s_k = leaf_splats(engine, members[k], mu, ls, 100 + k)
        # targets: a rendering of the leaf itself from slightly perturbed parameters is not
        # needed for timing; the loss runs on a fixed synthetic target per view
        rng = np.random.default_rng(7)
        targets = rng.random((B, H, W, 3), dtype=np.float32)
        cfg = engine.train_config(kd_depth=kd, batch_size=B, iterations=30000, deterministic=0)
        ro = engine.render_options(grad_skip_eps=0.0)
        ctx = engine.Context(0)
        ctx.set_table(table)
        ctx.set_options(ro, cfg)
        empty = engine.Splats.empty(0, 16)
        for j in range(K):
            ctx.load_subset(j, s_k if j == k else empty)
        tdev = ctx.upload_targets(targets)
        t_load = time.time() - ts
        stream = torch.cuda.ExternalStream(ctx.stream())
        for _ in range(a.warmup):
            ctx.train_step(cams, None, targets_device_ptr=tdev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = [ctx.train_step(cams, None, targets_device_ptr=tdev) for _ in range(a.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        ctx.set_profiling(True)
        for _ in range(2):
            ctx.train_step(cams, None, targets_device_ptr=tdev)
        st = {key: v[0] / 2 for key, v in ctx.stage_times().items()}
        ctx.set_profiling(False)
        ctx.set_collect_stats(True)
        rs = ctx.train_step(cams, None, targets_device_ptr=tdev)
        ctx.set_collect_stats(False)
        full_img = st.get("merge", 0.0) + st.get("loss", 0.0) + st.get("merge_bwd", 0.0)
        est = ms - full_img * (1.0 - 1.0 / K)
        px = W * H
        # per-rank NCCL payload per step of the 8-GPU run: partial rows of the
        # other 7 slices (+ halo) forward, gradient rows back, per view
        halo = 20 * W * 16 * (K - 1)
        payload = B * (2 * (K - 1) * (px // K) * 16 + halo)
        line = {"leaf": k, "members": int(s_k.n), "ms_per_step": ms, "rank_step_ms_estimate": est,
                "stages_ms_per_step": {key: round(v, 4) for key, v in st.items()},
                "pairs": rs["pairs"], "visible": rs["visible"], "contribs_fwd": rs["contribs_fwd"],
                "overflow_pixels": rs["overflow_pixels"], "replay_tiles_bwd": rs["replay_tiles_bwd"],
                "loss": res[-1]["loss"], "exchange_payload_bytes_per_step": payload,
                "exchange_ms_at_900GBps": payload / 900e9 * 1e3, "load_s": t_load}
        results.append(line)
        print(json.dumps(line), flush=True)
        ctx.close()
        del s_k
    worst = max(results, key=lambda r: r["rank_step_ms_estimate"])
    step_ms = worst["rank_step_ms_estimate"] + worst["exchange_ms_at_900GBps"]
    summary = {
        "summary": a.config, "metric": "Mpixel/s (fwd+bwd+merge+Adam), per-rank proxy of the 8-GPU step",
        "leaves_measured": [r["leaf"] for r in results],
        "slowest_leaf": worst["leaf"], "slowest_rank_step_ms": worst["rank_step_ms_estimate"],
        "predicted_8gpu_step_ms": step_ms, "predicted_8gpu_mpx_per_s": B * W * H / 1e6 / (step_ms / 1e3),
        "rank_imbalance_max_over_mean": worst["rank_step_ms_estimate"] /
                                        (sum(r["rank_step_ms_estimate"] for r in results) / len(results)),
        "caveats": "exchange not executed (payload / 900 GB/s added, not overlapped); merge/loss/adjoint over the "
                   "whole image measured and scaled to the rank's 1/8 slice; targets synthetic (timing only)",
    }
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
