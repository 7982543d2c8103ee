"""K8 sub-round count vs the pixel -> lane assignment: per warp, the union of its
32 pixels' contributor sets (a lower bound on the record walk's sub-rounds) and
the min-rule sub-round count simulated on list positions, for several warp shapes
inside a 16x16 tile.  C3 scene (10M, perturbed seed 5), ring view 0, default options."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2406_11836_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
W, H, CAP = 1920, 1080, 128
s = engine.perturb(engine.synth_splats(n, seed=11, sh_degree=3), 5)
cam = engine.ring_camera(W, H, 0, n_views=64)
ctx = engine.Context(0)
ctx.set_table(engine.build_kdtree(s.mu, 0))
ctx.set_options(engine.render_options(), engine.train_config())
ctx.load_subset(0, s)
ct, ids, cnt = ctx.render_partial(0, cam, dbg_cap=CAP)
off, ent = ctx.dump_bins(0, cam)
ids = ids.reshape(H, W, CAP)
cnt = np.minimum(cnt.reshape(H, W), CAP)
TX, TY = (W + 15) // 16, (H + 15) // 16
print("mean contributions", cnt.mean(), "max", cnt.max())

def shapes():
    yy, xx = np.mgrid[0:16, 0:16]
    out = {}
    # slot -> (y, x) inside the tile for each shape; 8 warps x 32 lanes
    def blocks(bw, bh):
        order = []
        for wy in range(16 // bh):
            for wx in range(16 // bw):
                for ly in range(bh):
                    for lx in range(bw):
                        order.append((wy * bh + ly, wx * bw + lx))
        return np.array(order)
    out["8x4 (current)"] = blocks(8, 4)
    out["4x8"] = blocks(4, 8)
    out["16x2"] = blocks(16, 2)
    out["32x1-ish 16x2 cols"] = blocks(2, 16)
    return out

rng = np.random.default_rng(0)
tiles = rng.choice(TX * TY, size=min(1200, TX * TY), replace=False)
res = {}
for name, order in shapes().items():
    tot_union = 0
    tot_rounds = 0
    tot_contrib = 0
    for t in tiles:
        tx, ty = t % TX, t // TX
        lst = ent[off[t]:off[t + 1]]
        pos = {int(m): i for i, m in enumerate(lst)}  # member index -> list position (ids == member ids here)
        for w in range(8):
            seqs = []
            for (y, x) in order[w * 32:(w + 1) * 32]:
                py, px = ty * 16 + y, tx * 16 + x
                if py >= H or px >= W:
                    continue
                c = int(cnt[py, px])
                seqs.append([pos.get(int(v), -1) for v in ids[py, px, :c]])
            allk = [p for sq in seqs for p in sq]
            tot_contrib += len(allk)
            tot_union += len(set(allk))
            # min-rule sub-rounds
            heads = [0] * len(seqs)
            rounds = 0
            while True:
                keys = [sq[h] if h < len(sq) else None for sq, h in zip(seqs, heads)]
                live = [k for k in keys if k is not None]
                if not live:
                    break
                pm = min(live)
                for i, k in enumerate(keys):
                    if k == pm:
                        heads[i] += 1
                rounds += 1
            tot_rounds += rounds
    res[name] = (tot_union, tot_rounds, tot_contrib)
    print(f"{name:22s} union {tot_union:9d}  min-rule rounds {tot_rounds:9d}  contributions {tot_contrib}  lanes/round {tot_contrib / tot_rounds:.2f}")
