"""Diagnostic: tile-list ordering quality of the binning at C3 scale."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2406_11836_b200 import engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
oracle = len(sys.argv) > 2 and sys.argv[2] == "oracle"
gt = engine.synth_splats(n, seed=11, sh_degree=3)
cam = engine.ring_camera(1920, 1080, 0, n_views=64)
table = engine.build_kdtree(gt.mu, 0)
ctx = engine.Context(0)
ctx.set_table(table)
ctx.set_options(engine.render_options(oracle=oracle), engine.train_config())
ctx.load_subset(0, gt)
ctx.set_collect_stats(True)
t = time.time(); ct = ctx.render_partial(0, cam); print("render s", time.time() - t)
recs, counts = ctx.dump_records(0)
yb = ctx.dump_order_bounds(0)
off, ent = ctx.dump_bins(0, cam)
rng = recs[:, 15]
print("pairs", off[-1], "visible", (counts > 0).sum(), "dmax", np.sqrt(recs[:, 3].max()))
viol = 0; desc = 0; gaps = []
for tt in range(len(off) - 1):
    e = ent[off[tt]:off[tt + 1]]
    if len(e) < 2: continue
    r = rng[e]
    sm = np.minimum.accumulate(r[::-1])[::-1]
    viol += int((yb[e, 1] > sm).sum())
    desc += int((np.diff(r) < 0).sum())
    gaps.append(float((r - yb[e, 1]).max()))
print("order-bound violations", viol, "descents", desc, "of", off[-1], "max(range - bound) per tile: median", np.median(gaps), "max", max(gaps))
e = ent[off[4000]:off[4001]]
print("tile 4000 first 40 ranges", np.round(rng[e[:40]], 5))
print("tile 4000 first 40 bounds", np.round(yb[e[:40], 1], 5))
