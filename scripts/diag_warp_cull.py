"""How many (splat, 8x4 warp block) candidate lists would an exact ellipse test
drop against K4's bounding-box sub-block test?  C3 scene, ring view 0; a random
sample of the visible splats.  bbox: the conservative x/y half-extents of the
m^2 <= 9 ellipse meet the warp block's pixel-centre rectangle; exact: the
minimum of the quadratic form over that rectangle is <= 9."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2406_11836_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
sample = int(sys.argv[2]) if len(sys.argv) > 2 else 300_000
s = engine.synth_splats(n, seed=11, sh_degree=3)
cam = engine.ring_camera(1920, 1080, 0, n_views=64)
ctx = engine.Context(0)
ctx.set_table(engine.build_kdtree(s.mu, 0))
ctx.set_options(engine.render_options(), engine.train_config())
ctx.load_subset(0, s)
ctx.render_partial(0, cam)
recs, counts = ctx.dump_records(0)
vis = np.nonzero(counts > 0)[0]
rng = np.random.default_rng(0)
pick = rng.choice(vis, size=min(sample, vis.size), replace=False)
r = recs[pick].astype(np.float64)
mx, my = r[:, 0], r[:, 1]
A = r[:, 4]; B = 0.5 * (r[:, 5] + r[:, 6]); Cc = r[:, 7]
det = A * Cc - B * B
rx, ry = 3 * np.sqrt(Cc / det), 3 * np.sqrt(A / det)


def qmin(xl, xh, yl, yh, A, B, C):
    inside = (xl <= 0) & (xh >= 0) & (yl <= 0) & (yh >= 0)
    best = np.full(xl.shape, np.inf)
    for xe in (xl, xh):
        dy = np.clip(-B * xe / C, yl, yh)
        best = np.minimum(best, A * xe * xe + 2 * B * xe * dy + C * dy * dy)
    for ye in (yl, yh):
        dx = np.clip(-B * ye / A, xl, xh)
        best = np.minimum(best, A * dx * dx + 2 * B * dx * ye + C * ye * ye)
    return np.where(inside, 0.0, best)


# warp blocks: 8 px wide, 4 px tall, over the bbox of every sampled splat
bx0 = np.floor((mx - rx) / 8).astype(np.int64); bx1 = np.floor((mx + rx) / 8).astype(np.int64)
by0 = np.floor((my - ry) / 4).astype(np.int64); by1 = np.floor((my + ry) / 4).astype(np.int64)
bx0 = np.clip(bx0, 0, 1920 // 8 - 1); bx1 = np.clip(bx1, 0, 1920 // 8 - 1)
by0 = np.clip(by0, 0, 1080 // 4 - 1); by1 = np.clip(by1, 0, 1080 // 4 - 1)
W = bx1 - bx0 + 1; H = by1 - by0 + 1
nb = ne = 0
for dy in range(int(H.max())):
    for dx in range(int(W.max())):
        sel = (dx < W) & (dy < H)
        if not sel.any():
            continue
        xl = (bx0[sel] + dx) * 8 + 0.5 - mx[sel]; xh = xl + 7.0
        yl = (by0[sel] + dy) * 4 + 0.5 - my[sel]; yh = yl + 3.0
        bb = ~((xl > rx[sel]) | (-xh > rx[sel]) | (yl > ry[sel]) | (-yh > ry[sel]))
        q = qmin(xl, xh, yl, yh, A[sel], B[sel], Cc[sel])
        nb += int(bb.sum()); ne += int((bb & (q <= 9.0 * 1.001)).sum())
print("sampled", pick.size, "bbox warp-block hits", nb, "exact", ne, "kept fraction", ne / max(nb, 1))
