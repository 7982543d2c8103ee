"""How many (splat, tile) pairs of the reference's bounding-box bins can contribute at all?
A pair is kept when the truncation ellipse m^2 <= 9 meets the tile's pixel-centre rectangle
(exact minimum of the quadratic form over the rectangle).  C3 scene, ring view 0."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2406_11836_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
s = engine.synth_splats(n, seed=11, sh_degree=3)
cam = engine.ring_camera(1920, 1080, 0, n_views=64)
ctx = engine.Context(0)
ctx.set_table(engine.build_kdtree(s.mu, 0))
ctx.set_options(engine.render_options(), engine.train_config())
ctx.load_subset(0, s)
ctx.render_partial(0, cam)
recs, counts = ctx.dump_records(0)
vis = counts > 0
r = recs[vis].astype(np.float64)
mx, my = r[:, 0], r[:, 1]
A = r[:, 4].copy(); Bm = 0.5 * (r[:, 5] + r[:, 6]); Cc = r[:, 7].copy()
det = A * Cc - Bm * Bm
c00, c11 = Cc / det, A / det  # cov2d diagonal
rx, ry = 3 * np.sqrt(c00), 3 * np.sqrt(c11)
TX, TY = 120, 68
x0 = np.clip(np.floor(mx - rx).astype(np.int64) // 16, 0, TX - 1); x1 = np.clip(np.floor(mx + rx).astype(np.int64) // 16, 0, TX - 1)
y0 = np.clip(np.floor(my - ry).astype(np.int64) // 16, 0, TY - 1); y1 = np.clip(np.floor(my + ry).astype(np.int64) // 16, 0, TY - 1)
total = ((x1 - x0 + 1) * (y1 - y0 + 1)).sum()
print("visible", vis.sum(), "bbox pairs", total, "(dumped counts sum", counts.sum(), ")")

def qmin(xl, xh, yl, yh):
    # min of A dx^2 + 2B dx dy + C dy^2 over dx in [xl,xh], dy in [yl,yh] (offsets from the mean)
    inside = (xl <= 0) & (xh >= 0) & (yl <= 0) & (yh >= 0)
    best = np.full(xl.shape, np.inf)
    for xe in (xl, xh):  # vertical edges
        dy = np.clip(-Bm * xe / Cc, yl, yh)
        best = np.minimum(best, A * xe * xe + 2 * Bm * xe * dy + Cc * dy * dy)
    for ye in (yl, yh):
        dx = np.clip(-Bm * ye / A, xl, xh)
        best = np.minimum(best, A * dx * dx + 2 * Bm * dx * ye + Cc * ye * ye)
    return np.where(inside, 0.0, best)

kept = 0
W = (x1 - x0 + 1); H = (y1 - y0 + 1)
for dyt in range(int(H.max())):
    for dxt in range(int(W.max())):
        sel = (dxt < W) & (dyt < H)
        if not sel.any():
            continue
        tx = x0[sel] + dxt; ty = y0[sel] + dyt
        xl = tx * 16 + 0.5 - mx[sel]; xh = xl + 15.0
        yl = ty * 16 + 0.5 - my[sel]; yh = yl + 15.0
        global_sel = sel
        Asel, Bsel, Csel = A[sel], Bm[sel], Cc[sel]
        A_, B_, C_ = A, Bm, Cc
        A, Bm, Cc = Asel, Bsel, Csel
        q = qmin(xl, xh, yl, yh)
        A, Bm, Cc = A_, B_, C_
        kept += int((q <= 9.0 * 1.001).sum())
print("ellipse-meeting pairs", kept, "fraction", kept / total)
