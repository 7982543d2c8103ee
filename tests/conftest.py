import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
REF_DUMP = ROOT / "oracle" / "_ref" / "ref_dump"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


class Golden:
    """One committed fixture set produced by oracle/_ref/ref_dump (tests/golden/make_golden.py)."""

    def __init__(self, name: str):
        self.name = name
        self.dir = GOLDEN / name
        self.args = json.loads((self.dir / "manifest.json").read_text())["args"]
        self._z = np.load(self.dir / "golden.npz")

    def __getitem__(self, k):
        return self._z[k]

    def __contains__(self, k):
        return k in self._z.files

    @property
    def oracle_mode(self) -> bool:
        return self.args.get("mode") == "oracle"

    @property
    def bg(self):
        return (self.args.get("bg_r", 0.0), self.args.get("bg_g", 0.0), self.args.get("bg_b", 0.0))

    def splats(self):
        from paper_2406_11836_b200.engine import Splats
        z = self._z
        return Splats(z["scene_id"].copy(), z["scene_mu"].copy(), z["scene_log_scale"].copy(),
                      z["scene_rotation"].copy(), z["scene_opacity_logit"].copy(), z["scene_sh"].copy())

    def camera(self, i=None):
        from paper_2406_11836_b200.capi import Camera
        return Camera.from_record(self._z["scene_cameras"][self.args["view"] if i is None else i])

    def subsets(self):
        return int(1 << self.args.get("kd", 0))


# scene goldens (ref_dump scene dumps); the init_pc fixtures (g5, g6) are used by their own tests
def _manifest(p):
    return json.loads((p / "manifest.json").read_text())


# (the camera_z_order set has its own tests: the C restatement covers the per-ray t order only)
GOLDEN_SETS = sorted(p.name for p in GOLDEN.iterdir()
                     if (p / "golden.npz").exists() and "save_scene" in _manifest(p).get("dumps", [])
                     and not _manifest(p)["args"].get("z_order"))


@pytest.fixture(params=GOLDEN_SETS)
def golden(request):
    return Golden(request.param)


def rel_err(got, want, floor=1e-8):
    """tests/test_helpers.hpp:124-127 rel_err with the 1e-8 denominator floor."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), floor)


GRAD_RTOL = 1e-3

# Rounding allowance of the gradient checks: K_ROUND unit roundoffs (u = 2^-24)
# of the entry's rounding-sensitivity scale B (orc_partial_backward_bound: the
# gradient evaluated with every term in absolute value) — the forward-error
# bound c u B of evaluating the same backward chain in float in another order.
# The reference itself deviates from exact per-splat sums by <= 6.4 u B on the
# goldens (tests/test_oracle_cpu.py test_rounding_bound_covers_reference).
K_ROUND = 16
U_F32 = 2.0 ** -24


def grad_ok(got, want, want_exact, bound, rtol=GRAD_RTOL, k_round=K_ROUND):
    """Gradient parity with the reference's own 1e-8 floor and no noise mask.
    An entry passes when it is within rtol of the reference, or within rtol of
    the same reference arithmetic with exact per-splat sums (oracle
    orc_set_exact_accumulation: the entries where the reference's float
    accumulation is itself off by > rtol), or within k_round u B of the
    reference (the cancellation-limited entries, e.g. quaternion gradients
    after the tangent projection, whose value no float evaluation determines
    to rtol).  Returns (ok, rel_err vs the reference, #admitted by clause 2,
    #admitted by clause 3, max |got - want| / (u B) over the entries beyond rtol)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    e = rel_err(got, want)
    ex = rel_err(got, want_exact)
    diff = np.abs(got - want)
    ub = U_F32 * np.asarray(bound, np.float64)
    c1 = e <= rtol
    c2 = ex <= rtol
    c3 = diff <= k_round * ub
    ok = c1 | c2 | c3
    ratio = float((diff[~c1] / np.maximum(ub[~c1], 1e-45)).max()) if (~c1).any() else 0.0
    return ok, e, int((~c1 & c2).sum()), int((~c1 & ~c2 & c3).sum()), ratio


def oracle_gradients(splats, planes_k, cam_record, oracle_mode, grad_ct, exact=False, bound=False,
                     grad_skip_eps=1e-5):
    """orc_partial_backward (engine.hpp:74-88) on the CPU restatement; exact=1
    sums the adjoints in double (the accumulation-rounding probe); bound=1
    returns the per-entry rounding-sensitivity scale B instead
    (orc_partial_backward_bound)."""
    import ctypes as C
    import oracle_binding as ob
    sc = ob.Scene(splats)
    sub = ob.subspace(planes_k)
    cam = ob.cam_of(cam_record)
    o = ob.opts(oracle_mode, grad_skip_eps=grad_skip_eps)
    gct = np.ascontiguousarray(grad_ct, np.float32)
    ob.lib().orc_set_exact_accumulation(int(exact))
    try:
        gr, arr = ob.empty_grads(splats.n, splats.sh_coeffs)
        fn = ob.lib().orc_partial_backward_bound if bound else ob.lib().orc_partial_backward
        assert fn(C.byref(sc.c), C.byref(sub), C.byref(cam), C.byref(o), ob.p(gct), C.byref(gr)) == 0
    finally:
        ob.lib().orc_set_exact_accumulation(0)
    return arr


def golden_bounds(g, members, scale=1.0):
    """Per subset k: the rounding-sensitivity scale B of every gradient entry of
    the golden's training step (its dC/dT inputs), field -> array."""
    from paper_2406_11836_b200 import engine
    s = g.splats()
    table = engine.build_kdtree(s.mu, g.args.get("kd", 0))
    rec = g["scene_cameras"][g.args["view"]]
    out = []
    for k, idx in enumerate(members):
        gct = np.concatenate([g[f"k{k}_dC"], g[f"k{k}_dT"][..., None]], axis=-1) * scale
        out.append(oracle_gradients(s.take(idx), table.planes[k], rec, g.oracle_mode, gct, bound=True))
    return out


def oracle_step_bounds(splats, members, planes, cam_records, targets, oracle_mode, bg=(0.0, 0.0, 0.0), lam=0.2):
    """The rounding-sensitivity scales of a Manager::train_step (manager.hpp:313-386)
    over the views of a batch: the C restatement's forward, merge, loss (gradient
    x 1/B) and merge adjoint give each subset's dL/d(C_k, T_k) per view, whose
    bounds add (the gradients sum over the views).  Returns per subset field -> B."""
    import ctypes as C
    import oracle_binding as ob
    K, Bv = len(members), len(cam_records)
    o = ob.opts(oracle_mode)
    subs = [ob.subspace(planes[k]) for k in range(K)]
    scenes = [ob.Scene(splats.take(members[k])) for k in range(K)]
    bga = np.asarray(bg, np.float32)
    total = [None] * K
    for v in range(Bv):
        cam = ob.cam_of(cam_records[v])
        W, H = int(cam.width), int(cam.height)
        ct = np.zeros((K, H, W, 4), np.float32)
        for k in range(K):
            assert ob.lib().orc_partial_render(C.byref(scenes[k].c), C.byref(subs[k]), C.byref(cam), C.byref(o),
                                               ob.p(ct[k]), 0, None, None) == 0
        order = np.zeros((H, W, K), np.uint16)
        count = np.zeros((H, W), np.uint16)
        ob.lib().orc_pixel_orders((ob.Sub * K)(*subs), K, C.byref(cam), ob.p(order), ob.p(count))
        rgb = np.zeros((H, W, 3), np.float32)
        ob.lib().orc_merge(ob.p(ct), ob.p(order), ob.p(count), K, W, H, ob.p(bga), ob.p(rgb), None)
        grad = np.zeros_like(rgb)
        means = np.zeros(3, np.float32)
        tgt = np.ascontiguousarray(targets[v], np.float32)
        ob.lib().orc_loss(ob.p(rgb), ob.p(tgt), W, H, C.c_float(lam), ob.p(grad), ob.p(means))
        grad *= np.float32(1.0 / Bv)
        gct = np.zeros((K, H, W, 4), np.float32)
        ob.lib().orc_merge_backward(ob.p(ct), ob.p(order), ob.p(count), K, W, H, ob.p(grad), ob.p(bga), ob.p(gct))
        for k in range(K):
            b = oracle_gradients(splats.take(members[k]), planes[k], cam_records[v], oracle_mode, gct[k], bound=True)
            total[k] = b if total[k] is None else {f: total[k][f] + b[f] for f in b}
    return total


# Legacy noise floor, kept only for the modes the C restatement does not
# model (camera_z_order; the multi-rank and grad_sync tests compare against
# single-rank references): entries below NOISE_FLOOR x max |g| of the field
# count as sign-undetermined.
NOISE_FLOOR = 1e-3


def adam_lr_rows(cfg, sh_coeffs):
    """Per-parameter learning rates in GradBuffers field order (optim.hpp:104-126) at step 1."""
    return {"mu": cfg.lr_position_start, "log_scale": cfg.lr_scale, "rotation": cfg.lr_rotation,
            "opacity_logit": cfg.lr_opacity,
            "sh": np.array([cfg.lr_sh_dc] + [cfg.lr_sh_rest] * (sh_coeffs - 1))[:, None]}


def post_adam_ok(got, want, grad_ref, lr, bound=None, rtol=GRAD_RTOL, floor_frac=NOISE_FLOOR):
    """Post-Adam parameters.  Adam's first step moves each entry by +-lr times
    sign(g) (optim.hpp:90-97), so an entry whose reference gradient sign is not
    determined by float arithmetic — |g| <= K_ROUND u B with B the rounding-
    sensitivity scale (`bound`; without one, the legacy floor_frac x max |g|) —
    may move by +-lr either way: |delta| <= 2 lr + rtol |want|.  Every other
    entry: rel_err <= rtol."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    g = np.abs(np.asarray(grad_ref, np.float64))
    if bound is not None:
        noisy = g <= K_ROUND * U_F32 * np.asarray(bound, np.float64).reshape(g.shape)
    else:
        scale = g.max() if g.size else 0.0
        noisy = g <= floor_frac * scale
    lr = np.broadcast_to(np.asarray(lr, np.float64), want.shape)
    e = rel_err(got, want)
    ok_strict = (e <= rtol) | noisy
    ok_noisy = (~noisy) | (np.abs(got - want) <= 2.0 * lr * (1 + 1e-3) + rtol * np.abs(want))
    return ok_strict & ok_noisy, e, noisy
