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


# Float-atomic accumulation order differs from the reference's chunked
# sequential sums: gradient entries whose magnitude is below
# NOISE_FLOOR x (max |g| of that field in that subset) are cancellation-
# dominated and are compared absolutely at that floor instead of relatively.
NOISE_FLOOR = 1e-3
GRAD_RTOL = 1e-3


def grad_errors(got, want, floor_frac=NOISE_FLOOR):
    want = np.asarray(want, np.float64)
    scale = float(np.abs(want).max()) if want.size else 0.0
    return rel_err(got, want, floor=max(floor_frac * scale, 1e-30))


def adam_lr_rows(cfg, sh_coeffs):
    """Per-parameter learning rates in GradBuffers field order (optim.hpp:104-126) at step 1."""
    return {"mu": cfg.lr_position_start, "log_scale": cfg.lr_scale, "rotation": cfg.lr_rotation,
            "opacity_logit": cfg.lr_opacity,
            "sh": np.array([cfg.lr_sh_dc] + [cfg.lr_sh_rest] * (sh_coeffs - 1))[:, None]}


def post_adam_ok(got, want, grad_ref, lr, rtol=GRAD_RTOL, floor_frac=NOISE_FLOOR):
    """Post-Adam parameters: rel_err <= rtol where the reference gradient is above
    the noise floor; elsewhere Adam's normalised step may take the other sign,
    so |delta| <= 2 lr + rtol |want| (optim.hpp:90-97: the first step is +-lr)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    g = np.abs(np.asarray(grad_ref, np.float64))
    scale = g.max() if g.size else 0.0
    noisy = g <= floor_frac * scale
    lr = np.broadcast_to(np.asarray(lr, np.float64), want.shape)
    e = rel_err(got, want)
    ok_strict = (e <= rtol) | noisy
    ok_noisy = (~noisy) | (np.abs(got - want) <= 2.0 * lr * (1 + 1e-3) + rtol * np.abs(want))
    return ok_strict & ok_noisy, e, noisy
