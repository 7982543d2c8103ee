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


GOLDEN_SETS = sorted(p.name for p in GOLDEN.iterdir() if (p / "golden.npz").exists())


@pytest.fixture(params=GOLDEN_SETS)
def golden(request):
    return Golden(request.param)


def rel_err(got, want, floor=1e-8):
    """tests/test_helpers.hpp:124-127 rel_err with the 1e-8 denominator floor."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), floor)
