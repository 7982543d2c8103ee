"""CPU: splat checkpoints in the 3DGS PLY convention (io.hpp:85-297).  The
writer is byte-identical to the reference's save_splats_ply (fixture written
by oracle/_ref/ref_dump save_ply); the loader reads binary files back bit-exactly
(ascii rows carry the stream's default 6 significant digits, as in the
reference)."""
import filecmp

import numpy as np

from conftest import Golden
from paper_2406_11836_b200 import engine

FIELDS = ("mu", "log_scale", "rotation", "opacity_logit", "sh")


def test_ply_writer_matches_reference_bytes(tmp_path):
    g = Golden("g3_random_kd0_oracle")
    s = g.splats()
    out = tmp_path / "ours.ply"
    engine.save_splats_ply(s, str(out))
    assert filecmp.cmp(out, g.dir / "scene_perturbed.ply", shallow=False)


def test_ply_round_trip_binary_and_ascii(tmp_path):
    s = Golden("g1_synth_kd1_oracle").splats()
    for binary in (True, False):
        path = tmp_path / f"rt_{int(binary)}.ply"
        engine.save_splats_ply(s, str(path), binary=binary)
        t = engine.load_splats_ply(str(path))
        np.testing.assert_array_equal(t.id, np.arange(s.n, dtype=np.uint64))
        for f in FIELDS:
            if binary:
                np.testing.assert_array_equal(getattr(t, f), getattr(s, f), err_msg=f)
            else:  # the reference's ascii rows use the default stream precision (6 digits)
                np.testing.assert_allclose(getattr(t, f), getattr(s, f), rtol=1e-5, atol=1e-6, err_msg=f)


def test_reference_file_loads():
    g = Golden("g3_random_kd0_oracle")
    t = engine.load_splats_ply(str(g.dir / "scene_perturbed.ply"))
    s = g.splats()
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(t, f), getattr(s, f), err_msg=f)
