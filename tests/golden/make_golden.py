"""Regenerate the committed golden fixtures from the reference itself.

Runs oracle/_ref/ref_dump (the UNMODIFIED reference headers compiled against
the Eigen shim, see oracle/Makefile) and stores its outputs here with a
manifest of the exact arguments.  Needs /root/reference only at build time of
oracle/_ref (this container); the fixtures themselves travel with the repo.
"""
import json
import shutil
import subprocess
import sys

import numpy as np
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = HERE.parent.parent / "oracle" / "_ref" / "ref_dump"

SETS = {
    # C1-style synthetic scene, 2-way KD split, oracle options (stop = 0): contributor lists exact.
    "g1_synth_kd1_oracle": dict(scene="synth", count=2000, w=64, h=48, n_views=8, seed=11, kd=1, mode="oracle",
                                view=0, perturb=5),
    # clustered scene, 4-way split, default options (early termination), another view.
    "g2_synth_kd2_default": dict(scene="synth", count=1200, clustered=1, w=80, h=64, n_views=8, seed=7, kd=2,
                                 mode="default", view=3, perturb=9),
    # tests/test_helpers.hpp random_splats (SH degree 1, large splats), monolithic.
    "g3_random_kd0_oracle": dict(scene="random", count=60, seed=2, sh_degree=1, w=24, h=24, n_views=4, kd=0,
                                 mode="oracle", view=1, perturb=3),
    # Manager::train_step with a batch of 3 views (summed GradBuffers, one Adam step), 4-way split.
    "g7_synth_kd2_batch3": dict(scene="synth", count=1500, w=56, h=40, n_views=8, seed=13, kd=2, mode="default",
                                view=0, perturb=6, dump_batch=1, batch_views="0,3,5"),
    # camera_z_order fast mode (splat.hpp:126, raster.hpp:162): per-view depth order, ties by id.
    "g8_synth_kd1_zorder": dict(scene="synth", count=2000, w=64, h=48, n_views=8, seed=19, kd=1, mode="oracle",
                                view=5, perturb=8, z_order=1),
    # non-zero background, 8-way split, default options.
    "g4_synth_kd3_bg": dict(scene="synth", count=2000, w=48, h=48, n_views=6, seed=23, kd=3, mode="default",
                            view=2, perturb=4, bg_r=0.2, bg_g=0.5, bg_b=0.9),
}
# init_from_pointcloud (trainer.hpp:24-91) on a numpy-generated cloud (committed with the fixture)
INIT_SETS = {
    # target <= points: std::sample without replacement, no jitter
    "g5_init_pc_sample": dict(points=6000, target=4000, seed=17, sh_degree=3, cloud_seed=5),
    # target > points: uniform picks with replacement + 1e-3 * bbox-diagonal jitter
    "g6_init_pc_oversample": dict(points=1500, target=5000, seed=29, sh_degree=1, cloud_seed=6),
}
PLY_SETS = {"g3_random_kd0_oracle"}
DUMPS = ["save_scene", "dump_table", "dump_orders", "dump_project", "dump_partials", "contributors", "dump_render",
         "dump_step", "dump_g2d"]


def run(name, args, out):
    tmp = out / "_npy"
    tmp.mkdir()
    argv = [str(REF)] + [f"{k}={v}" for k, v in args.items()] + DUMPS + [f"out={tmp}"]
    if name in PLY_SETS:  # the reference's save_splats_ply of the (perturbed) scene, io.hpp:257-297
        argv.append(f"save_ply={out / 'scene_perturbed.ply'}")
    subprocess.run(argv, check=True)
    arrays = {f.stem: np.load(f) for f in sorted(tmp.glob("*.npy"))}
    np.savez_compressed(out / "golden.npz", **arrays)
    shutil.rmtree(tmp)
    (out / "manifest.json").write_text(json.dumps({"name": name, "args": args, "dumps": DUMPS,
                                                   "generator": "oracle/_ref/ref_dump"}, indent=1))


def run_init(name, args, out):
    tmp = out / "_npy"
    tmp.mkdir()
    rng = np.random.default_rng(args["cloud_seed"])
    pts = (rng.random((args["points"], 3)) * 2 - 1).astype(np.float32)
    pts[: args["points"] // 3] *= 0.2  # a dense cluster: uneven neighbour distances
    cols = rng.random((args["points"], 3)).astype(np.float32)
    np.save(tmp / "pc_points.npy", pts)
    np.save(tmp / "pc_colors.npy", cols)
    argv = [str(REF), "init_pc=1", f"pc_points={tmp / 'pc_points.npy'}", f"pc_colors={tmp / 'pc_colors.npy'}",
            f"target={args['target']}", f"seed={args['seed']}", f"sh_degree={args['sh_degree']}", f"out={tmp}"]
    subprocess.run(argv, check=True)
    arrays = {f.stem: np.load(f) for f in sorted(tmp.glob("*.npy"))}
    np.savez_compressed(out / "golden.npz", **arrays)
    shutil.rmtree(tmp)
    (out / "manifest.json").write_text(json.dumps({"name": name, "args": args, "dumps": ["init_pc"],
                                                   "generator": "oracle/_ref/ref_dump init_pc"}, indent=1))


def main():
    if not REF.exists():
        sys.exit("build oracle/_ref first: make -C oracle ref")
    only = sys.argv[1:]
    for name, args in SETS.items():
        if only and name not in only:
            continue
        out = HERE / name
        shutil.rmtree(out, ignore_errors=True)
        out.mkdir(parents=True)
        run(name, args, out)
        print(name, sum(f.stat().st_size for f in out.iterdir()) // 1024, "KiB")
    for name, args in INIT_SETS.items():
        if only and name not in only:
            continue
        out = HERE / name
        shutil.rmtree(out, ignore_errors=True)
        out.mkdir(parents=True)
        run_init(name, args, out)
        print(name, sum(f.stat().st_size for f in out.iterdir()) // 1024, "KiB")


if __name__ == "__main__":
    main()
