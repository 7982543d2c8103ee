"""Diagnostic: the batch-4 4K step vs the reference, view by view."""
import sys, subprocess, tempfile
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from conftest import REF_DUMP
from capi_helpers import camera_from_record
from paper_2406_11836_b200 import engine
out = tempfile.mkdtemp()
args = dict(scene="synth", count=600, w=int(sys.argv[1]), h=int(sys.argv[2]), n_views=64, seed=31, kd=2, mode="oracle",
            view=0, perturb=7, batch_views="0,16,33,48")
subprocess.run([str(REF_DUMP)] + [f"{k}={v}" for k, v in args.items()] + ["dump_batch", "save_scene", "dump_table", f"out={out}"], check=True)
z = {k: np.load(f"{out}/{k}.npy") for k in ["scene_id","scene_mu","scene_log_scale","scene_rotation","scene_opacity_logit","scene_sh","batch_cameras","batch_targets","batch_loss"]}
s = engine.Splats(z["scene_id"], z["scene_mu"], z["scene_log_scale"], z["scene_rotation"], z["scene_opacity_logit"], z["scene_sh"])
cams = [camera_from_record(r) for r in z["batch_cameras"]]
mgr = engine.Manager(s, engine.train_config(kd_depth=2), engine.render_options(oracle=True))
ls = []
for v, c in enumerate(cams):
    rgb, t = mgr.render(c)
    l, _, _ = mgr.ctx.loss(rgb, z["batch_targets"][v])
    ls.append(l)
    print("view", v, "loss", l, "rgb mean", float(rgb.mean()), "target mean", float(z["batch_targets"][v].mean()), "T min", float(t.min()))
print("mean per-view loss", np.mean(ls), "ref batch loss", float(z["batch_loss"][0]))
mgr.close()
mgr = engine.Manager(s, engine.train_config(kd_depth=2, batch_size=4), engine.render_options(oracle=True))
print("batch step loss", mgr.train_step(cams, z["batch_targets"])["loss"])
mgr.close()
mgr = engine.Manager(s, engine.train_config(kd_depth=2, batch_size=4), engine.render_options(oracle=True))
tdev = mgr.ctx.upload_targets(z["batch_targets"])
print("batch step loss (device targets)", mgr.train_step(cams, None, targets_device_ptr=tdev)["loss"])
