"""Summarise a scripts/profile_round.sh output directory into profiles/.

  python scripts/summarize_profile.py gpurun_out/prof1 r1

Writes profiles/<tag>_launches.csv (every kernel launch of one training step:
gpu__time_duration and DRAM bytes, serialised and cold-cache under ncu),
profiles/<tag>_ncu_full_summary.csv (ncu --set full, last launch of each hot
kernel: time, DRAM bytes, issue/occupancy, top stall reasons),
profiles/<tag>_bench.json (the bench line) and profiles/traffic.json
(dram read + write bytes per launch, the `traffic` field of bench.py).
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

src = Path(sys.argv[1])
tag = sys.argv[2] if len(sys.argv) > 2 else "r1"
dst = Path(__file__).resolve().parent.parent / "profiles"
dst.mkdir(exist_ok=True)

# ---- launch list: keep the launches of the last training step ----------------
rows = list(csv.reader(open(src / "launches.csv")))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i0]
per = {}
for r in rows[i0 + 1:]:
    if len(r) < len(hdr):
        continue
    key = int(r[0])
    d = per.setdefault(key, {"kernel": r[hdr.index("Kernel Name")]})
    d[r[hdr.index("Metric Name")]] = (r[hdr.index("Metric Value")], r[hdr.index("Metric Unit")])
ids = sorted(per)
# the last step starts at the last k_preprocess launch
starts = [i for i in ids if "k_preprocess" in per[i]["kernel"]]
step = [i for i in ids if i >= starts[-1]] if starts else ids


def val(d, m, scale_to):
    v, u = d.get(m, ("0", ""))
    v = float(v.replace(",", ""))
    f = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}.get(u, 1.0)
    return v * f / scale_to


with open(dst / f"{tag}_launches.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["launch", "kernel", "time_ms", "dram_read_MB", "dram_write_MB"])
    tot = 0.0
    for i in step:
        d = per[i]
        t = val(d, "gpu__time_duration.sum", 1.0)
        tot += t
        w.writerow([i, d["kernel"][:110], round(t, 4), round(val(d, "dram__bytes_read.sum", 1e6), 2),
                    round(val(d, "dram__bytes_write.sum", 1e6), 2)])
    w.writerow(["total", "", round(tot, 4), "", ""])
print(f"launch list: {len(step)} launches, {tot:.3f} ms serialised")

# ---- full-set summary ------------------------------------------------------------
raw = subprocess.run(["ncu", "-i", str(src / "full.ncu-rep"), "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
last = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("dgs_b200::", "").lstrip("<")
    if "Onesweep" in short:
        short = f"cub::Onesweep(grid {r[hdr.index('Grid Size')]})"
    last[short] = r
traffic = {}
with open(dst / f"{tag}_ncu_full_summary.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel"] + [f"{m} [{units[hdr.index(m)]}]" for m in want if m in hdr] + ["top stalls"])
    for k, r in last.items():
        st = sorted(((float(r[hdr.index(h)] or 0), h) for h in stall), reverse=True)[:3]
        sts = "; ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                        f" {v:.2f}" for v, h in st)
        w.writerow([k] + [r[hdr.index(m)] for m in want if m in hdr] + [sts])
        rd = float(r[hdr.index("dram__bytes_read.sum")]) if "dram__bytes_read.sum" in hdr else 0.0
        wr = float(r[hdr.index("dram__bytes_write.sum")]) if "dram__bytes_write.sum" in hdr else 0.0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
        wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
        traffic[k] = int(rd + wr)
print("full-set kernels:", ", ".join(last))
key_map = {"k_adam_stream4": "adam", "k_preprocess": "preprocess", "k_grad_record": "project_bwd"}
out = {"note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture "
               f"({tag}_ncu_full_summary.csv)"}
if (src / "bench.json").exists():  # the workload these bytes belong to (bench.py matches it)
    cfg = json.loads((src / "bench.json").read_text()).get("config", {})
    out.update({k: cfg.get(k) for k in ("gaussians", "width", "height", "batch", "kd_subsets")})
for k, v in traffic.items():
    for pre, name in key_map.items():
        if k.startswith(pre):
            out[name] = v
(dst / "traffic.json").write_text(json.dumps(out, indent=1) + "\n")
if (src / "bench.json").exists():
    (dst / f"{tag}_bench.json").write_text((src / "bench.json").read_text())
print("wrote", dst)
