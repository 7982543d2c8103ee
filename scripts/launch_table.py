"""Per-launch table from an `ncu --metrics ... --csv --log-file` capture (long format)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i0]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[i0 + 1:]:
    if len(r) != len(h):
        continue
    e = d.setdefault(r[ii], {"name": r[ki]})
    e[r[mi]] = r[vi].replace(",", "")
for k, e in d.items():
    n = e["name"].split("(")[0].replace("void ", "").replace("dgs_b200::", "").replace("<unnamed>::", "")[-60:]
    t = float(e.get("gpu__time_duration.sum", 0)) / 1e3
    rd = float(e.get("dram__bytes_read.sum", 0)) / 1e6
    wr = float(e.get("dram__bytes_write.sum", 0)) / 1e6
    ins = float(e.get("smsp__inst_executed.sum", 0)) / 1e6
    print(f"{k:>4} {n:60s} {t:9.1f} us  rd {rd:8.1f} MB  wr {wr:8.1f} MB  inst {ins:8.1f} M")
