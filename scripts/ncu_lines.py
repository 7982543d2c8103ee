"""Aggregate an ncu 'source --print-source cuda,sass' CSV by CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
by_file = {}
cur_file = None
hdr = None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
line_no = None
src_text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    # rows: CUDA line rows have Line No in col 0; SASS rows follow with empty col 0?
    ln, src = r[0], r[1]
    if ln.strip():
        line_no = (cur_file, int(ln))
        src_text[line_no] = src
        try:
            ie = float(r[hdr.index("Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            ie, st = 0.0, 0.0
        agg[line_no][0] += ie
        agg[line_no][1] += st
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
for key, (ie, st, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    f, ln = key
    print(f"{ie / tot_i * 100:5.1f}% inst {st / tot_s * 100:5.1f}% stall {f.split('/')[-1]}:{ln:<4} {src_text[key].strip()[:90]}")
