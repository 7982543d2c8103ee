"""Top source lines by warp-stall samples from an `ncu --page source --csv --print-source cuda,sass` export."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = "?"
agg = []
tot = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            s = int(r[4]); ni = int(r[7])
        except ValueError:
            continue
        tot += s
        agg.append((s, ni, f, int(r[0]), r[1].strip()[:90]))
agg.sort(reverse=True)
print("total samples", tot)
for s, ni, f, ln, src in agg[:top]:
    print(f"{100*s/tot:5.1f}% {ni/1e6:8.2f}M {f}:{ln} {src}")
