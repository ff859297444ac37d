"""Aggregate ncu warp-stall samples per CUDA source line from a --print-source cuda,sass CSV."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
path = None
agg = collections.Counter()
src = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or r[0] in ("Function Name",):
        continue
    if r[0] != "-" and r[0].isdigit():
        key = (path, int(r[0]))
        src[key] = r[1]
        try:
            agg[key] += float(r[4] or 0)
        except ValueError:
            pass
tot = sum(agg.values())
print("total", tot)
for (f, l), s in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{s/tot*100:5.1f}% {f}:{l}  {src[(f, l)][:90]}")
