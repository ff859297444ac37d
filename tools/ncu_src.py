"""Per-source-line summary of an ncu report's source page (stall samples, instructions, top stall reasons).

ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
python tools/ncu_src.py src.csv FILE.cu [units]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
path = None
hdr = None
st = collections.Counter()
ins = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit() or path != want:
        continue
    k = int(r[0])
    src[k] = r[1]
    try:
        st[k] += float(r[4] or 0)
        ins[k] += float(r[7] or 0)
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                reasons[k][h[6:]] += float(r[i] or 0)
    except ValueError:
        pass
ts = sum(st.values()) or 1.0
ti = sum(ins.values()) or 1.0
glob = collections.Counter()
for k in reasons:
    glob.update(reasons[k])
print(f"stall samples {ts:.0f}  instructions {ti:.0f}  per unit {ti / units:.0f}")
print("global:", ", ".join(f"{a} {b / ts * 100:.1f}%" for a, b in glob.most_common(8)))
for k in sorted(src):
    if st[k] / ts > 0.005 or ins[k] / ti > 0.005:
        top = ", ".join(f"{a} {b / max(st[k], 1) * 100:.0f}%" for a, b in reasons[k].most_common(2))
        print(f"{k:5d} st {st[k] / ts * 100:5.1f}% ins {ins[k] / units:8.0f} [{top}]  {src[k].strip()[:70]}")
