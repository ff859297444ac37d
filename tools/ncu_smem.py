"""Per-source-line shared-memory wavefronts (actual / ideal) from an ncu source-page CSV.

ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
python tools/ncu_smem.py src.csv FILE.cu [units]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
path = hdr = None
wf = collections.Counter()
ideal = collections.Counter()
src = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r or not r[0].isdigit() or path != want:
        continue
    k = int(r[0])
    src[k] = r[1]
    try:
        wf[k] += float(r[hdr["L1 Wavefronts Shared"]] or 0)
        ideal[k] += float(r[hdr["L1 Wavefronts Shared Ideal"]] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(wf.values()) or 1.0
print(f"shared wavefronts per unit {tot / units:.0f} (ideal {sum(ideal.values()) / units:.0f})")
for k in sorted(src):
    if wf[k] / tot > 0.01:
        print(f"{k:5d} {wf[k] / units:8.0f} ideal {ideal[k] / units:8.0f}  {src[k].strip()[:80]}")
