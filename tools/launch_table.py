"""Markdown table of an ncu launch list (--metrics gpu__time_duration.sum --csv).

python tools/launch_table.py launches.csv [top]
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    k = r[4].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    agg[k][0] += 1
    agg[k][1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
print(f"Total kernel time in the capture: {tot / 1e6:.1f} ms over {len(rows)} launches.\n")
print("| kernel | launches | total ms | share |")
print("|---|---:|---:|---:|")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"| `{k}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
