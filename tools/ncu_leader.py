"""Leader-CTA view of an ncu source-page CSV of the TMFG kernel: stall samples by reason over the
source lines only the leader runs (round loop, window refresh, replay), and the hottest lines."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
ranges = [tuple(int(x) for x in r.split("-")) for r in sys.argv[3].split(",")] if len(sys.argv) > 3 else [(440, 740), (1075, 1270), (1620, 1960)]   # lean refresh, replay_warp, the round loop (line ranges of tmfg.cu at HEAD)
hdr = None; path = None
reasons = collections.Counter(); lines = collections.Counter(); src = {}; inst = collections.Counter()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or not r or not r[0].isdigit() or path != "tmfg.cu":
        continue
    ln = int(r[0])
    if not any(a <= ln <= b for a, b in ranges):
        continue
    d = dict(zip(hdr, r))
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v:
            try: reasons[k] += float(v)
            except ValueError: pass
    try:
        lines[ln] += float(d["Warp Stall Sampling (All Samples)"] or 0)
        inst[ln] += float(d["Instructions Executed"] or 0)
    except ValueError: pass
    src[ln] = r[1]
tot = sum(reasons.values())
print("leader samples", tot)
for k, v in reasons.most_common(): print(f"  {v/tot*100:5.1f}%  {k}")
print("warp-instructions executed in these lines:", sum(inst.values()))
for ln, s in lines.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{s/tot*100:5.1f}%  inst {inst[ln]:10.0f}  {ln}: {src[ln][:100]}")
