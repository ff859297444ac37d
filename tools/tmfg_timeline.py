"""Per-insertion timeline of the TMFG kernel: time, rounds, refills and pops per slice of the
insertion sequence.  Needs the timeline builds of tmfg.cu (-DTM_PROFILE=1 -DTM_TS=1..4 as
paper_2408_09399_b200/_lib/libtmfg_b200_ts{1..4}.so; TM_TS selects what host_fid records)."""
import os, subprocess, sys, json
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
if len(sys.argv) > 3:   # worker: one variant
    sys.path.insert(0, str(REPO))
    os.environ["TG_LIB"] = str(REPO / "paper_2408_09399_b200" / "_lib" / f"libtmfg_b200_ts{sys.argv[3]}.so")
    import torch, numpy as np
    from paper_2408_09399_b200 import simmatrix, synth, tmfg, _native as N
    n, cfg = int(sys.argv[1]), int(sys.argv[2])
    N.load()
    x, _ = synth.generate(cfg, n=n)
    S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
    order, rowsum = simmatrix.sort_rows_device(S)
    clique = tmfg.initial_clique_device(S, rowsum)
    for rep in range(2):
        out = tmfg.build_tmfg_heap_device(S, order, clique)
    torch.cuda.synchronize()
    print(json.dumps(out["host_fid"].cpu().numpy().astype("int64").tolist()))
    sys.exit(0)
import numpy as np
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cols = {}
for v, name in ((1, "clock"), (2, "rounds"), (3, "refills"), (4, "pops")):
    o = subprocess.run([sys.executable, __file__, str(n), str(cfg), str(v)], capture_output=True, text=True)
    cols[name] = np.array(json.loads(o.stdout.strip().splitlines()[-1]), dtype=np.int64)
ts = ((cols["clock"] - cols["clock"][0]) & 0xffffffff) * 64 / 1.965e6   # ms
m = len(ts)
marks = sorted(set([0, m // 10, m // 4, m // 2, 3 * m // 4, m * 9 // 10, m * 95 // 100, m - 1000, m - 500, m - 200, m - 100, m - 50, m - 1]))
print(f"{'insertions':>16} {'ms':>8} {'us/ins':>8} {'rounds/ins':>10} {'pops/ins':>9} {'refills':>8} {'us/round':>8}")
for a, b in zip(marks[:-1], marks[1:]):
    d = b - a
    dr = cols["rounds"][b] - cols["rounds"][a]
    print(f"{a:7d}..{b:7d} {ts[b]-ts[a]:8.2f} {1e3*(ts[b]-ts[a])/d:8.2f} {dr/d:10.2f} {(cols['pops'][b]-cols['pops'][a])/d:9.1f} "
          f"{cols['refills'][b]-cols['refills'][a]:8d} {1e3*(ts[b]-ts[a])/max(dr,1):8.2f}")
