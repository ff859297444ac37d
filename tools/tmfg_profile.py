"""Time the TMFG kernel at config-3 size and print its internal phase profile."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import simmatrix, synth, tmfg, _native as N
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N.load()
x, _ = synth.generate(cfg, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, rowsum = simmatrix.sort_rows_device(S)
clique = tmfg.initial_clique_device(S, rowsum)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = tmfg.build_tmfg_heap_device(S, order, clique)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
st = out["stats"].cpu().numpy()
names = ["pops", "refreshes", "gain_inc", "status", "a", "b", "c", "d", "rounds", "refills", "cyc_par_done", "cyc_replay_done",
         "cyc_merge", "cyc_insert", "cyc_refill", "pool"]
d = {k: int(v) for k, v in zip(names, st)}
d["ms"] = dt * 1e3
d["us_per_insert"] = dt * 1e6 / (n - 4)
print(json.dumps(d))
