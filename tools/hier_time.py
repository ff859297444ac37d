"""Time build_hierarchy alone (device-resident inputs) for a BASELINE config: median of reps."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
cfg = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
x, lab = synth.generate(cfg, n=n) if n else synth.generate(cfg)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
lists = P.sort_neighbor_lists(S)
g = P.build_tmfg_heap(S, lists)
o = P.apsp_hub(P.to_weighted(g, S))
dt = P.orient_edges(P.build_bubble_tree(g), S)
asg = P.assign_vertices(g, dt, o)
ts = []
for _ in range(7):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = P.build_hierarchy(asg, dt, o)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
ts.sort()
print(f"cfg {cfg} n {S.shape[0]} build_hierarchy ms median {ts[3]:.2f} min {ts[0]:.2f}", "digest", hash(d.heights.tobytes()))
