"""Kernel-time table (torch.profiler, CUPTI) of the DBHT hierarchy stage for a BASELINE config.

python tools/prof_stage_kernels.py CONFIG [n]
"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
cfg = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else None
x, lab = synth.generate(cfg, n=n) if n else synth.generate(cfg)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
lists = P.sort_neighbor_lists(S)
g = P.build_tmfg_heap(S, lists)
w = P.to_weighted(g, S)
o = P.apsp_hub(w)
tree = P.build_bubble_tree(g)
dt = P.orient_edges(tree, S)
asg = P.assign_vertices(g, dt, o)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    d = P.build_hierarchy(asg, dt, o)
    torch.cuda.synchronize()
    print("build_hierarchy ms", (time.perf_counter() - t0) * 1e3, flush=True)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    d = P.build_hierarchy(asg, dt, o)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
