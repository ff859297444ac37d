"""Kernel timeline of one build_hierarchy call (torch.profiler / CUPTI): start offset + duration per kernel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
cfg = int(sys.argv[1])
x, lab = synth.generate(cfg)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
lists = P.sort_neighbor_lists(S)
g = P.build_tmfg_heap(S, lists)
o = P.apsp_hub(P.to_weighted(g, S))
dt = P.orient_edges(P.build_bubble_tree(g), S)
asg = P.assign_vertices(g, dt, o)
P.build_hierarchy(asg, dt, o); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    P.build_hierarchy(asg, dt, o); torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = min(e.time_range.start for e in prof.events())
for e in ev:
    print(f"{(e.time_range.start - t0)/1e3:9.3f} ms  dur {(e.time_range.end - e.time_range.start)/1e3:8.3f} ms  {e.name[:70]}")
