"""Run the DBHT hierarchy stage once for a BASELINE config (for ncu captures of its kernels)."""
import sys
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
w = P.to_weighted(g, S)
o = P.apsp_hub(w)
tree = P.build_bubble_tree(g)
dt = P.orient_edges(tree, S)
asg = P.assign_vertices(g, dt, o)
d = P.build_hierarchy(asg, dt, o)
torch.cuda.synchronize()
print("ok")
