"""Print the linkage problem sizes of build_hierarchy's three layers at config-3 size."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x, lab = synth.generate(cfg, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
lists = P.sort_neighbor_lists(S)
g = P.build_tmfg_heap(S, lists)
w = P.to_weighted(g, S)
o = P.apsp_hub(w)
tree = P.build_bubble_tree(g)
dt = P.orient_edges(tree, S)
asg = P.assign_vertices(g, dt, o)
vb, vc = asg.vertex_bubble, asg.vertex_converging
bub, cnt = np.unique(vb, return_counts=True)
print("bubbles with members", len(bub), "layer-1 sizes: max", cnt.max(), "sum sq", int((cnt.astype(np.int64) ** 2).sum()),
      "hist", np.bincount(np.minimum(cnt, 10)))
conv_of_bubble = {int(b): int(vc[np.nonzero(vb == b)[0][0]]) for b in bub}
cg = {}
for b, c in conv_of_bubble.items():
    cg.setdefault(c, []).append(b)
m2 = sorted((len(v) for v in cg.values()), reverse=True)
print("conv groups", len(cg), "layer-2 sizes top", m2[:10], "n>48:", sum(1 for s in m2 if s > 48))
print("layer-3 size", len(cg))
