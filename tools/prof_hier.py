"""cProfile the host side of build_hierarchy at config-3 size."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
x, lab = synth.generate(3, n=n)
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
    print("build_hierarchy s", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
d = P.build_hierarchy(asg, dt, o)
lab2 = P.cut(d, 20)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
