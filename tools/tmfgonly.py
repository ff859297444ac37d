"""One TMFG kernel launch at config-3 size (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import simmatrix, synth, tmfg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
x, _ = synth.generate(3, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, scr = simmatrix.sort_rows_device(S)
clique = tmfg.initial_clique_device(S, scr)
out = tmfg.build_tmfg_heap_device(S, order, clique)
torch.cuda.synchronize()
print("ok", int(out["stats"][0]))
