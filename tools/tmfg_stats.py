"""Print the TMFG kernel's pops / refreshes / gain increases (and a trace hash) for a config."""
import hashlib, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import simmatrix, synth, tmfg
n = int(sys.argv[1]); cfg = int(sys.argv[2])
x, _ = synth.generate(cfg, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, scr = simmatrix.sort_rows_device(S)
clique = tmfg.initial_clique_device(S, scr)
out = tmfg.build_tmfg_heap_device(S, order, clique)
st = out["stats"].cpu().numpy()
tr = out["trace"].cpu().numpy()
print(n, cfg, "pops", st[0], "refreshes", st[1], "gain_inc", st[2], "rounds", st[8], "trace", hashlib.sha256(tr.tobytes()).hexdigest()[:16])
