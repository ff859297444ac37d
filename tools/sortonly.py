"""Run the row sort once on a config-3-like S (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import simmatrix, synth, _native as N
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
N.load()
x, _ = synth.generate(3, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, rowsum = simmatrix.sort_rows_device(S, with_screen=(sys.argv[2:3] != ['nosum']))
torch.cuda.synchronize()
print("ok", int(order[0, 0]))
