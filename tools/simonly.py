"""Run the fast (TMA SYRK) Pearson similarity once at a BASELINE config's size (for ncu captures)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import simmatrix, synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
x, _ = synth.generate(cfg)
X = torch.from_numpy(x).cuda()
for _ in range(2):
    S = simmatrix.pearson_similarity_device(X)
torch.cuda.synchronize()
print("ok", x.shape, float(S[0, 1]))
