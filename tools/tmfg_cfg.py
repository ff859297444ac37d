"""Run the TMFG kernel once on a BASELINE config (or a synth size) and print time + trace hash."""
import sys, time, hashlib
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2408_09399_b200 import simmatrix, synth, tmfg
cfg = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else None
x, _ = synth.generate(cfg, n=n) if n else synth.generate(cfg)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, screen = simmatrix.sort_rows_device(S)
clique = tmfg.initial_clique_device(S, screen)
torch.cuda.synchronize(); t0 = time.perf_counter()
out = tmfg.build_tmfg_heap_device(S, order, clique)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
tr = out["trace"].cpu().numpy()
print(f"cfg {cfg} n {x.shape[0]} ms {dt*1e3:.1f} trace {hashlib.sha256(tr.tobytes()).hexdigest()[:16]} stats {out['stats'][:4].tolist()}", flush=True)
