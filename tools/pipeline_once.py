"""One device-resident pipeline pass at config-3 size (for ncu launch lists)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
mode = "hub" if cfg in (3, 5) else "exact"
x, lab = synth.generate(cfg, n=n)
X = torch.from_numpy(x).cuda()
k = synth.num_clusters(cfg)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S = simmatrix.pearson_similarity_device(X)
    rep_, g, d, flat = P.run_stages(P.PipelineConfig(apsp_mode=mode, k=k), S, None, sync_stages=True)
    torch.cuda.synchronize()
    print(f"pass {rep}: {(time.perf_counter() - t0) * 1e3:.1f} ms", {kk: round(v * 1e3, 2) for kk, v in rep_.stage_seconds.items()})
