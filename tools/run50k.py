"""Config-5 (n = 50k) pipeline passes with per-stage times (device-resident S)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
x5, _ = synth.generate(5)
X5 = torch.from_numpy(x5).cuda()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    S5 = simmatrix.pearson_similarity_device(X5)
    rep5, _, _, _ = P.run_stages(P.PipelineConfig(apsp_mode="hub", k=synth.num_clusters(5)), S5, None, sync_stages=True)
    torch.cuda.synchronize()
    print(round((time.perf_counter() - t0) * 1e3, 1), {k: round(v * 1e3, 1) for k, v in rep5.stage_seconds.items()}, flush=True)
    del S5
    torch.cuda.empty_cache()
