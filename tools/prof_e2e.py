"""cProfile of the public end-to-end call (run_series) at config-3 size."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import synth
from paper_2408_09399_b200.pipeline import run_series
x, lab = synth.generate(3)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rep, d, flat = run_series(x, k=20, apsp_mode="hub")
    torch.cuda.synchronize(); print("run_series ms", (time.perf_counter() - t0) * 1e3, {k: round(v * 1e3, 2) for k, v in rep.stage_seconds.items()})
pr = cProfile.Profile()
pr.enable()
rep, d, flat = run_series(x, k=20, apsp_mode="hub")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
