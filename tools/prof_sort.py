"""Kernel table (torch.profiler) of one row sort at size n (config-3 generator)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_09399_b200 import simmatrix, synth, _native as N
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N.load()
x, _ = synth.generate(cfg, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, _ = simmatrix.sort_rows_device(S, with_screen=True)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    order, _ = simmatrix.sort_rows_device(S, with_screen=True)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=50))
