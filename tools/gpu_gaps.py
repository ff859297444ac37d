"""GPU idle gaps inside one device-resident pipeline step at config-3 size (torch.profiler / CUPTI):
every gap > 50 us between consecutive kernels / copies, with the kernel that follows it."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth
from torch.profiler import profile, ProfilerActivity
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
x, lab = synth.generate(cfg)
X = torch.from_numpy(x).cuda()
k = synth.num_clusters(cfg)
def step():
    S = simmatrix.pearson_similarity_device(X)
    return P.run_stages(P.PipelineConfig(apsp_mode="hub", k=k), S, None, sync_stages=False)
for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = ev[0].time_range.end
for e in ev[:3]:
    print(f"first: {(e.time_range.start - t0)/1e3:8.3f} ms dur {(e.time_range.end - e.time_range.start)/1e3:.3f} {e.name[:70]}")
prev = ev[0].name
busy = 0.0
tot_gap = 0.0
for e in ev[1:]:
    gap = e.time_range.start - end
    if gap > 50:
        tot_gap += gap
        print(f"gap {gap/1e3:7.3f} ms at {(e.time_range.start - t0)/1e3:8.3f} ms after {prev[:40]} before {e.name[:60]}")
    end = max(end, e.time_range.end)
    prev = e.name
print(f"span {(end - t0)/1e3:.3f} ms, gaps > 50 us total {tot_gap/1e3:.3f} ms")
