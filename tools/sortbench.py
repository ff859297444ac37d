"""Row-sort timing + check against torch's stable sort (TG_LIB selects a variant library).

python tools/sortbench.py [n ...]   (config-3 generator; config 4 tie stress at n=4000 too)
"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2408_09399_b200 import simmatrix, synth, _native as N

N.load()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def check(S, order):
    n = S.shape[0]
    for r0 in range(0, n, 2048):
        r1 = min(n, r0 + 2048)
        blk = S[r0:r1]
        idx = torch.sort(-blk, dim=1, stable=True).indices.to(torch.int32)
        rows = torch.arange(r0, r1, device=S.device, dtype=torch.int32)[:, None]
        keep = idx != rows
        ref = idx[keep].view(r1 - r0, n - 1)
        if not torch.equal(ref, order[r0:r1]):
            bad = (ref != order[r0:r1]).any(1).nonzero()[0].item() + r0
            return f"MISMATCH row {bad}"
    return "ok"


def run(cfg, n):
    x, _ = synth.generate(cfg, n=n)
    S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
    ts = []
    for rep in range(6):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        order, _ = simmatrix.sort_rows_device(S, with_screen=True)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts[1:]))
    byt = 8 * n * n + 4 * n * (n - 1)
    print(f"cfg{cfg} n={n}: {ms:.4f} ms  {byt / ms / 1e6:.1f} GB/s  {n * (n - 1) / ms / 1e6:.1f} Gkeys/s  {check(S, order)}",
          flush=True)
    del S, order
    torch.cuda.empty_cache()


sizes = [int(a) for a in sys.argv[1:]] or [10000]
for n in sizes:
    run(3, n)
run(4, 4000)
