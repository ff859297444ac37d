"""Time tg_nn_chain_batch on single random symmetric matrices (CUDA events)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2408_09399_b200 import linkage
for m in [int(a) for a in sys.argv[1:]] or (64, 256, 512, 1056, 2048, 4096, 5906):
    rng = np.random.default_rng(m)
    A = rng.random((m, m))
    D = (A + A.T) / 2
    np.fill_diagonal(D, 0.0)
    blocks = torch.from_numpy(D.reshape(-1).copy()).cuda()
    ts = []
    for rep in range(3):
        b = blocks.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        le, ri, he, mo = linkage.nn_chain_raw_batch(b, np.array([m]), np.array([0], dtype=np.int64))
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    # steps of the NN-chain on the CPU (same algorithm) to get per-step cost
    print(f"m={m}: {min(ts):.3f} ms, {min(ts) * 1e3 / (m - 1):.2f} us per merge")
