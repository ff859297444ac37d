"""Repeat the heap TMFG on one S and count traces that differ from the CPU oracle's.

python tools/tmfg_stress.py CONFIG N REPS
"""
import sys, hashlib
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from oracle import oracle as orc
from paper_2408_09399_b200 import simmatrix, synth, tmfg
cfg, n, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
x, _ = synth.generate(cfg, n=n)
Sd = simmatrix.pearson_similarity_refexact_device(x)
S = Sd.cpu().numpy()
ref = orc.build_tmfg_heap(S, orc.sort_neighbor_lists(S))
order, scr = simmatrix.sort_rows_device(Sd)
clique = tmfg.initial_clique_device(Sd, scr)
bad = 0
for r in range(reps):
    try:
        out = tmfg.build_tmfg_heap_device(Sd, order, clique)
        tr = out["trace"].cpu().numpy()
        ok = np.array_equal(tr, ref["trace"])
    except Exception as e:  # noqa: BLE001
        print("exception", type(e).__name__, str(e)[:120], flush=True)
        ok = False
        break
    if not ok:
        bad += 1
        d = np.nonzero((tr != ref["trace"]).any(axis=1))[0]
        print(f"rep {r}: mismatch from trace row {d[0]} of {len(tr)}", flush=True)
print(f"cfg {cfg} n {n}: {bad} / {reps} mismatches", flush=True)
