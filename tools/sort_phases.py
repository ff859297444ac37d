"""Per-phase cycles of the row sort (debug build with RS_DEBUG_PHASES=1)."""
import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["TG_LIB"] = str(Path(__file__).resolve().parent.parent / "paper_2408_09399_b200" / "_lib" / "libtmfg_b200_rsdbg.so")
import numpy as np
import torch
from paper_2408_09399_b200 import simmatrix, synth, _native as N
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
lib = N.load()
x, _ = synth.generate(3, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
buf = (ctypes.c_longlong * 8)()
for rep in range(3):
    lib.tg_row_sort_debug_phases(buf)
    simmatrix.sort_rows_device(S, with_screen=True)
    torch.cuda.synchronize()
lib.tg_row_sort_debug_phases(buf)
names = ["wait_row", "pass1", "rest (alloc .. rank)", "-", "-", "-", "end barrier"]
per_row = [buf[k] / n for k in range(7)]
print({names[k]: round(per_row[k]) for k in range(7)}, "total", round(sum(per_row)))
