"""Small end-to-end cases for compute-sanitizer (racecheck / synccheck / memcheck).

Runs, on the oracle-free device path, at sizes where the sanitizer finishes in minutes:
* the fp64 Pearson SYRK + validate + row sort (fk kernel) at n = 300 and 2000,

* the heap TMFG cluster kernel (smem scan state) at n = 300 and 2000,
* APSP (exact and hub), DBHT and the 3-layer hierarchy (NN-chain kernels) at n = 300 / 2000.
Checks digests between the two APSP modes' own repeat runs so a race that changes results is
visible even when the tool reports nothing.

compute-sanitizer --tool racecheck python tools/sanitize_case.py [--sizes 300,2000]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_2408_09399_b200 as P
from paper_2408_09399_b200 import simmatrix, synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="300,2000")
    ap.add_argument("--modes", default="exact,hub")
    args = ap.parse_args()
    P._native.load()
    for n in [int(s) for s in args.sizes.split(",")]:
        x, lab = synth.generate(2, n=n)
        X = torch.from_numpy(x).cuda()
        S = simmatrix.pearson_similarity_device(X)
        for mode in args.modes.split(","):
            digests = set()
            for _ in range(2):
                rep, g, d, flat = P.run_stages(P.PipelineConfig(apsp_mode=mode, k=10), S, None)
                digests.add(rep.digest)
            torch.cuda.synchronize()
            print(f"n={n} mode={mode} digest={sorted(digests)[0][:16]} repeat_equal={len(digests) == 1}",
                  flush=True)
            if len(digests) != 1:
                raise SystemExit("non-deterministic result")
    print("sanitize_case ok")


if __name__ == "__main__":
    main()
