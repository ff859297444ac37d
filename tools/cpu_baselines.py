"""CPU baselines on the GPU box's host cores (recorded in profiles/, not part of bench.py's default run).

* the oracle port (C/OpenMP + numpy restatement of the reference, bit-identical outputs) at
  BASELINE config 5 (n = 50,000, L = 256, hub APSP) on all host threads: per-stage seconds;
* the unmodified Python reference (baseline/_ref, numba, all cores) at config 3 (n = 10,000)
  with its own six stage timers (pipeline.py:25) and pearson_similarity timed separately.

python tools/cpu_baselines.py [--skip-50k] [--skip-python]  -> JSON on stdout
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402  (host_info, _python_reference_once)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-50k", action="store_true")
    ap.add_argument("--skip-python", action="store_true")
    args = ap.parse_args()
    out = {"host": bench.host_info()}
    if not args.skip_50k:
        from oracle import oracle as orc
        from paper_2408_09399_b200 import synth
        orc.set_threads(os.cpu_count() or 1)
        x, _ = synth.generate(5)
        t0 = time.perf_counter()
        S = orc.pearson_similarity(x)
        sim = time.perf_counter() - t0
        r = orc.run_stages(S, synth.num_clusters(5), "hub")
        total = time.perf_counter() - t0
        out["oracle_config5"] = {"total_s": round(total, 2), "similarity_s": round(sim, 2),
                                 "stage_s": {k: round(v, 2) for k, v in r["seconds"].items()},
                                 "digest": r["digest"], "threads": orc.num_threads(),
                                 "kind": "port (C/OpenMP + numpy restatement of the reference)"}
        print(json.dumps(out), flush=True)
        del S
    if not args.skip_python:
        out["python_reference_config3"] = bench._python_reference_once(3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
