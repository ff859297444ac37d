"""Measured fp64 peaks on this B200 (run under gpurun; writes profiles/fp64_peak.json).

* cuBLAS DGEMM: torch.matmul float64 8192^3 (2 N^3 flops), best of 10 after warm-up (burst),
  and back to back for ~4 s (sustained), CUDA events.
* DMMA from registers (tools/micro/dmma_peak): the fp64 tensor pipe with no memory traffic.
  This is the ceiling the similarity SYRK (mma.sync m8n8k4 f64 = DMMA.8x8x4) is measured against.

python tools/fp64_peak.py [--out profiles/fp64_peak.json]
"""

from __future__ import annotations

import argparse
import json
import subprocess
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "fp64_peak.json"))
    args = ap.parse_args()
    N = 8192
    A = torch.randn(N, N, dtype=torch.float64, device="cuda")
    B = torch.randn(N, N, dtype=torch.float64, device="cuda")
    C = torch.empty_like(A)
    for _ in range(3):
        torch.matmul(A, B, out=C)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = 2.0 * N ** 3
    burst = flops / (best * 1e-3) / 1e12
    reps = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(4):
            torch.matmul(A, B, out=C)
        reps += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained = flops * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    out = {"cublas_dgemm_8192_tflops_burst": round(burst, 2),
           "cublas_dgemm_8192_tflops_sustained": round(sustained, 2),
           "gpu_name": torch.cuda.get_device_name(0)}
    exe = ROOT / "tools" / "micro" / "dmma_peak"
    if exe.exists():
        r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
        rows = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
        out["dmma_sweep"] = [x for x in rows if "warps_per_sm" in x]
        peak = [x for x in rows if "dmma_peak_tflops" in x]
        if peak:
            out["dmma_register_peak_tflops"] = peak[0]["dmma_peak_tflops"]
    out["how"] = ("cuBLAS: torch.matmul float64 8192^3, best of 10 (burst) and back to back for 4 s "
                  "(sustained), CUDA events; DMMA: mma.sync.m8n8k4 f64 from registers, 8 chains per warp, "
                  "4-32 warps per SM (tools/micro/dmma_peak.cu)")
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
