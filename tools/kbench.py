"""Kernel micro-timings on the GPU box (CUDA events, warm-up, L2 flush between reps).

python tools/kbench.py [--n 10000] [--L 512] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import paper_2408_09399_b200 as p
from paper_2408_09399_b200 import _native as N
from paper_2408_09399_b200 import simmatrix, synth, tmfg


def timed(fn, reps, flush):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--L", type=int, default=512)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    N.load()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    out = {}
    x, _ = synth.generate(args.config, n=args.n)
    n, L = x.shape
    X = torch.from_numpy(x).cuda()
    S = simmatrix.pearson_similarity_device(X)
    torch.cuda.synchronize()
    # fp64 similarity
    mn, md = timed(lambda: simmatrix.pearson_similarity_device(X), args.reps, flush)
    flops = n * (n + 1) * L
    out["pearson_ms"] = [mn, md]
    out["pearson_tflops_alg"] = flops / (mn * 1e-3) / 1e12
    # cuBLAS DGEMM reference (full square) for the fp64 peak
    A = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    mn2, _ = timed(lambda: A @ A, 3, flush)
    out["cublas_dgemm_8192_tflops"] = 2 * 8192 ** 3 / (mn2 * 1e-3) / 1e12
    # row sort
    order = torch.empty((n, n - 1), dtype=torch.int32, device="cuda")
    rowsum = torch.empty((2 * n,), dtype=torch.float64, device="cuda")   # row-sum screen
    ws = p._device.Workspace.get(N.size("tg_row_sort_workspace_bytes", n))

    def sort():
        N.call("tg_row_sort_f64", N.ptr(S), n, N.ptr(order), N.ptr(rowsum), N.ptr(ws), ws.numel(), N.stream_ptr())

    def sort_nosum():
        N.call("tg_row_sort_f64", N.ptr(S), n, N.ptr(order), N.ptr(None), N.ptr(ws), ws.numel(), N.stream_ptr())

    mn, md = timed(sort, args.reps, flush)
    byt = 8 * n * n + 4 * n * (n - 1)
    out["sort_ms"] = [mn, md]
    out["sort_gbs"] = byt / (mn * 1e-3) / 1e9
    out["sort_gkeys"] = n * (n - 1) / (mn * 1e-3) / 1e9
    mn, md = timed(sort_nosum, args.reps, flush)
    out["sort_nosum_ms"] = [mn, md]
    out["sort_nosum_gbs"] = byt / (mn * 1e-3) / 1e9
    sort()
    mn, md = timed(lambda: tmfg.initial_clique_device(S, rowsum), args.reps, flush)
    out["clique_screened_ms"] = [mn, md]
    mn, md = timed(lambda: tmfg.initial_clique_device(S, None), args.reps, flush)
    out["clique_exact_all_rows_ms"] = [mn, md]
    # validate
    flags = torch.empty(1, dtype=torch.int32, device="cuda")
    mn, md = timed(lambda: N.call("tg_validate_f64", N.ptr(S), n, N.ptr(flags), N.stream_ptr()), args.reps, flush)
    out["validate_ms"] = [mn, md]
    out["validate_gbs"] = 8 * n * n / (mn * 1e-3) / 1e9
    # plain copy roofline reference
    src = torch.empty(n * n, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    mn, _ = timed(lambda: dst.copy_(src), args.reps, flush)
    out["copy_gbs"] = 16 * n * n / (mn * 1e-3) / 1e9
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
