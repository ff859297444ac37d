"""bench.py -- TMFG-DBHT on B200: one pipeline pass per step (BASELINE.json config 3).

Workload (BASELINE.json configs[2], the headline size): n = 10,000 clustered time
series of length L = 512 (20 Dirichlet(1) clusters, random-walk prototypes,
N(0,1) x U(0.5,2) noise, z-normalised; seeded synthetic data standing in for the
paper's UCR workloads), hub-approximate APSP.

A step = fp64 Pearson similarity -> validation -> per-row neighbour sort (+ fused
clique row sums) -> heap TMFG -> CSR -> hub APSP -> bubble tree / orientation /
assignment -> 3-layer complete-linkage dendrogram -> cut; the dendrogram and the
labels are read back to the host.

  value  : device-resident step time (series already in HBM), ms, lower is better
  e2e    : the same through the public API with HOST buffers (H2D of the series,
           D2H of dendrogram + labels inside the timed region)
  roofline: the row-sort kernel (the metric's second half) against measured HBM
  cpu_baseline: the CPU oracle (C + numpy restatement of the reference) on this
           host's cores, one full step
Multi-GPU: the path does not shard (the TMFG insertion chain is serial), so
`--gpus N` runs N independent replicas (different seeds), no collective in the
data path ("replicas only"); value is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

METRIC = "TMFG-DBHT wall ms at n=10k; row-sort Gkeys/s & fraction of HBM roofline"
UNIT = "ms"


def _peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6458.1)), "measured"
    return 6650.0, "fallback"


class NvmlSampler:
    """SM clock / throttle reasons sampled in-process through NVML (nvidia_ml_py) every 50 ms.

    Preferred over the nvidia-smi subprocess below: one `nvidia-smi --query-gpu` pass holds driver
    locks for tens of ms, and a CUDA call of the step's host phase (the hierarchy stage makes
    hundreds) that lands behind it stalls -- two rounds of measurements read 36-50 ms outliers in
    single steps with the subprocess sampler and none without it."""

    def __init__(self, index: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        # NVML enumerates physical devices: honour CUDA_VISIBLE_DEVICES when it is a plain index list
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        phys = int(ids[index]) if ids and index < len(ids) and ids[index].isdigit() else index
        self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
        self.rows = []
        self._first = 0
        self._stop = threading.Event()
        self._thr = None

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((float(sm), float(mx), int(rs)))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.05)

    def start(self):
        self._sample()   # fails here (caught by the caller) rather than silently in the thread
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def wait_first(self, timeout: float = 5.0):
        return self

    def mark(self):
        self._first = len(self.rows)
        return self

    def stop(self) -> dict:
        self._stop.set()
        if self._thr is not None:
            self._thr.join(timeout=1.0)
        rows = self.rows[self._first:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        nv = self.nv
        bits = {"hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4)}
        reasons = sorted({k for r in rows for k, b in bits.items() if r[2] & b})
        return {"sm_mhz": statistics.median([r[0] for r in rows]), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "sampler": "nvml"}


def make_sampler(index: int):
    try:
        return NvmlSampler(index).start()
    except Exception:
        return ClockSampler(index).start()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (fallback without NVML)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def wait_first(self, timeout: float = 5.0):
        """Block until nvidia-smi has produced a sample (its start-up queries the driver and can
        stall CUDA calls for tens of ms: keep that out of the timed region)."""
        t0 = time.perf_counter()
        while self._proc is not None and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)
        return self

    def mark(self):
        """Samples before this call are discarded: only the timed region's samples count."""
        self._first = len(self.rows)
        return self

    def stop(self) -> dict:
        if self._proc is not None:
            time.sleep(0.25)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()
        self.rows = self.rows[getattr(self, "_first", 0):]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of a per-rank timing over all ranks (works over nccl or gloo)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_seed(rank: int) -> int:
    """Replicas-only scaling: every rank clusters its own synthetic instance."""
    from paper_2408_09399_b200 import synth
    return synth.DEFAULT_SEED + rank


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ B200 arm
def run_b200(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    import paper_2408_09399_b200 as P
    from paper_2408_09399_b200 import _native as N
    from paper_2408_09399_b200 import apsp, dbht, linkage, simmatrix, synth, tmfg
    from paper_2408_09399_b200.pipeline import run_series

    N.load()
    cfg = args.config
    x_host, labels = synth.generate(cfg, n=args.n, seed=replica_seed(rank))
    n, L = x_host.shape
    k = synth.num_clusters(cfg)
    mode = "hub" if cfg in (3, 5) else args.apsp
    X = torch.from_numpy(x_host).to(device)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)  # > L2 (126 MB)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    # S (8n^2 B) and order (4n^2 B) are output buffers allocated once, as a serving process
    # would: otherwise the caching allocator's occasional cudaMalloc for 1.2 GB lands inside
    # the similarity stage (2 -> up to 14 ms); the e2e path below still allocates per call
    S_buf = torch.empty((n, n), dtype=torch.float64, device=device)
    order_buf = torch.empty((n, n - 1), dtype=torch.int32, device=device)

    def step(record: dict | None):
        """One device-resident pipeline pass with per-stage CUDA events."""
        marks = [ev() for _ in range(8)]
        marks[0].record()
        S = simmatrix.pearson_similarity_device(X, out=S_buf)
        marks[1].record()
        simmatrix.validate_device(S)
        order, screen = simmatrix.sort_rows_device(S, with_screen=True, out=order_buf)
        marks[2].record()
        clique = tmfg.initial_clique_device(S, screen)
        out = tmfg.build_tmfg_heap_device(S, order, clique)
        marks[3].record()
        graph = tmfg.TmfgGraph(n=n, edges=out["edges"], weights=tmfg.edge_weights_device(S, out["edges"]),
                               initial_clique=clique, trace=out["trace"], faces=out["faces"], variant="heap",
                               host_fid=out["host_fid"], S_device=S)
        graph._S_host = S
        ip, nb, ln, st = apsp.to_weighted_device(S, out["edges"], n)
        w = apsp.WeightedTmfg(n=n, indptr=ip, neighbors=nb, lengths=ln, strength=st)
        oracle = apsp.apsp_hub(w) if mode == "hub" else apsp.apsp_exact(w)
        marks[4].record()
        tree = dbht.build_bubble_tree(graph)
        dtree = dbht.orient_edges(tree, S)
        asg = dbht.assign_vertices(graph, dtree, oracle)
        marks[5].record()
        d = dbht.build_hierarchy(asg, dtree, oracle)
        flat = linkage.cut(d, k)
        marks[6].record()
        torch.cuda.synchronize()
        if record is not None:
            names = ["similarity", "validate+sort", "tmfg_insertion", "apsp", "dbht_assign", "linkage"]
            for i, nm in enumerate(names):
                record.setdefault(nm, []).append(marks[i].elapsed_time(marks[i + 1]))
        return d, flat, S, order

    # the clock sampler starts before the warm-up and has answered once before the timed region
    sampler = make_sampler(local) if rank == 0 else None
    # warm-up (also the sort-kernel timing source below)
    for _ in range(max(args.warmup, 0)):
        step(None)
    torch.cuda.synchronize()
    if sampler:
        sampler.wait_first().mark()

    # ---- timed region (device-resident).  The interpreter's cyclic garbage collector is run
    # before, and paused through, the timed measurements (steps, sort roofline, e2e, n = 50k): a
    # generation-2 collection (12-35 ms here) landing in the hierarchy's host phase stalled the
    # GPU inside one step (one run read a 159 ms step among 93 ms ones); no pipeline work is
    # skipped, and reference counting still frees every buffer.
    gc.collect()
    gc.disable()
    stage = {}
    per_step = []
    launches0 = N.load().tg_launch_count()
    _barrier(world)
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (not inside a step's events)
        a, b = ev(), ev()
        a.record()
        d, flat, S, order = step(stage)
        b.record()
        torch.cuda.synchronize()
        per_step.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    _barrier(world)
    wall = time.perf_counter() - wall0
    launches = int(N.load().tg_launch_count() - launches0)
    clocks = sampler.stop() if sampler else None
    ms = float(np.mean(per_step))
    ms_max = _max_over_ranks(ms, world, device)

    # ---- row-sort roofline: kernel timed alone on the stream it runs on
    sort_ms = []
    for _ in range(5):
        flush.zero_()
        a, b = ev(), ev()
        a.record()
        simmatrix.sort_rows_device(S, with_screen=True, out=order_buf)
        b.record()
        torch.cuda.synchronize()
        sort_ms.append(a.elapsed_time(b))
    sort_avg = float(np.mean(sort_ms))
    sort_bytes = 8 * n * n + 4 * n * (n - 1)
    hbm_peak, peak_kind = _peaks()
    achieved = sort_bytes / (sort_avg * 1e-3) / 1e9
    traffic = None
    traffic_src = None
    tp = REPO / "profiles" / "sort_traffic.json"   # ncu --set full capture of the CURRENT sort kernel
    if tp.exists():
        try:
            tj = json.loads(tp.read_text())
            if int(tj.get("n", n)) == n:
                traffic = tj.get("dram_bytes_per_launch")
                traffic_src = tj.get("kernel")
        except Exception:
            traffic = None
    # fp64 similarity (secondary kernel)
    sim_ms = float(np.mean(stage["similarity"]))
    sim_flops = n * (n + 1) * L

    # ---- e2e through the public API with host buffers
    e2e_ms = []
    h2d = x_host.nbytes
    d2h = 0
    x_pinned = torch.from_numpy(np.ascontiguousarray(x_host)).pin_memory()   # the input in pinned host memory
    run_series(x_pinned, k=k, apsp_mode=mode)   # warm-up of the host-buffer path (first-call allocations)
    gc.collect()   # (collection stays paused: see the timed region)
    for _ in range(max(1, min(args.steps, 5))):
        gc.collect()   # outside the timed region (collection is paused): a cycle left by the previous call would
        # keep its 1.2 GB of S / order away from the allocator's cache and put a cudaMalloc inside this one
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep, dend, lab_out = run_series(x_pinned, k=k, apsp_mode=mode)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        d2h = dend.lefts.nbytes + dend.rights.nbytes + dend.heights.nbytes + dend.sizes.nbytes + lab_out.nbytes
    e2e = float(np.mean(e2e_ms))
    e2e = _max_over_ranks(e2e, world, device)

    # ---- the top of the north star's n range: config 5 (n = 50,000, 20 GB S in HBM),
    # device-resident pass after one warm-up pass (reported beside, not the value)
    big = None
    if rank == 0 and world == 1 and not args.no_50k and cfg == 3 and args.n is None:   # side measurement, N = 1 only
        del S, order, S_buf, order_buf
        gc.collect()
        torch.cuda.empty_cache()
        x5, _ = synth.generate(5)
        X5 = torch.from_numpy(x5).to(device)
        # S (20 GB) is an output buffer allocated once, as in the timed loop above, and the caching
        # allocator keeps the other buffers (order: 10 GB) between passes: a pass that has to
        # cudaMalloc tens of GB right after they were freed waits for the driver inside whichever
        # stage allocates next (passes of 670 and 1009 ms in one run, apsp stage 12 vs 271 ms)
        S5_buf = torch.empty((x5.shape[0], x5.shape[0]), dtype=torch.float64, device=device)
        st5 = {}
        passes = []
        for rep_i in range(4):   # pass 1 warms up
            gc.collect()   # between passes, outside the timed region (collection is paused): cycles
            # would keep the previous pass's buffers away from the allocator's cache
            flush.zero_()
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record()
            S5 = simmatrix.pearson_similarity_device(X5, out=S5_buf)
            a2 = ev()
            a2.record()
            rep5, _, _, _ = P.run_stages(P.PipelineConfig(apsp_mode="hub", k=synth.num_clusters(5)), S5, None,
                                         sync_stages=True)
            b.record()
            torch.cuda.synchronize()
            st5 = {kk: round(v * 1e3, 2) for kk, v in rep5.stage_seconds.items()}
            st5["similarity"] = round(a.elapsed_time(a2), 2)
            ms5 = round(a.elapsed_time(b), 1)
            if rep_i > 0:
                passes.append((ms5, st5))
            del S5, rep5
        stage_names = passes[0][1].keys()
        big = {"workload": "BASELINE config 5: n=50000, L=256, hub APSP, heap TMFG",
               "ms": round(float(np.mean([p[0] for p in passes])), 1),
               "ms_passes": [p[0] for p in passes],
               "stage_ms": {kk: round(float(np.mean([p[1][kk] for p in passes])), 2) for kk in stage_names},
               "stage_ms_passes": [p[1] for p in passes],
               "passes": "mean of passes 2-4 (pass 1 = warm-up)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(cfg, args.n)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms_max, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 3), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, n, L, mode, k),
            "stage_ms": {kk: round(float(np.mean(vv)), 3) for kk, vv in stage.items()},
            "roofline": {"bound": "hbm", "kernel": "row_sort_v2_kernel (per-row neighbour sort)",
                         "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "traffic": traffic, "traffic_kernel": traffic_src,
                         "algorithmic_bytes": sort_bytes, "kernel_ms": round(sort_avg, 4),
                         "gkeys_per_s": round(n * (n - 1) / (sort_avg * 1e-3) / 1e9, 2),
                         "peak_kind": peak_kind},
            "similarity": {"ms": round(sim_ms, 3), "tflops_alg": round(sim_flops / (sim_ms * 1e-3) / 1e12, 2),
                           "flops_alg": sim_flops},
            "e2e": {"value": round(e2e, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_runs": [round(x, 3) for x in e2e_ms]},
            "gpu_launches": launches // max(args.steps, 1),
            "gc": "collected before, paused through the timed measurements",
            "gpu_launches_timed_total": launches,
            "wall_s_timed": round(wall, 3), "step_ms": [round(x, 3) for x in per_step],
            "stage_ms_steps": {kk: [round(float(x), 2) for x in vv] for kk, vv in stage.items()},
            "clocks": clocks,
            "cpu_baseline": cpu,
            "n50k": big,
        }
        print(json.dumps(line))
    gc.enable()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def cpu_baseline_sample(cfg, n_override=None) -> dict:
    """The CPU oracle on this host's cores: one full pipeline step of the same workload."""
    from oracle import oracle as orc
    from paper_2408_09399_b200 import synth

    x, labels = synth.generate(cfg, n=n_override)
    k = synth.num_clusters(cfg)
    mode = "hub" if cfg in (3, 5) else "exact"
    orc.set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    S = orc.pearson_similarity(x)
    orc.run_stages(S, k, mode)
    dt = (time.perf_counter() - t0) * 1e3
    return {"value": round(dt, 1), "unit": UNIT, "cores": orc.num_threads(), "kind": "port",
            "sample": f"one full step (Pearson + sort + heap TMFG + {mode} APSP + DBHT + cut) of config {cfg}, "
                      f"n={x.shape[0]}, C/OpenMP + numpy oracle", "host": host_info()}


# ------------------------------------------------------------------ reference arm
def host_info() -> dict:
    """CPU model, logical cores and RAM of the host the CPU baselines run on."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal:"):
                    ram = round(int(line.split()[1]) / 1024 ** 2, 1)
                    break
    except Exception:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "ram_gib": ram}


def workload_config(cfg: int, n: int, L: int, mode: str, k: int) -> dict:
    """The config dict both arms print (identical keys and values for the same workload)."""
    return {"workload": f"BASELINE config {cfg}: n={n} series, L={L}, {mode} APSP, heap TMFG",
            "n": n, "L": L, "apsp": mode, "k": k, "parallelism": "replicas",
            "l2": "flushed (256 MB write) between timed GPU steps; S (8n^2 B) exceeds L2"}


def _python_reference_once(cfg: int, n_override=None) -> dict | None:
    """The unmodified reference package (baseline/_ref, Python + numba) on this host, one step.

    Runs in a child process (numba threads = all cores) so its JIT and thread pool never
    share the bench process.  Warm-up: one call of every kernel at n = 64 (JIT excluded).
    """
    ref = REPO / "baseline" / "_ref"
    if not (ref / "tmfgclust").is_dir():
        return None
    code = f"""
import json, sys, time
sys.path.insert(0, {str(ref)!r}); sys.path.insert(0, {str(REPO)!r})
import numpy as np, tmfgclust as tc
from tmfgclust.pipeline import PipelineConfig, run_stages
from paper_2408_09399_b200 import synth
xs, ls = synth.generate(1, n=64)
ds = tc.Dataset(labels=ls, series=xs)
Ss = tc.pearson_similarity(ds)
run_stages(PipelineConfig(apsp_mode='exact', k=3), Ss, ls)
run_stages(PipelineConfig(apsp_mode='hub', k=3), Ss, ls)
x, labels = synth.generate({cfg}, n={n_override!r})
t0 = time.perf_counter()
S = tc.pearson_similarity(tc.Dataset(labels=labels, series=x))
sim = time.perf_counter() - t0
mode = 'hub' if {cfg} in (3, 5) else 'exact'
rep, *_ = run_stages(PipelineConfig(apsp_mode=mode, k=synth.num_clusters({cfg})), S, labels)
print(json.dumps({{"similarity_s": sim, "stage_seconds": rep.stage_seconds, "digest": rep.digest,
                  "total_s": sim + sum(rep.stage_seconds.values())}}))
"""
    env = dict(os.environ)
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/tg_numba_cache")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)
        rows = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if not rows:
            return {"error": (r.stderr or r.stdout)[-300:]}
        d = json.loads(rows[-1])
        return {"ms": round(d["total_s"] * 1e3, 1),
                "stage_ms": {k: round(v * 1e3, 1) for k, v in d["stage_seconds"].items()},
                "similarity_ms": round(d["similarity_s"] * 1e3, 1), "digest": d["digest"],
                "kind": "reference (unmodified tmfgclust, Python + numba, all cores)", "steps": 1}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)[:300]}


def run_reference(args, world, rank):
    """The reference's CPU path on all host threads.

    ``value``: the oracle port (C/OpenMP + numpy restatement of the reference, outputs
    bit-identical to it), K full steps after W full-size warm-up steps.  Beside it, once:
    the unmodified Python reference (baseline/_ref, numba) on the same workload.
    """
    if world > 1 and rank != 0:
        return
    from oracle import oracle as orc
    from paper_2408_09399_b200 import synth

    cfg = args.config
    x, labels = synth.generate(cfg, n=args.n)
    n, L = x.shape
    k = synth.num_clusters(cfg)
    mode = "hub" if cfg in (3, 5) else args.apsp
    orc.set_threads(os.cpu_count() or 1)
    for _ in range(max(args.warmup, 0)):   # full-size warm-up: S and the sort buffers first-touched
        orc.run_stages(orc.pearson_similarity(x), k, mode)
    times, stages = [], {}
    gc.collect()   # the same interpreter GC treatment as the GPU arm's timed region
    gc.disable()
    for _ in range(max(args.steps, 1)):
        t0 = time.perf_counter()
        S = orc.pearson_similarity(x)
        t1 = time.perf_counter()
        r = orc.run_stages(S, k, mode)
        times.append((time.perf_counter() - t0) * 1e3)
        stages.setdefault("similarity", []).append((t1 - t0) * 1e3)
        for kk, vv in r["seconds"].items():
            stages.setdefault(kk, []).append(vv * 1e3)
        del S
    gc.enable()
    v = float(np.mean(times))
    py_ref = None if args.no_python_reference else _python_reference_once(cfg, args.n)
    line = {
        "metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(v, 1), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": workload_config(cfg, int(n), int(L), mode, k),
        "stage_ms": {kk: round(float(np.mean(vv)), 1) for kk, vv in stages.items()},
        "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": orc.num_threads(), "kind": "port",
                         "sample": f"{len(times)} full steps of config {cfg} (Pearson + sort + heap TMFG + {mode} "
                                   "APSP + DBHT + cut; C/OpenMP + numpy restatement of the reference, outputs "
                                   "bit-identical to it) after full-size warm-up",
                         "host": host_info()},
        "python_reference": py_ref,
        "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--apsp", default="hub", choices=["exact", "hub"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-50k", action="store_true", help="skip the config-5 (n=50k) side measurement")
    ap.add_argument("--no-python-reference", action="store_true",
                    help="reference arm: skip the one-step timing of the unmodified Python reference")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_b200(args, world, rank, local)


if __name__ == "__main__":
    main()
