"""Time the TMFG kernel at config-3 size and print its internal phase profile."""
import os, sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
_prof = Path(__file__).resolve().parent.parent / "paper_2408_09399_b200" / "_lib" / "libtmfg_b200_prof.so"
if _prof.exists():   # built by `make -C paper_2408_09399_b200/csrc PROFILE=1`
    os.environ.setdefault("TG_LIB", str(_prof))
import torch
from paper_2408_09399_b200 import simmatrix, synth, tmfg, _native as N
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N.load()
x, _ = synth.generate(cfg, n=n)
S = simmatrix.pearson_similarity_device(torch.from_numpy(x).cuda())
order, rowsum = simmatrix.sort_rows_device(S)
clique = tmfg.initial_clique_device(S, rowsum)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = tmfg.build_tmfg_heap_device(S, order, clique)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
st = out["stats"].cpu().numpy()
names = ["pops", "refreshes", "gain_inc", "status", "a4", "a5", "a6", "tails", "rounds", "refills", "cyc_warp_max", "cyc_ne_max", "cyc_rf_max", "cyc_S_max", "cyc_refill", "pool", "cyc_par", "cyc_replay", "cyc_merge", "cyc_insert", "spec_refreshes", "fg_lookups", "fg_scans", "fg_tail_batches", "rf_select", "rf_take", "rf_place", "rf_fill", "rc_hit", "bg_scans", "helper_passes", "helper_wp"]
d = {k: int(v) for k, v in zip(names, st)}
d["ms"] = dt * 1e3
d["us_per_insert"] = dt * 1e6 / (n - 4)
for kk in ("cyc_warp_max", "cyc_ne_max", "cyc_rf_max", "cyc_S_max", "cyc_refill", "cyc_par", "cyc_replay", "cyc_merge", "cyc_insert", "spec_refreshes"):
    d[kk + "_per_round"] = round(d[kk] / max(d["rounds"], 1))
d["cyc_per_round_total"] = round(dt * 1.965e9 / max(d["rounds"], 1))
for q, nm in enumerate(["rp_scan_winner", "rp_split", "rp_sort", "merge_warp_max"]):
    d[nm] = round(int(st[4 + q]) / max(d["rounds"], 1))
print(json.dumps(d))
if "helper_wp" in d:
    d["helper_wp_vertices"] = d["helper_wp"] >> 32; d["helper_wp_batches"] = d["helper_wp"] & 0xffffffff
keys = ["rp_scan_winner", "rp_split", "rp_sort", "merge_warp_max", "cyc_insert_per_round", "helper_wp_vertices", "helper_wp_batches", "ms", "rounds", "rc_hit", "spec_refreshes", "fg_scans", "fg_tail_batches", "bg_scans", "cyc_per_round_total",
        "cyc_par_per_round", "cyc_ne_max_per_round", "cyc_rf_max_per_round", "cyc_S_max_per_round",
        "cyc_replay_per_round", "cyc_merge_per_round", "cyc_refill_per_round", "helper_passes"]
print("SHORT", os.environ.get("TG_LIB", "").split("/")[-1], os.environ.get("TG_TMFG_CLUSTER", "8"),
      {k.replace("_per_round", ""): (round(d[k], 1) if isinstance(d[k], float) else d[k]) for k in keys})
