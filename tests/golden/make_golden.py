"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nbcache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--configs 1,2,4,3]

It imports ``tmfgclust`` from /root/reference/pkg/src (read-only), runs every
hot-path stage on a set of inputs and writes

* ``small_cases.npz``  -- full input S and every stage output for small n;
* ``digests.json``     -- sha256 of every stage output (all cases, including the
                          full-size BASELINE configs 1, 2, 4 and 3), the dendrogram
                          digests, stats and labels hashes.

The inputs are either the reference-style fixture matrices (uniform / quantized /
rounded, regenerated bit-identically from their seeds by ``synth``) or Pearson
matrices of seeded synthetic series (``synth.generate``), whose S is produced by
the reference's own ``pearson_similarity``.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import tmfgclust as tc  # noqa: E402  (the reference)
from tmfgclust import apsp as ref_apsp  # noqa: E402
from tmfgclust.dbht import bubble_sinks  # noqa: E402
from tmfgclust.datasets import generate_class_dataset  # noqa: E402
from tmfgclust.linkage import serialize_dendrogram  # noqa: E402
from tmfgclust.pipeline import PipelineConfig, run_stages  # noqa: E402

from paper_2408_09399_b200 import synth  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_inputs():
    """name -> (S, series-or-None, k)."""
    cases = {}
    cases["n4_u"] = (synth.uniform_matrix(4, 0), None, 2)
    S = np.full((5, 5), 0.5)
    np.fill_diagonal(S, 1.0)
    cases["n5_flat"] = (S, None, 2)
    cases["n6_u"] = (synth.uniform_matrix(6, 1), None, 3)
    S = np.round(synth.uniform_matrix(20, 2), 1)
    np.fill_diagonal(S, 1.0)
    cases["n20_round"] = (S, None, 3)
    cases["n30_u"] = (synth.uniform_matrix(30, 4), None, 3)
    cases["n40_q"] = (synth.quantized_matrix(40, 3), None, 4)
    cases["n60_u"] = (synth.uniform_matrix(60, 4), None, 3)
    cases["n120_q"] = (synth.quantized_matrix(120, 5), None, 4)
    d = generate_class_dataset(50, 128, 5, seed=2)
    cases["n50_s"] = (tc.pearson_similarity(d, workers=1), None, 5)
    d = generate_class_dataset(200, 96, 6, seed=7)
    cases["n200_s"] = (tc.pearson_similarity(d, workers=1), None, 6)
    x, lab = synth.generate(1, n=300)
    cases["c1_n300"] = (None, x, 5)
    x, lab = synth.generate(4, n=400)
    cases["c4_n400"] = (None, x, 8)
    return cases


def run_case(name, S, x, k, store_full):
    rec = {}
    arrays = {}
    if x is not None:
        data = tc.Dataset(labels=np.zeros(x.shape[0], dtype=np.int64), series=x)
        t0 = time.perf_counter()
        S = tc.pearson_similarity(data, workers=8)
        rec["pearson_s"] = time.perf_counter() - t0
        arrays["X"] = x
    n = S.shape[0]
    rec["n"] = n
    rec["k"] = k
    rec["S"] = sha(S)
    arrays["S"] = S
    lists = tc.sort_neighbor_lists(S, workers=8)
    rec["order"] = sha(lists.order)
    arrays["order"] = lists.order
    rec["clique"] = list(tc.select_initial_clique(S))
    g = tc.build_tmfg_heap(S, lists)
    for key in ("edges", "weights", "trace", "faces", "initial_clique"):
        rec[f"tmfg_{key}"] = sha(getattr(g, key))
        arrays[f"tmfg_{key}"] = getattr(g, key)
    if n <= 200:
        try:
            gc = tc.build_tmfg_heap(S, lists, check_invariants=True)
            rec["tmfg_stats"] = dict(gc.debug_stats)
        except AssertionError as exc:  # the reference's own invariant check can fire on ties
            rec["tmfg_check_error"] = str(exc)
    w = tc.to_weighted(g, S)
    for key in ("indptr", "neighbors", "lengths", "strength"):
        rec[f"w_{key}"] = sha(getattr(w, key))
        arrays[f"w_{key}"] = getattr(w, key)
    tree = tc.build_bubble_tree(g)
    dtree = tc.orient_edges(tree, S)
    for key in ("bubbles", "links", "link_faces"):
        rec[f"tree_{key}"] = sha(getattr(tree, key))
        arrays[f"tree_{key}"] = getattr(tree, key)
    rec["dtree_sources"] = sha(dtree.sources)
    rec["dtree_targets"] = sha(dtree.targets)
    arrays["dtree_sources"] = dtree.sources
    arrays["dtree_targets"] = dtree.targets
    sinks = bubble_sinks(dtree, g)
    rec["sinks"] = sha(sinks)
    arrays["sinks"] = sinks
    modes = ["exact", "hub"] if n <= 4000 else ["hub"]
    for mode in modes:
        t0 = time.perf_counter()
        if mode == "exact":
            o = tc.apsp_exact(w, workers=8)
            rec["exact_D"] = sha(o.matrix)
            if store_full:
                arrays["exact_D"] = o.matrix
        else:
            o = tc.apsp_hub(w, workers=8)
            for key in ("hubs", "hub_dist", "nearest_hub", "nearest_dist", "radii",
                        "near_indptr", "near_ids", "near_dist"):
                rec[f"hub_{key}"] = sha(getattr(o, key))
                arrays[f"hub_{key}"] = getattr(o, key)
        rec[f"{mode}_apsp_s"] = time.perf_counter() - t0
        asg = tc.assign_vertices(g, dtree, o)
        rec[f"{mode}_vertex_bubble"] = sha(asg.vertex_bubble)
        rec[f"{mode}_vertex_converging"] = sha(asg.vertex_converging)
        arrays[f"{mode}_vertex_bubble"] = asg.vertex_bubble
        arrays[f"{mode}_vertex_converging"] = asg.vertex_converging
        t0 = time.perf_counter()
        d = tc.build_hierarchy(asg, dtree, o, workers=8)
        rec[f"{mode}_hierarchy_s"] = time.perf_counter() - t0
        text = serialize_dendrogram(d)
        rec[f"{mode}_digest"] = hashlib.sha256(text.encode()).hexdigest()
        for key in ("lefts", "rights", "heights", "sizes"):
            arrays[f"{mode}_dend_{key}"] = getattr(d, key)
        labels = tc.cut(d, k)
        rec[f"{mode}_labels"] = sha(labels)
        arrays[f"{mode}_labels"] = labels
        rec[f"{mode}_num_converging"] = int(np.unique(asg.vertex_converging).size)
        # the reference's own pipeline driver must agree with the stage-by-stage run
        cfg = PipelineConfig(variant="heap", apsp_mode=mode, k=k, workers=8)
        report, _, _, _ = run_stages(cfg, S, None)
        assert report.digest == rec[f"{mode}_digest"], (name, mode)
        rec[f"{mode}_stage_seconds"] = report.stage_seconds
    return rec, arrays


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,3")
    ap.add_argument("--skip-small", action="store_true")
    args = ap.parse_args()
    out_json = HERE / "digests.json"
    digests = json.loads(out_json.read_text()) if out_json.exists() else {}
    digests["_meta"] = {"numpy": np.__version__, "reference": "tmfgclust 0.1.0 (/root/reference/pkg)",
                        "seed": synth.DEFAULT_SEED}
    if not args.skip_small:
        store = {}
        for name, (S, x, k) in small_inputs().items():
            rec, arrays = run_case(name, S, x, k, store_full=True)
            digests[name] = rec
            for key, a in arrays.items():
                store[f"{name}/{key}"] = a
            print(name, "done", flush=True)
        np.savez_compressed(HERE / "small_cases.npz", **store)
    for c in [int(c) for c in args.configs.split(",") if c]:
        x, labels = synth.generate(c)
        t0 = time.perf_counter()
        rec, _ = run_case(f"config{c}", None, x, synth.num_clusters(c), store_full=False)
        rec["labels_true"] = sha(labels)
        rec["total_s"] = time.perf_counter() - t0
        digests[f"config{c}"] = rec
        print(f"config{c}", "done", rec["total_s"], flush=True)
        out_json.write_text(json.dumps(digests, indent=1, sort_keys=True) + "\n")
    out_json.write_text(json.dumps(digests, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
