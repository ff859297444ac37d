"""Golden records for the exact and corr TMFG builders, made by running the REFERENCE itself.

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nbcache PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_variants.py

For every small case of small_cases.npz (its S) and for BASELINE configs 1 and 2 (S from the
reference's own pearson_similarity), runs tmfgclust.tmfg.build_tmfg_exact (tmfg.py:208-263)
and build_tmfg_corr (tmfg.py:280-341) with prefix_size 1 and larger prefixes
(tmfg.py:185-205), and records sha256 of trace / edges / faces / initial_clique / weights.
For config 1 it also records the dendrogram digest and labels of run_stages with each
variant (pipeline.py:173-239) and the edge_sum_delta rows of compare_variants' arithmetic.
Writes tests/golden/variants.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import tmfgclust as tc  # noqa: E402  (the reference)
from tmfgclust.pipeline import PipelineConfig, run_stages  # noqa: E402

from paper_2408_09399_b200 import synth  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_rec(g) -> dict:
    return {k: sha(getattr(g, k)) for k in ("trace", "edges", "faces", "initial_clique", "weights")}


def main():
    raw = np.load(HERE / "small_cases.npz")
    cases = {}
    for key in raw.files:
        name, field = key.split("/", 1)
        if field == "S":
            cases[name] = raw[key]
    out = {"_meta": {"reference": "tmfgclust (pkg/src) at /root/reference, unmodified",
                     "prefixes": [1, 3, 17]}}
    for cfg in (1, 2):
        x, labels = synth.generate(cfg)
        cases[f"config{cfg}"] = tc.pearson_similarity(tc.Dataset(labels=labels, series=x))
    for name, S in sorted(cases.items()):
        rec = {"S": sha(S), "n": int(S.shape[0])}
        lists = tc.sort_neighbor_lists(S)
        for p in (1, 3, 17):
            for variant in ("exact", "corr"):
                cfg = tc.BuildConfig(variant=variant, prefix_size=p)
                g = tc.build_tmfg_exact(S, cfg) if variant == "exact" else tc.build_tmfg_corr(S, lists, cfg)
                rec[f"{variant}_p{p}"] = graph_rec(g)
        out[name] = rec
        print(name, flush=True)
    # whole pipeline with each variant on config 1 (exact APSP)
    x, labels = synth.generate(1)
    S = tc.pearson_similarity(tc.Dataset(labels=labels, series=x))
    base = tc.build_tmfg_exact(S, tc.BuildConfig(variant="exact"))
    pipe = {}
    for variant, p in (("exact", 1), ("exact", 3), ("corr", 1), ("heap", 1)):
        rep, g, d, flat = run_stages(PipelineConfig(variant=variant, prefix_size=p, k=5), S, labels)
        pipe[f"{variant}_p{p}"] = {"digest": rep.digest, "labels": sha(np.asarray(flat)),
                                   "edge_sum": rep.edge_sum, "ari": rep.ari,
                                   "edge_sum_delta": float(tc.edge_sum_delta(g, base, S))}
    out["config1_pipeline"] = pipe
    (HERE / "variants.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
