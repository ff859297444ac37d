"""Pin the CPU oracle to the reference: every stage, every golden case, bit-exact.

The fixtures in tests/golden/ were produced by running the reference package
itself (tests/golden/make_golden.py); these tests need neither the reference nor
a GPU.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN  # noqa: F401

SMALL = ["n4_u", "n5_flat", "n6_u", "n20_round", "n30_u", "n40_q", "n60_u", "n120_q",
         "n50_s", "n200_s", "c1_n300", "c4_n400"]


def _run(orc, S, k):
    out = {}
    out["order"] = orc.sort_neighbor_lists(S)
    out["clique"] = list(orc.select_initial_clique(S))
    g = orc.build_tmfg_heap(S, out["order"])
    out["graph"] = g
    w = orc.to_weighted(g, S)
    out["w"] = w
    tree = orc.build_bubble_tree(g)
    dtree = orc.orient_edges(tree, S)
    out["tree"], out["dtree"] = tree, dtree
    out["sinks"] = orc.bubble_sinks(dtree, g)
    for mode in ("exact", "hub"):
        o = orc.apsp_exact(w) if mode == "exact" else orc.apsp_hub(w)
        asg = orc.assign_vertices(g, dtree, o)
        d = orc.build_hierarchy(asg, dtree, o)
        out[mode] = dict(oracle=o, asg=asg, dend=d, digest=orc.dendrogram_digest(d),
                         labels=orc.cut(d, k))
    return out


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference_small(name, small_cases, digests, oracle):
    c = small_cases[name]
    rec = digests[name]
    if "X" in c:
        S = oracle.pearson_similarity(c["X"])
        assert np.array_equal(S, c["S"]), "oracle Pearson must be bit-identical to numba's"
    S = c["S"]
    out = _run(oracle, S, rec["k"])
    assert np.array_equal(out["order"], c["order"])
    assert out["clique"] == rec["clique"]
    g = out["graph"]
    for key in ("edges", "weights", "trace", "faces", "initial_clique"):
        assert np.array_equal(g[key], c[f"tmfg_{key}"]), key
    if "tmfg_stats" in rec:
        assert g["stats"] == rec["tmfg_stats"]
    for key in ("indptr", "neighbors", "lengths", "strength"):
        assert np.array_equal(out["w"][key], c[f"w_{key}"]), key
    for key in ("bubbles", "links", "link_faces"):
        assert np.array_equal(out["tree"][key], c[f"tree_{key}"]), key
    assert np.array_equal(out["dtree"]["sources"], c["dtree_sources"])
    assert np.array_equal(out["dtree"]["targets"], c["dtree_targets"])
    assert np.array_equal(out["sinks"], c["sinks"])
    assert np.array_equal(out["exact"]["oracle"]["matrix"], c["exact_D"])
    o = out["hub"]["oracle"]
    for key in ("hubs", "hub_dist", "nearest_hub", "nearest_dist", "radii", "near_indptr",
                "near_ids", "near_dist"):
        assert np.array_equal(o[key], c[f"hub_{key}"]), key
    for mode in ("exact", "hub"):
        r = out[mode]
        assert np.array_equal(r["asg"]["vertex_bubble"], c[f"{mode}_vertex_bubble"])
        assert np.array_equal(r["asg"]["vertex_converging"], c[f"{mode}_vertex_converging"])
        for key in ("lefts", "rights", "heights", "sizes"):
            assert np.array_equal(r["dend"][key], c[f"{mode}_dend_{key}"]), (mode, key)
        assert r["digest"] == rec[f"{mode}_digest"], mode
        assert np.array_equal(r["labels"], c[f"{mode}_labels"])


@pytest.mark.parametrize("config", [1, 2, 4])
def test_oracle_matches_reference_configs(config, digests, oracle):
    """Full-size BASELINE configs: every stage hash equals the reference's."""
    from paper_2408_09399_b200 import synth
    rec = digests[f"config{config}"]
    x, labels = synth.generate(config)
    assert oracle.sha(labels) == rec["labels_true"]
    S = oracle.pearson_similarity(x)
    assert oracle.sha(S) == rec["S"]
    order = oracle.sort_neighbor_lists(S)
    assert oracle.sha(order) == rec["order"]
    g = oracle.build_tmfg_heap(S, order)
    for key in ("edges", "weights", "trace", "faces"):
        assert oracle.sha(g[key]) == rec[f"tmfg_{key}"], key
    w = oracle.to_weighted(g, S)
    tree = oracle.build_bubble_tree(g)
    dtree = oracle.orient_edges(tree, S)
    assert oracle.sha(dtree["sources"]) == rec["dtree_sources"]
    for mode in ("exact", "hub"):
        o = oracle.apsp_exact(w) if mode == "exact" else oracle.apsp_hub(w)
        if mode == "exact":
            assert oracle.sha(o["matrix"]) == rec["exact_D"]
        else:
            for key in ("hubs", "hub_dist", "near_indptr", "near_ids", "near_dist"):
                assert oracle.sha(o[key]) == rec[f"hub_{key}"], key
        asg = oracle.assign_vertices(g, dtree, o)
        assert oracle.sha(asg["vertex_bubble"]) == rec[f"{mode}_vertex_bubble"]
        d = oracle.build_hierarchy(asg, dtree, o)
        assert oracle.dendrogram_digest(d) == rec[f"{mode}_digest"], mode
        assert oracle.sha(oracle.cut(d, rec["k"])) == rec[f"{mode}_labels"]
