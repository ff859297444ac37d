"""GPU parity for APSP + DBHT + the whole pipeline vs the reference goldens.

Every array is compared bit-exactly (distances included: the label-correcting
searches reach the same fp64 fixed point as binary-heap Dijkstra), and the
dendrogram parity fingerprint is the sha256 of serialize_dendrogram
(pipeline.py:226-227).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SMALL = ["n4_u", "n5_flat", "n6_u", "n20_round", "n30_u", "n40_q", "n60_u", "n120_q", "n50_s", "n200_s",
         "c1_n300", "c4_n400"]


@pytest.fixture(scope="module")
def pkg():
    import paper_2408_09399_b200 as p
    p._native.load()
    return p


@pytest.mark.parametrize("name", SMALL)
def test_stages_match_golden(name, small_cases, digests, pkg):
    c = small_cases[name]
    rec = digests[name]
    S = c["S"]
    lists = pkg.sort_neighbor_lists(S)
    g = pkg.build_tmfg_heap(S, lists)
    w = pkg.to_weighted(g, S)
    for key in ("indptr", "neighbors", "lengths", "strength"):
        assert np.array_equal(getattr(w, key), c[f"w_{key}"]), key
    tree = pkg.build_bubble_tree(g)
    for key in ("bubbles", "links", "link_faces"):
        assert np.array_equal(getattr(tree, key), c[f"tree_{key}"]), key
    dtree = pkg.orient_edges(tree, S)
    assert np.array_equal(dtree.sources, c["dtree_sources"])
    assert np.array_equal(dtree.targets, c["dtree_targets"])
    assert np.array_equal(pkg.bubble_sinks(dtree, g), c["sinks"])
    for mode in ("exact", "hub"):
        o = pkg.apsp_exact(w) if mode == "exact" else pkg.apsp_hub(w)
        if mode == "exact":
            assert np.array_equal(o.matrix, c["exact_D"])
        else:
            for key in ("hubs", "hub_dist", "nearest_hub", "nearest_dist", "radii", "near_indptr", "near_ids",
                        "near_dist"):
                assert np.array_equal(getattr(o, key), c[f"hub_{key}"]), key
        asg = pkg.assign_vertices(g, dtree, o)
        assert np.array_equal(asg.vertex_bubble, c[f"{mode}_vertex_bubble"]), mode
        assert np.array_equal(asg.vertex_converging, c[f"{mode}_vertex_converging"]), mode
        d = pkg.build_hierarchy(asg, dtree, o)
        for key in ("lefts", "rights", "heights", "sizes"):
            assert np.array_equal(getattr(d, key), c[f"{mode}_dend_{key}"]), (mode, key)
        import hashlib
        assert hashlib.sha256(pkg.serialize_dendrogram(d).encode()).hexdigest() == rec[f"{mode}_digest"]
        assert np.array_equal(pkg.cut(d, rec["k"]), c[f"{mode}_labels"])


@pytest.mark.parametrize("config,mode", [(1, "exact"), (1, "hub"), (2, "exact"), (2, "hub"), (4, "exact"),
                                         (4, "hub"), (3, "hub")])
def test_pipeline_digest_configs(config, mode, digests, oracle, pkg):
    """Full BASELINE configs on the reference's own S: same dendrogram digest and labels."""
    from paper_2408_09399_b200 import synth
    rec = digests[f"config{config}"]
    x, labels = synth.generate(config)
    S = oracle.pearson_similarity(x)
    assert oracle.sha(S) == rec["S"]
    report, graph, dend, flat = pkg.run_stages(pkg.PipelineConfig(apsp_mode=mode, k=rec["k"]), S, labels)
    assert report.digest == rec[f"{mode}_digest"]
    assert oracle.sha(flat) == rec[f"{mode}_labels"]
    assert report.num_converging == rec[f"{mode}_num_converging"]


@pytest.mark.parametrize("n", [13000, 26000])
def test_pipeline_mid_size_vs_oracle(n, oracle, pkg):
    """Sizes between the BASELINE configs (n = 13,000: one row buffer in the sort, the TMFG scan
    state still in shared memory; n = 26,000: the partitioned long-row sort, the scan state in
    global memory, the cluster NN-chain): the whole device pipeline on the reference-order S
    against the oracle run in the test."""
    from paper_2408_09399_b200 import simmatrix, synth
    x, labels = synth.generate(3, n=n)
    Sd = simmatrix.pearson_similarity_refexact_device(x)
    S = Sd.cpu().numpy()
    ref = oracle.run_stages(S, 20, "hub")
    report, graph, dend, flat = pkg.run_stages(pkg.PipelineConfig(apsp_mode="hub", k=20), Sd, labels)
    assert report.digest == ref["digest"]
    assert np.array_equal(flat, ref["labels"])
    assert report.num_converging == ref["num_converging"]


def test_hub_query_and_block_semantics(small_cases, pkg):
    c = small_cases["n200_s"]
    S = c["S"]
    g = pkg.build_tmfg_heap(S, pkg.sort_neighbor_lists(S))
    o = pkg.apsp_hub(pkg.to_weighted(g, S))
    rows = np.array([0, 3, 7, 29, 150])
    cols = np.array([1, 3, 15, 199])
    blk = o.block(rows, cols)
    hd = o.hub_dist
    for i, u in enumerate(rows):
        for j, v in enumerate(cols):
            e = float(np.min(hd[:, u] + hd[:, v]))
            a = o._near_lookup(int(u), int(v))
            b = o._near_lookup(int(v), int(u))
            want_block = b if b is not None else (a if a is not None else e)
            assert blk[i, j] == want_block
            lo, hi = min(u, v), max(u, v)
            q1, q2 = o._near_lookup(int(lo), int(hi)), o._near_lookup(int(hi), int(lo))
            want_q = 0.0 if u == v else (q1 if q1 is not None else (q2 if q2 is not None else e))
            assert o.query(int(u), int(v)) == want_q


def test_corrupt_trace_raises(small_cases, pkg):
    S = small_cases["n30_u"]["S"]
    g = pkg.build_tmfg_heap(S, pkg.sort_neighbor_lists(S))
    bad = g.trace.copy()
    v, x, y, _ = bad[2]
    bad[2, 1:] = sorted((int(v), int(x), int(y)))
    g2 = pkg.TmfgGraph(n=g.n, edges=g.edges, weights=g.weights, initial_clique=g.initial_clique, trace=bad,
                       faces=g.faces)
    with pytest.raises(pkg.TraceError):
        pkg.build_bubble_tree(g2)


def test_pipeline_config5_50k(pkg):
    """BASELINE config 5 (n = 50,000, 20 GB S resident in HBM): the reference's own S
    (reference-order Pearson on the GPU), then the whole pipeline; golden record
    from the pinned C oracle (tests/golden/make_config5.py)."""
    import json
    from pathlib import Path

    from oracle import oracle as orc
    from paper_2408_09399_b200 import simmatrix, synth
    path = Path(__file__).parent / "golden" / "config5.json"
    if not path.exists():
        pytest.skip("tests/golden/config5.json not generated")
    rec = json.loads(path.read_text())
    x, labels = synth.generate(5)
    Sd = simmatrix.pearson_similarity_refexact_device(x)
    assert orc.sha(Sd[:64].cpu().numpy()) == rec["S_rows"]
    n = rec["n"]
    band = Sd.reshape(-1)[pkg._device.torch().arange(n, device=Sd.device) * n
                          + (pkg._device.torch().arange(n, device=Sd.device) * 7919) % n]
    assert orc.sha(band.cpu().numpy()) == rec["S_diag_band"]
    report, graph, dend, flat = pkg.run_stages(pkg.PipelineConfig(apsp_mode="hub", k=rec["k"]), Sd, labels)
    assert orc.sha(np.asarray(graph.edges, dtype=np.int32)) == rec["tmfg_edges"]
    assert report.digest == rec["hub_digest"]
    assert orc.sha(np.asarray(flat, dtype=np.int64)) == rec["hub_labels"]
    assert report.num_converging == rec["hub_num_converging"]


def test_nan_is_stage_error_tmfg_insertion(pkg):
    """pipeline.py:149-153 + test_pipeline.py:116-120: a NaN in S surfaces as
    StageError('tmfg_insertion') (the sort accepts it; validation inside the TMFG stage raises)."""
    rng = np.random.default_rng(12)
    A = rng.random((60, 60))
    S = (A + A.T) / 2
    np.fill_diagonal(S, 1.0)
    S[5, 9] = S[9, 5] = np.nan
    with pytest.raises(pkg.StageError) as ei:
        pkg.run_stages(pkg.PipelineConfig(k=3), S)
    assert ei.value.stage == "tmfg_insertion"
    assert isinstance(ei.value.cause, pkg.DataError)
    assert str(ei.value.cause) == "similarity matrix contains NaN"


@pytest.mark.parametrize("n", [4, 5, 6])
def test_degenerate_sizes_through_the_pipeline(n, pkg):
    """n = 4 (no insertion), 5, 6 through every stage of both APSP modes, against the
    exhaustive-free structural invariants: 3n-6 edges, 2n-4 faces, n-1 merges."""
    rng = np.random.default_rng(n)
    A = rng.random((n, n))
    S = (A + A.T) / 2
    np.fill_diagonal(S, 1.0)
    for mode in ("exact", "hub"):
        report, g, d, flat = pkg.run_stages(pkg.PipelineConfig(apsp_mode=mode, k=2), S)
        assert g.edges.shape == (3 * n - 6, 2) and g.faces.shape == (2 * n - 4, 3)
        assert d.n_merges == n - 1
        d.validate()
        assert flat.shape == (n,) and flat.max() == 1
