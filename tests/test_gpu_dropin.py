"""The drop-in route north_star names: the reference's OWN pipeline and tests on the B200 path.

* ``tmfgclust.pipeline.run_stages`` (pipeline.py:173-239, resolving stage functions on its modules
  at call time, 191-223) after ``paper_2408_09399_b200.install()``: dendrogram digest, cut labels
  and converging-group count equal the goldens made by running the unmodified reference
  (tests/golden/make_golden.py) on BASELINE configs 1, 2, 4 (exact and hub) and 3 (hub).
* The reference's unmodified test suite (pkg/tests: simmatrix, tmfg, apsp, dbht, linkage,
  pipeline, metrics, acceptance criteria 1-9) run under ``install()`` in a child pytest
  (tests/ref_install_plugin.py).  Criterion 10 is a CPU thread-scaling benchmark of the
  reference itself and is deselected.
* Exception compatibility: after install() the B200 path raises the reference's own
  TraceError / DataError (reference tests/test_dbht.py:90, tests/test_pipeline.py:116-120).

``baseline/_ref`` holds the reference package and its tests (tools/install_reference.sh); it is
git-ignored and travels to the GPU box with the snapshot.  Without it these tests skip.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent
REF = REPO / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "tmfgclust").is_dir():
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tg_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import tmfgclust
    import tmfgclust.pipeline

    import paper_2408_09399_b200 as p
    p._native.load()
    saved = p.install(tmfgclust)
    yield tmfgclust
    p.uninstall(saved)


def test_install_rebinds_reference_modules(ref):
    import paper_2408_09399_b200 as p
    assert ref.simmatrix.sort_neighbor_lists is p.sort_neighbor_lists
    assert ref.tmfg.build_tmfg_heap is p.build_tmfg_heap
    assert ref.apsp.apsp_hub is p.apsp_hub
    assert ref.dbht.build_hierarchy is p.build_hierarchy
    assert p.dbht.TraceError is ref.tmfg.TraceError
    assert p.simmatrix.DataError is ref.simmatrix.DataError


@pytest.mark.parametrize("config,mode", [(1, "exact"), (1, "hub"), (2, "exact"), (2, "hub"), (4, "exact"),
                                         (4, "hub"), (3, "hub")])
def test_reference_run_stages_under_install(config, mode, ref, digests, oracle):
    from paper_2408_09399_b200 import synth
    rec = digests[f"config{config}"]
    x, labels = synth.generate(config)
    S = oracle.pearson_similarity(x)
    assert oracle.sha(S) == rec["S"]
    cfg = ref.pipeline.PipelineConfig(apsp_mode=mode, k=rec["k"])
    report, graph, dend, flat = ref.pipeline.run_stages(cfg, S, labels)
    assert report.digest == rec[f"{mode}_digest"]
    assert oracle.sha(np.asarray(flat)) == rec[f"{mode}_labels"]
    assert report.num_converging == rec[f"{mode}_num_converging"]
    assert oracle.sha(graph.edges) == rec["tmfg_edges"]
    assert set(report.stage_seconds) == set(ref.pipeline.STAGES)


def test_reference_corrupt_trace_raises_reference_traceerror(ref, small_cases):
    c = small_cases["n50_s"]
    S = c["S"]
    g = ref.tmfg.build_tmfg_heap(S, ref.simmatrix.sort_neighbor_lists(S))
    trace = g.trace.copy()
    v, x, y, _ = trace[2]
    trace[2, 1:] = sorted((int(v), int(x), int(y)))   # a face containing the vertex itself: never live
    bad = ref.tmfg.TmfgGraph(n=g.n, edges=g.edges, weights=g.weights, initial_clique=g.initial_clique,
                             trace=trace, faces=g.faces, variant="heap")
    with pytest.raises(ref.tmfg.TraceError):
        ref.dbht.build_bubble_tree(bad)


def test_reference_nan_is_stage_error_under_install(ref):
    rng = np.random.default_rng(3)
    A = rng.random((40, 40))
    S = (A + A.T) / 2
    np.fill_diagonal(S, 1.0)
    S[3, 7] = S[7, 3] = np.nan
    with pytest.raises(ref.pipeline.StageError) as ei:
        ref.pipeline.run_stages(ref.pipeline.PipelineConfig(k=3), S)
    assert ei.value.stage == "tmfg_insertion"
    assert isinstance(ei.value.cause, ref.simmatrix.DataError)


def test_reference_test_suite_under_install(ref):
    """The reference's unmodified pkg/tests, run with install() active (child pytest)."""
    tests = REF / "tests"
    if not tests.is_dir():
        pytest.skip("baseline/_ref/tests not present")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(REPO / "tests"), str(REPO)])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/tg_numba_cache")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_install_plugin", "-p", "no:cacheprovider",
           "--deselect", "test_acceptance.py::test_criterion_10_performance", "-rfE", "."]
    r = subprocess.run(cmd, cwd=str(tests), env=env, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    log = REPO / "gpurun_out"
    if log.is_dir():
        (log / "reference_suite_under_install.log").write_text(out)
    print(out[-3000:])
    assert "rebound to the B200 path" in out
    assert r.returncode == 0, out[-6000:]


def test_in_place_edit_between_stage_calls_is_seen(oracle):
    """An in-place edit of S between sort_neighbor_lists and build_tmfg_heap (and before
    to_weighted) gives the reference's result for the edited S: no stale device copy."""
    import paper_2408_09399_b200 as p
    from paper_2408_09399_b200 import synth
    p._native.load()
    x, _ = synth.generate(2, n=600, seed=11)
    S = oracle.pearson_similarity(x)
    order0 = oracle.sort_neighbor_lists(S)
    ref0 = oracle.build_tmfg_heap(S, order0)
    lists = p.sort_neighbor_lists(S)
    # weaken an edge the unedited TMFG inserts early, far from any strided sample position
    a, b = (int(v) for v in ref0["edges"][40])
    S[a, b] = S[b, a] = -0.25
    ref1 = oracle.build_tmfg_heap(S, order0)
    assert not np.array_equal(ref1["trace"], ref0["trace"]), "edit must change the reference's result"
    g = p.build_tmfg_heap(S, lists)
    assert np.array_equal(g.trace, ref1["trace"])
    assert np.array_equal(g.edges, ref1["edges"])
    assert np.array_equal(g.weights, ref1["weights"])
    S[int(ref1["edges"][7][0]), int(ref1["edges"][7][1])] = 0.5   # asymmetric edit: lengths read S[e0, e1]
    w = p.to_weighted(g, S)
    wref = oracle.to_weighted(ref1, S)
    assert np.array_equal(w.lengths, wref["lengths"])


def test_reference_compare_variants_under_install(ref, oracle, tmp_path):
    """compare_variants (pipeline.py:295-315) through the reference's own driver: every builder,
    including exact:3 and corr, runs on the B200 after install()."""
    import json as _json
    from paper_2408_09399_b200 import synth
    var = _json.loads((REPO / "tests" / "golden" / "variants.json").read_text())["config1_pipeline"]
    x, labels = synth.generate(1)
    S = oracle.pearson_similarity(x)
    path = tmp_path / "S.bin"
    ref.simmatrix.write_matrix_binary(path, S)
    cfg = ref.pipeline.PipelineConfig(input_path=str(path), input_format="matrix", k=5)
    rows = ref.pipeline.compare_variants(cfg, ["exact:3", "corr", "heap"])
    for row in rows:
        name, p = ref.pipeline.parse_variant_token(row["variant"])
        assert row["report"].digest == var[f"{name}_p{p}"]["digest"]
        assert row["edge_sum_delta"] == var[f"{name}_p{p}"]["edge_sum_delta"]
