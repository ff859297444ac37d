"""GPU parity of the exact and corr TMFG builders (tmfg.py:208-341) against the reference.

Golden records: tests/golden/variants.json, made by running the unmodified reference
(tests/golden/make_variants.py) -- sha256 of trace / edges / faces / clique / weights for
every small case and BASELINE configs 1 and 2, prefix sizes 1, 3 and 17; and the config-1
pipeline (dendrogram digest, labels, edge_sum, ARI, edge_sum_delta) per variant.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

VAR = json.loads((GOLDEN / "variants.json").read_text())
CASES = sorted(k for k in VAR if not k.startswith("_") and k != "config1_pipeline")


@pytest.fixture(scope="module")
def pkg():
    import paper_2408_09399_b200 as p
    p._native.load()
    return p


def _S(name, small_cases, oracle):
    if name.startswith("config"):
        from paper_2408_09399_b200 import synth
        x, _ = synth.generate(int(name[-1]))
        return oracle.pearson_similarity(x)
    return small_cases[name]["S"]


@pytest.mark.parametrize("name", CASES)
def test_exact_and_corr_builders_match_reference(name, small_cases, oracle, pkg):
    rec = VAR[name]
    S = _S(name, small_cases, oracle)
    assert oracle.sha(S) == rec["S"]
    lists = pkg.sort_neighbor_lists(S)
    for p in (1, 3, 17):
        for variant in ("exact", "corr"):
            cfg = pkg.BuildConfig(variant=variant, prefix_size=p)
            g = pkg.build_tmfg(S, lists, cfg)
            assert g.variant == variant
            for key, want in rec[f"{variant}_p{p}"].items():
                assert oracle.sha(getattr(g, key)) == want, (variant, p, key)


def test_variant_graphs_are_valid_tmfgs(small_cases, pkg):
    S = small_cases["n200_s"]["S"]
    lists = pkg.sort_neighbor_lists(S)
    for variant, p in (("exact", 1), ("corr", 5)):
        g = pkg.build_tmfg(S, lists, pkg.BuildConfig(variant=variant, prefix_size=p))
        edges, live = pkg.replay_trace(g)
        assert edges == {tuple(e) for e in g.edges.tolist()}
        assert live == {tuple(f) for f in g.faces.tolist()}
        assert g.edges.shape == (3 * 200 - 6, 2) and g.faces.shape == (2 * 200 - 4, 3)


@pytest.mark.parametrize("variant,p", [("exact", 1), ("exact", 3), ("corr", 1), ("heap", 1)])
def test_pipeline_variants_match_reference(variant, p, oracle, pkg):
    from paper_2408_09399_b200 import synth
    rec = VAR["config1_pipeline"][f"{variant}_p{p}"]
    x, labels = synth.generate(1)
    S = oracle.pearson_similarity(x)
    report, g, d, flat = pkg.run_stages(pkg.PipelineConfig(variant=variant, prefix_size=p, k=5), S, labels)
    assert report.digest == rec["digest"]
    assert oracle.sha(np.asarray(flat)) == rec["labels"]
    assert report.edge_sum == rec["edge_sum"]
    assert report.ari == rec["ari"]


def test_compare_variants_and_run_pipeline_from_matrix_file(tmp_path, oracle, pkg):
    from paper_2408_09399_b200 import synth
    x, labels = synth.generate(1)
    S = oracle.pearson_similarity(x)
    path = tmp_path / "S.bin"
    pkg.write_matrix_binary(path, S)
    cfg = pkg.PipelineConfig(input_path=str(path), input_format="matrix", k=5, out_dir=str(tmp_path / "out"))
    rows = pkg.compare_variants(cfg, ["exact:3", "corr", "heap"])
    for row in rows:
        name, p = pkg.parse_variant_token(row["variant"])
        rec = VAR["config1_pipeline"][f"{name}_p{p}"]
        assert row["report"].digest == rec["digest"]
        assert row["edge_sum_delta"] == rec["edge_sum_delta"]
    rep = pkg.run_pipeline(pkg.PipelineConfig(input_path=str(path), input_format="matrix", k=5,
                                              out_dir=str(tmp_path / "out"), include_baseline_delta=True))
    assert rep.digest == VAR["config1_pipeline"]["heap_p1"]["digest"]
    assert rep.edge_sum_delta == VAR["config1_pipeline"]["heap_p1"]["edge_sum_delta"]
    d = pkg.load_dendrogram(tmp_path / "out" / "dendrogram.txt")
    import hashlib
    assert hashlib.sha256(pkg.serialize_dendrogram(d).encode()).hexdigest() == rep.digest
    assert json.loads((tmp_path / "out" / "report.json").read_text())["digest"] == rep.digest
