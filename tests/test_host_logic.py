"""Host-side bookkeeping of the B200 package, checked on CPU against the oracle.

The GPU kernels produce raw NN-chain merges; canonicalisation, dendrogram
assembly and the cut are vectorised host code -- tested here without a GPU.
"""

from __future__ import annotations

import numpy as np
import pytest


def _raw_batch(oracle, mats):
    le, ri, he, off = [], [], [], [0]
    for M in mats:
        raw = oracle.nn_chain_raw(M)
        le += [r[0] for r in raw]
        ri += [r[1] for r in raw]
        he += [r[2] for r in raw]
        off.append(off[-1] + len(raw))
    return (np.array(le, dtype=np.int64), np.array(ri, dtype=np.int64), np.array(he, dtype=np.float64),
            np.array(off, dtype=np.int64))


@pytest.mark.parametrize("seed", range(4))
def test_canonicalize_batch_matches_nn_chain_merges(seed, oracle):
    from paper_2408_09399_b200.linkage import canonicalize_batch
    rng = np.random.default_rng(seed)
    mats = []
    for m in rng.integers(2, 40, size=6):
        A = np.round(rng.random((m, m)), 1)    # many equal heights
        mats.append((A + A.T) / 2)
    le, ri, he, off = _raw_batch(oracle, mats)
    sizes = np.array([M.shape[0] for M in mats])
    a, b, h = canonicalize_batch(le, ri, he, off, sizes)
    for k, M in enumerate(mats):
        ref = oracle.nn_chain_merges(M)
        got = list(zip(a[off[k]:off[k + 1]].tolist(), b[off[k]:off[k + 1]].tolist(), h[off[k]:off[k + 1]].tolist()))
        assert got == ref


@pytest.mark.parametrize("name", ["n30_u", "n120_q", "n200_s", "c1_n300"])
def test_dendrogram_and_cut_match_golden(name, small_cases, digests):
    from paper_2408_09399_b200.linkage import Dendrogram, cut, dendrogram_from_merges, serialize_dendrogram
    c = small_cases[name]
    for mode in ("exact", "hub"):
        rows = (c[f"{mode}_dend_lefts"], c[f"{mode}_dend_rights"], c[f"{mode}_dend_heights"])
        d = dendrogram_from_merges(c["S"].shape[0], rows)
        assert np.array_equal(d.sizes, c[f"{mode}_dend_sizes"])
        d.validate()
        import hashlib
        assert hashlib.sha256(serialize_dendrogram(d).encode()).hexdigest() == digests[name][f"{mode}_digest"]
        assert np.array_equal(cut(d, digests[name]["k"]), c[f"{mode}_labels"])
        for k in (1, 2, d.n_leaves):
            assert cut(d, k).max() == k - 1
        with pytest.raises(ValueError):
            cut(d, 0)


def test_group_tile_layout():
    """Tiles cover every sub-problem, row-major, with per-sub tile offsets."""
    from paper_2408_09399_b200.dbht import _SUB_DT, _TILE_DT, group_layout
    subs = [[np.arange(0, 70), np.arange(70, 75)], [np.arange(100, 101), np.arange(200, 330)]]
    perm, gid, sub_arr, tile_arr, out_len = group_layout(subs)
    assert sub_arr.dtype == _SUB_DT and tile_arr.dtype == _TILE_DT
    assert perm.tolist() == list(range(0, 75)) + [100] + list(range(200, 330))
    assert gid.tolist() == [0] * 70 + [1] * 5 + [0] + [1] * 130
    assert sub_arr["len"].tolist() == [75, 131]
    assert sub_arr["tile_off"].tolist() == [0, 4]
    assert tile_arr.shape[0] == 4 + 9
    assert out_len == 4 + 4


def test_pipeline_config_validation():
    from paper_2408_09399_b200 import PipelineConfig
    with pytest.raises(ValueError):
        PipelineConfig(apsp_mode="nope")
    with pytest.raises(ValueError):
        PipelineConfig(apsp_mode="exact", hub_count=3)
    with pytest.raises(ValueError):
        PipelineConfig(variant="nope")
    with pytest.raises(ValueError):
        PipelineConfig(prefix_size=0)
    PipelineConfig(variant="exact", prefix_size=7)
    PipelineConfig(apsp_mode="hub", hub_count=3, radius_factor=1.5, k=4)


def test_synth_configs_are_deterministic():
    from paper_2408_09399_b200 import synth
    for cfg in (1, 2, 3, 4):
        a, la = synth.generate(cfg, n=120)
        b, lb = synth.generate(cfg, n=120)
        assert np.array_equal(a, b) and np.array_equal(la, lb)
        assert a.shape == (120, synth.CONFIGS[cfg].length)
    x, lab = synth.generate(4, n=100)
    assert set(np.unique(x).tolist()) <= {-3.0, -2.0, -1.0, 0.0, 1.0, 2.0, 3.0}


def test_serialize_dendrogram_matches_python_format():
    """The C++ serializer is byte-identical to linkage.py:181-187's f"{h:.17g}" rows."""
    from paper_2408_09399_b200 import linkage
    rng = np.random.default_rng(5)
    k = 4000
    h = rng.standard_normal(k) * 10.0 ** rng.integers(-300, 300, k)
    h[:20] = [0.0, -0.0, 1e-12, 9.999999999999999e-13, 1.0, 0.1, 1e300, 5e-324, 2.5, 100.0, 1e16,
              123456789012345678.0, np.inf, -np.inf, 1e17, 1e-5, 1e-4, 123456.7, 1.7976931348623157e308,
              2.2250738585072014e-308]
    d = linkage.Dendrogram(n_leaves=k + 1, lefts=rng.integers(0, 10**6, k), rights=rng.integers(0, 10**6, k),
                           heights=h, sizes=rng.integers(2, 10**5, k))
    ref = "\n".join(f"{int(a)} {int(b)} {x:.17g} {int(s)}" for a, b, x, s in zip(d.lefts, d.rights, d.heights, d.sizes))
    assert linkage.serialize_dendrogram(d) == ref + "\n"
    empty = linkage.Dendrogram(n_leaves=1, lefts=np.zeros(0, np.int64), rights=np.zeros(0, np.int64),
                               heights=np.zeros(0), sizes=np.zeros(0, np.int64))
    assert linkage.serialize_dendrogram(empty) == ""


def test_cut_matches_oracle_every_k():
    """tg_cut_labels (C++ union-find) against the oracle's restatement of linkage.py:151-178 on
    a random n = 700 dendrogram for every k, and an out-of-range child id -> IndexError."""
    import random

    from oracle import oracle as orc
    from paper_2408_09399_b200.linkage import Dendrogram, cut

    n = 700
    rnd = random.Random(11)
    active, L, R, nxt = list(range(n)), [], [], n
    for _ in range(n - 1):
        a = active.pop(rnd.randrange(len(active)))
        b = active.pop(rnd.randrange(len(active)))
        L.append(min(a, b))
        R.append(max(a, b))
        active.append(nxt)
        nxt += 1
    lefts, rights = np.array(L, dtype=np.int64), np.array(R, dtype=np.int64)
    d = Dendrogram(n_leaves=n, lefts=lefts, rights=rights, heights=np.arange(n - 1, dtype=np.float64),
                   sizes=np.ones(n - 1, dtype=np.int64))
    od = {"n_leaves": n, "lefts": lefts, "rights": rights}
    for k in range(1, n + 1):
        assert np.array_equal(cut(d, k), orc.cut(od, k)), k
    bad = Dendrogram(n_leaves=n, lefts=np.where(np.arange(n - 1) == 3, 5 * n, lefts), rights=rights,
                     heights=d.heights, sizes=d.sizes)
    with pytest.raises(IndexError):
        cut(bad, 1)
