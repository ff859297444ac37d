"""GPU parity for the NN-chain linkage and the group-max kernels vs the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2408_09399_b200 as p
    p._native.load()
    return p


@pytest.mark.parametrize("m", [2, 3, 5, 17, 48, 49, 64, 130, 400, 2049, 2600, 7300])
def test_nn_chain_matches_oracle(m, oracle, pkg):
    rng = np.random.default_rng(m)
    A = rng.random((m, m))
    D = (A + A.T) / 2
    T = rng.random((m, m)) < 0.2
    T = T | T.T
    D[T] = 0.5                            # ties (kept symmetric)
    np.fill_diagonal(D, 0.0)
    assert pkg.nn_chain_merges(D) == oracle.nn_chain_merges(D)
    # hub-mode matrices are symmetric up to a few ulps: perturb some entries by 1 ulp
    B = D.copy()
    pick = rng.random((m, m)) < 0.05
    B[pick] = np.nextafter(B[pick], np.inf)
    assert pkg.nn_chain_merges(B) == oracle.nn_chain_merges(B)


@pytest.mark.parametrize("m", [60, 400, 1056, 2100])
def test_nn_chain_inf_and_signed_zero(m, oracle, pkg):
    """+inf entries (np.argmin over an all-inf row: index 0) and -0.0 == +0.0 ties (first index)."""
    rng = np.random.default_rng(100 + m)
    A = rng.random((m, m))
    D = (A + A.T) / 2
    I = rng.random((m, m)) < 0.3
    D[I | I.T] = np.inf
    Z = rng.random((m, m)) < 0.01
    D[Z] = 0.0
    D[Z.T & ~Z] = -0.0
    np.fill_diagonal(D, 0.0)
    D[: m // 10, :] = np.inf              # whole rows at +inf
    D[:, : m // 10] = np.inf
    assert pkg.nn_chain_merges(D) == oracle.nn_chain_merges(D)


def test_nn_chain_batch_mixed_sizes(oracle, pkg):
    import torch
    from paper_2408_09399_b200 import linkage
    rng = np.random.default_rng(7)
    sizes = np.array([2, 40, 49, 300, 5, 64], dtype=np.int64)
    mats = []
    for m in sizes:
        A = rng.random((m, m))
        mats.append((A + A.T) / 2)
    flat = np.concatenate([M.reshape(-1) for M in mats])
    off = np.zeros(len(sizes), dtype=np.int64)
    off[1:] = np.cumsum(sizes * sizes)[:-1]
    le, ri, he, mo = linkage.nn_chain_raw_batch(torch.from_numpy(flat).cuda(), sizes, off)
    for b, M in enumerate(mats):
        ref = oracle.nn_chain_raw(M)
        got = list(zip(le[mo[b]:mo[b + 1]].tolist(), ri[mo[b]:mo[b + 1]].tolist(), he[mo[b]:mo[b + 1]].tolist()))
        assert got == ref, b


@pytest.mark.parametrize("mode", ["exact", "hub"])
def test_group_max_matches_oracle(mode, small_cases, oracle, pkg):
    S = small_cases["n200_s"]["S"]
    g = pkg.build_tmfg_heap(S, pkg.sort_neighbor_lists(S))
    w = pkg.to_weighted(g, S)
    o = pkg.apsp_exact(w) if mode == "exact" else pkg.apsp_hub(w)
    og = oracle.build_tmfg_heap(S, oracle.sort_neighbor_lists(S))
    ow = oracle.to_weighted(og, S)
    oo = oracle.apsp_exact(ow) if mode == "exact" else oracle.apsp_hub(ow)
    rng = np.random.default_rng(3)
    perm = rng.permutation(200)
    for sizes in ([200], [1, 199], [50, 50, 100], [7] * 20 + [60], [3] * 66 + [2]):
        groups, s0 = [], 0
        for sz in sizes:
            groups.append(np.sort(perm[s0:s0 + sz]))
            s0 += sz
        got = pkg.dbht._cluster_max_matrix(o, groups)
        ref = oracle.cluster_max_matrix(oo, groups)
        m = len(groups)
        off = ~np.eye(m, dtype=bool)
        assert np.array_equal(got[off], ref[off]), sizes


def test_group_max_batched_subproblems(small_cases, oracle, pkg):
    """Several vertex-disjoint sub-problems in one launch equal separate calls."""
    S = small_cases["n200_s"]["S"]
    g = pkg.build_tmfg_heap(S, pkg.sort_neighbor_lists(S))
    o = pkg.apsp_hub(pkg.to_weighted(g, S))
    og = oracle.build_tmfg_heap(S, oracle.sort_neighbor_lists(S))
    oo = oracle.apsp_hub(oracle.to_weighted(og, S))
    perm = np.random.default_rng(5).permutation(200)
    subs = [[np.sort(perm[0:30]), np.sort(perm[30:90])], [np.sort(perm[90:91]), np.sort(perm[91:200])],
            [np.sort(perm[[0]])]][:2]
    out, meta = pkg.dbht.group_max_batch(o, subs)
    out = out.cpu().numpy()
    for p, groups in enumerate(subs):
        m = len(groups)
        got = out[meta["out_off"][p]: meta["out_off"][p] + m * m].reshape(m, m)
        ref = oracle.cluster_max_matrix(oo, groups)
        off = ~np.eye(m, dtype=bool)
        assert np.array_equal(got[off], ref[off])


def test_group_max_hub_screen_adversarial(pkg):
    """fp32-screened hub group max on hostile hub distances: exact zeros, ties, values that
    collide in fp32 but not fp64, denormals, values that overflow fp32, +inf -- against a
    direct fp64 evaluation of max_{u in I, v in J} min_h (hd[h,u] + hd[h,v]) (apsp.py:136-143)."""
    from paper_2408_09399_b200.apsp import HubOracle
    rng = np.random.default_rng(11)
    n, H = 300, 37
    hd = rng.uniform(0.5, 4.0, size=(H, n))
    hd[:, :20] = np.round(hd[:, :20], 1)                      # ties
    hd[:, 20:40] = 1.0 + rng.integers(0, 4, size=(H, 20)) * 2.0 ** -40   # fp32-equal, fp64-distinct
    hd[:, 40:45] = 0.0                                        # zero distances
    hd[3, 45:50] = 1e-310                                     # denormals
    hd[:, 50:55] = 1e39 * rng.uniform(1, 2, size=(H, 5))      # overflow fp32
    hd[:, 55:58] = np.inf                                     # unreachable
    nearest = np.zeros(n, dtype=np.int64)
    o = HubOracle(hubs=np.arange(H, dtype=np.int64), hub_dist=hd, nearest_hub=nearest,
                  nearest_dist=np.zeros(n), radii=np.zeros(n), near_indptr=np.zeros(n + 1, dtype=np.int64),
                  near_ids=np.zeros(0, dtype=np.int64), near_dist=np.zeros(0))
    perm = rng.permutation(n)
    for sizes in ([300], [10] * 30, [1, 2, 3, 4, 290], [64, 65, 171]):
        groups, s0 = [], 0
        for sz in sizes:
            groups.append(np.sort(perm[s0:s0 + sz]))
            s0 += sz
        got = pkg.dbht._cluster_max_matrix(o, groups)
        m = len(groups)
        for a in range(m):
            for b in range(m):
                if a == b:
                    continue
                I, J = groups[a], groups[b]
                est = (hd[:, I][:, :, None] + hd[:, J][:, None, :]).min(axis=0)
                assert got[a, b] == est.max(), (sizes, a, b)
