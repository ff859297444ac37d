"""CPU oracle for the TMFG-DBHT hot path -- TEST INFRASTRUCTURE ONLY.

Restates the reference package (`/root/reference/pkg/src/tmfgclust`, read-only
and absent on the GPU box) with plain C (``tmfg_oracle.c``, built into
``oracle/_build/liboracle.so``) for the loops the reference runs in numba or
pure Python, and numpy for the steps the reference itself does with numpy
(row centring, ``np.add.at`` strength, ``lexsort`` hub ranking, ...).

Who may use this module: ``tests/`` (as the checker), ``__graft_entry__.smoke()``
(as the checker) and ``bench.py`` (the ``cpu_baseline`` leg and ``--impl
reference``).  The product package ``paper_2408_09399_b200`` never imports it.

Parity of the oracle with the reference is pinned by ``tests/golden/``:
fixtures and digests produced by running the reference itself
(``tests/golden/make_golden.py``), checked by ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

HEIGHT_BUMP = 1e-12  # dbht.py:25


def build(force: bool = False) -> Path:
    """Compile tmfg_oracle.c with gcc (OpenMP, no FP contraction)."""
    src = _HERE / "tmfg_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        _LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
        subprocess.check_call(["make", "-s", "-C", str(_HERE)])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        _lib.orc_nn_chain.restype = ctypes.c_int64
        _lib.orc_tmfg_heap.restype = ctypes.c_int64
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _i(x) -> ctypes.c_int64:
    return ctypes.c_int64(int(x))


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- similarity
def pearson_similarity(x: np.ndarray) -> np.ndarray:
    """simmatrix.py:105-123 + _kernels.py:17-37 (numpy prologue, C kernel)."""
    x = np.asarray(x, dtype=np.float64)
    xc = x - x.mean(axis=1, keepdims=True)
    norm = np.sqrt(np.einsum("ij,ij->i", xc, xc))
    inv = np.zeros_like(norm)
    nz = norm > 0.0
    inv[nz] = 1.0 / norm[nz]
    xc = np.ascontiguousarray(xc)
    n, L = xc.shape
    out = np.empty((n, n))
    lib().orc_pearson(_p(xc), _p(inv), _i(n), _i(L), _p(out))
    return out


def validate_similarity(S: np.ndarray) -> str | None:
    """simmatrix.py:126-139; returns the DataError message or None."""
    if S.ndim != 2 or S.shape[0] != S.shape[1]:
        return f"similarity matrix must be square, got shape {S.shape}"
    if np.isnan(S).any():
        return "similarity matrix contains NaN"
    if not np.array_equal(S, S.T):
        return "similarity matrix is not symmetric"
    if not np.array_equal(np.diag(S), np.ones(S.shape[0])):
        return "similarity matrix diagonal must be exactly 1"
    if S.min() < -1.0 or S.max() > 1.0:
        return "similarity values must lie in [-1, 1]"
    return None


def sort_neighbor_lists(S: np.ndarray) -> np.ndarray:
    """simmatrix.py:225-249: (n, n-1) int32 ids by (S desc, id asc), v removed."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    n = S.shape[0]
    order = np.empty((n, max(n - 1, 0)), dtype=np.int32)
    lib().orc_sort_rows(_p(S), _i(n), _p(order))
    return order


def select_initial_clique(S: np.ndarray) -> tuple:
    """tmfg.py:71-79 (numpy pairwise row sums, restated in C)."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    out = np.empty(4, dtype=np.int32)
    lib().orc_initial_clique(_p(S), _i(S.shape[0]), _p(out))
    return tuple(int(v) for v in out)


# ---------------------------------------------------------------------- TMFG
def build_tmfg_heap(S: np.ndarray, order: np.ndarray) -> dict:
    """tmfg.py:344-436.  Returns the TmfgGraph arrays + host face ids + stats."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    n = S.shape[0]
    clique = np.array(select_initial_clique(S), dtype=np.int32)
    trace = np.zeros((max(n - 4, 0), 4), dtype=np.int32)
    host = np.zeros(max(n - 4, 0), dtype=np.int32)
    edges = np.zeros((3 * n - 6, 2), dtype=np.int32)
    faces = np.zeros((2 * n - 4, 3), dtype=np.int32)
    stats = np.zeros(3, dtype=np.int64)
    order = np.ascontiguousarray(order, dtype=np.int32)
    nt = lib().orc_tmfg_heap(_p(S), _p(order), _i(n), _p(clique), _p(trace), _p(host),
                             _p(edges), _p(faces), _p(stats))
    assert nt == n - 4
    weights = S[edges[:, 0], edges[:, 1]].astype(np.float64)
    return dict(n=n, edges=edges, weights=weights, initial_clique=clique, trace=trace,
                host_fid=host, faces=faces,
                stats={"pops": int(stats[0]), "refreshes": int(stats[1]),
                       "gain_increases": int(stats[2])})


# ---------------------------------------------------------------------- APSP
def to_weighted(graph: dict, S: np.ndarray) -> dict:
    """apsp.py:52-77: lengths sqrt(max(2(1-s),0)); CSR filled in edge order."""
    n = graph["n"]
    e = graph["edges"].astype(np.int64)
    sims = S[e[:, 0], e[:, 1]]
    lengths = np.sqrt(np.maximum(2.0 * (1.0 - sims), 0.0))
    # the reference's cursor loop visits (i->j), (j->i) per edge in edge order;
    # a stable sort of that interleaved sequence by source vertex is the same CSR
    src = np.stack([e[:, 0], e[:, 1]], axis=1).reshape(-1)
    dst = np.stack([e[:, 1], e[:, 0]], axis=1).reshape(-1)
    wl = np.repeat(lengths, 2)
    perm = np.argsort(src, kind="stable")
    deg = np.bincount(src, minlength=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=indptr[1:])
    strength = np.zeros(n)
    np.add.at(strength, e[:, 0], sims)
    np.add.at(strength, e[:, 1], sims)
    return dict(n=n, indptr=indptr, neighbors=dst[perm].astype(np.int64),
                lengths=wl[perm].astype(np.float64), strength=strength)


def dijkstra_rows(w: dict, sources: np.ndarray) -> np.ndarray:
    n = w["n"]
    sources = np.ascontiguousarray(sources, dtype=np.int64)
    out = np.empty((sources.shape[0], n))
    lib().orc_dijkstra_rows(_p(w["indptr"]), _p(w["neighbors"]), _p(w["lengths"]), _i(n),
                            _p(sources), _i(sources.shape[0]), _p(out))
    return out


def apsp_exact(w: dict) -> dict:
    """apsp.py:164-171."""
    return dict(mode="exact", matrix=dijkstra_rows(w, np.arange(w["n"], dtype=np.int64)))


def select_hubs(w: dict, hub_count: int) -> np.ndarray:
    """apsp.py:178-186: (strength desc, id asc)."""
    ids = np.arange(w["n"])
    return ids[np.lexsort((ids, -w["strength"]))][:hub_count].astype(np.int64)


def apsp_hub(w: dict, hub_count: int | None = None, radius_factor: float = 2.0) -> dict:
    """apsp.py:189-230."""
    n = w["n"]
    H = hub_count or min(n, math.ceil(math.sqrt(n)))
    hubs = select_hubs(w, H)
    hub_dist = dijkstra_rows(w, hubs)
    nearest_idx = np.argmin(hub_dist, axis=0)
    nearest_dist = hub_dist[nearest_idx, np.arange(n)]
    nearest_hub = hubs[nearest_idx]
    radii = np.ascontiguousarray(radius_factor * nearest_dist)
    counts = np.zeros(n, dtype=np.int64)
    L = lib()
    L.orc_truncated_counts(_p(w["indptr"]), _p(w["neighbors"]), _p(w["lengths"]), _i(n),
                           _p(radii), _p(counts))
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    ids = np.empty(offsets[-1], dtype=np.int64)
    dists = np.empty(offsets[-1], dtype=np.float64)
    off = np.ascontiguousarray(offsets[:-1])
    L.orc_truncated_fill(_p(w["indptr"]), _p(w["neighbors"]), _p(w["lengths"]), _i(n),
                         _p(radii), _p(off), _p(ids), _p(dists))
    seg = np.repeat(np.arange(n), counts)
    perm = np.lexsort((ids, seg))
    return dict(mode="hub", hubs=hubs, hub_dist=hub_dist, nearest_hub=nearest_hub,
                nearest_dist=nearest_dist, radii=radii, near_indptr=offsets,
                near_ids=ids[perm], near_dist=dists[perm])


def _near_lookup(o, u, v):
    lo, hi = o["near_indptr"][u], o["near_indptr"][u + 1]
    ids = o["near_ids"][lo:hi]
    k = np.searchsorted(ids, v)
    if k < ids.shape[0] and ids[k] == v:
        return float(o["near_dist"][lo + k])
    return None


def query(o: dict, u: int, v: int) -> float:
    """apsp.py:88-90 / 127-136."""
    if o["mode"] == "exact":
        return float(o["matrix"][u, v])
    if u == v:
        return 0.0
    u, v = (u, v) if u < v else (v, u)
    d = _near_lookup(o, u, v)
    if d is None:
        d = _near_lookup(o, v, u)
    if d is not None:
        return d
    return float(np.min(o["hub_dist"][:, u] + o["hub_dist"][:, v]))


def block(o: dict, rows, cols) -> np.ndarray:
    """apsp.py:92-94 / 138-158 (dense block; used for the small layer-1 groups)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if o["mode"] == "exact":
        return o["matrix"][np.ix_(rows, cols)]
    hd = o["hub_dist"]
    est = np.min(hd[:, rows][:, :, None] + hd[:, cols][:, None, :], axis=0)
    n = hd.shape[1]
    ip, ni, nd = o["near_indptr"], o["near_ids"], o["near_dist"]
    cpos = np.full(n, -1, dtype=np.int64)
    cpos[cols] = np.arange(cols.shape[0])
    for i, u in enumerate(rows):
        p = cpos[ni[ip[u]:ip[u + 1]]]
        k = p >= 0
        est[i, p[k]] = nd[ip[u]:ip[u + 1]][k]
    rpos = np.full(n, -1, dtype=np.int64)
    rpos[rows] = np.arange(rows.shape[0])
    for j, v in enumerate(cols):
        p = rpos[ni[ip[v]:ip[v + 1]]]
        k = p >= 0
        est[p[k], j] = nd[ip[v]:ip[v + 1]][k]
    return est


def _reverse_near(o: dict):
    """Transposed near table: for each u, the (v, near_v(u)) with u in near(v)."""
    if "_rev" in o:
        return o["_rev"]
    n = o["near_indptr"].shape[0] - 1
    counts = np.diff(o["near_indptr"])
    owner = np.repeat(np.arange(n, dtype=np.int64), counts)
    perm = np.argsort(o["near_ids"], kind="stable")
    rev_ids = owner[perm]
    rev_dist = o["near_dist"][perm]
    rev_indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(o["near_ids"], minlength=n), out=rev_indptr[1:])
    o["_rev"] = (rev_indptr, np.ascontiguousarray(rev_ids), np.ascontiguousarray(rev_dist))
    return o["_rev"]


def cluster_max_matrix(o: dict, member_lists) -> np.ndarray:
    """dbht.py:217-230."""
    concat = np.ascontiguousarray(np.concatenate([np.asarray(m, dtype=np.int64) for m in member_lists]))
    starts = np.zeros(len(member_lists) + 1, dtype=np.int64)
    np.cumsum([len(m) for m in member_lists], out=starts[1:])
    m = len(member_lists)
    out = np.empty((m, m))
    L = lib()
    if o["mode"] == "exact":
        D = np.ascontiguousarray(o["matrix"])
        L.orc_segment_pair_max(_p(D), _i(D.shape[0]), _p(concat), _p(starts), _i(m), _p(out))
    else:
        rip, rid, rdd = _reverse_near(o)
        hd = np.ascontiguousarray(o["hub_dist"])
        L.orc_hub_group_max(_p(hd), _i(hd.shape[0]), _i(hd.shape[1]), _p(o["near_indptr"]),
                            _p(o["near_ids"]), _p(o["near_dist"]), _p(rip), _p(rid), _p(rdd),
                            _p(concat), _p(starts), _i(m), _p(out))
    return out


# ---------------------------------------------------------------------- DBHT
def build_bubble_tree(graph: dict) -> dict:
    """dbht.py:64-89: bubble per trace row, linked to the owner of the host face."""
    a, b, c, d = (int(x) for x in graph["initial_clique"])
    bubbles = [(a, b, c, d)]
    owner = {(a, b, c): 0, (a, b, d): 0, (a, c, d): 0, (b, c, d): 0}
    links, link_faces = [], []
    for row in graph["trace"].tolist():
        v, x, y, z = row
        host = tuple(sorted((x, y, z)))
        ob = owner.pop(host)
        bid = len(bubbles)
        bubbles.append(tuple(sorted((v, x, y, z))))
        links.append((ob, bid))
        link_faces.append(host)
        for f in ((v, x, y), (v, x, z), (v, y, z)):
            owner[tuple(sorted(f))] = bid
    return dict(n=graph["n"], bubbles=np.array(bubbles, dtype=np.int32),
                links=np.array(links, dtype=np.int32).reshape(-1, 2),
                link_faces=np.array(link_faces, dtype=np.int32).reshape(-1, 3))


def _apex(bubble, face) -> int:
    fs = set(int(x) for x in face)
    for w in bubble:
        if int(w) not in fs:
            return int(w)
    raise ValueError("bubble does not extend the face")


def _gain(face, v, S) -> float:
    a, b, c = sorted(int(x) for x in face)
    return float(S[a, v] + S[b, v] + S[c, v])


def orient_edges(tree: dict, S: np.ndarray) -> dict:
    """dbht.py:100-117: toward the larger apex gain; ties toward the lower index."""
    L = tree["links"].shape[0]
    sources = np.empty(L, dtype=np.int64)
    targets = np.empty(L, dtype=np.int64)
    for i in range(L):
        b1, b2 = int(tree["links"][i, 0]), int(tree["links"][i, 1])
        face = tree["link_faces"][i]
        g1 = _gain(face, _apex(tree["bubbles"][b1], face), S)
        g2 = _gain(face, _apex(tree["bubbles"][b2], face), S)
        if g2 > g1:
            s, t = b1, b2
        elif g1 > g2:
            s, t = b2, b1
        else:
            s, t = (b1, b2) if b2 < b1 else (b2, b1)
        sources[i], targets[i] = s, t
    return dict(tree=tree, sources=sources, targets=targets)


def converging_bubbles(dtree: dict) -> list:
    """dbht.py:120-122."""
    m = dtree["tree"]["bubbles"].shape[0]
    out = np.zeros(m, dtype=np.int64)
    np.add.at(out, dtree["sources"], 1)
    return [int(b) for b in np.flatnonzero(out == 0)]


def bubble_sinks(dtree: dict, graph: dict) -> np.ndarray:
    """dbht.py:143-175: next hop by max apex gain from edge weights, then path follow."""
    tree = dtree["tree"]
    m = tree["bubbles"].shape[0]
    wts = {(int(i), int(j)): float(x) for (i, j), x in zip(graph["edges"], graph["weights"])}
    best = np.full(m, -np.inf)
    hops = np.full(m, -1, dtype=np.int64)
    for i in range(dtree["sources"].shape[0]):
        s, t = int(dtree["sources"][i]), int(dtree["targets"][i])
        face = tree["link_faces"][i]
        apex = _apex(tree["bubbles"][t], face)
        g = 0.0
        for w in sorted(int(x) for x in face):
            g += wts[(w, apex) if w < apex else (apex, w)]
        if g > best[s] or (g == best[s] and t < hops[s]):
            best[s], hops[s] = g, t
    sinks = np.full(m, -1, dtype=np.int64)
    for b in range(m):
        path, cur = [], b
        while sinks[cur] < 0 and hops[cur] >= 0:
            path.append(cur)
            cur = int(hops[cur])
        sink = cur if sinks[cur] < 0 else int(sinks[cur])
        sinks[cur] = sink
        for node in path:
            sinks[node] = sink
    return sinks


def assign_vertices(graph: dict, dtree: dict, o: dict) -> dict:
    """dbht.py:178-214 (per-vertex loop in C)."""
    tree = dtree["tree"]
    n = tree["n"]
    bubbles = np.ascontiguousarray(tree["bubbles"], dtype=np.int32)
    flat = bubbles.reshape(-1).astype(np.int64)
    bid = np.repeat(np.arange(bubbles.shape[0], dtype=np.int64), 4)
    perm = np.argsort(flat, kind="stable")
    cont_ids = np.ascontiguousarray(bid[perm])
    cont_ip = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(flat, minlength=n), out=cont_ip[1:])
    vb = np.empty(n, dtype=np.int64)
    dummy = np.zeros(1)
    dummy_i = np.zeros(2, dtype=np.int64)
    if o["mode"] == "exact":
        D = np.ascontiguousarray(o["matrix"])
        lib().orc_assign(0, _p(D), _p(dummy), _i(0), _p(dummy_i), _p(dummy_i), _p(dummy), _i(n),
                         _p(bubbles), _p(cont_ip), _p(cont_ids), _p(vb))
    else:
        hd = np.ascontiguousarray(o["hub_dist"])
        lib().orc_assign(1, _p(dummy), _p(hd), _i(hd.shape[0]), _p(o["near_indptr"]),
                         _p(o["near_ids"]), _p(o["near_dist"]), _i(n), _p(bubbles), _p(cont_ip),
                         _p(cont_ids), _p(vb))
    sinks = bubble_sinks(dtree, graph)
    return dict(vertex_bubble=vb, vertex_converging=sinks[vb].astype(np.int64))


# ------------------------------------------------------------------- linkage
def nn_chain_raw(D: np.ndarray) -> list:
    """linkage.py:50-94."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    m = D.shape[0]
    if m < 2:
        return []
    lefts = np.empty(m, dtype=np.int64)
    rights = np.empty(m, dtype=np.int64)
    heights = np.empty(m)
    k = lib().orc_nn_chain(_p(D), _i(m), _p(lefts), _p(rights), _p(heights))
    if k < 0:
        raise RuntimeError("NN-chain does not terminate on this (non-reducible) matrix")
    return [(int(lefts[t]), int(rights[t]), float(heights[t])) for t in range(k)]


def nn_chain_merges(D: np.ndarray) -> list:
    """linkage.py:97-116: stable height sort, renumber m+rank, (min, max, h)."""
    m = D.shape[0]
    raw = nn_chain_raw(D)
    order = sorted(range(len(raw)), key=lambda t: raw[t][2])
    remap = {m + t: m + r for r, t in enumerate(order)}
    rows = []
    for t in order:
        a, b, h = raw[t]
        a, b = remap.get(a, a), remap.get(b, b)
        rows.append((min(a, b), max(a, b), h))
    return rows


def dendrogram_from_merges(n_leaves: int, merges) -> dict:
    """linkage.py:136-148."""
    sizes = np.empty(len(merges), dtype=np.int64)
    size_of = {}
    for t, (a, b, _) in enumerate(merges):
        s = size_of.get(a, 1) + size_of.get(b, 1)
        size_of[n_leaves + t] = s
        sizes[t] = s
    return dict(n_leaves=n_leaves,
                lefts=np.array([r[0] for r in merges], dtype=np.int64),
                rights=np.array([r[1] for r in merges], dtype=np.int64),
                heights=np.array([r[2] for r in merges], dtype=np.float64),
                sizes=sizes)


def build_hierarchy(asg: dict, dtree: dict, o: dict) -> dict:
    """dbht.py:233-339: three complete-linkage layers with a running height floor."""
    n = asg["vertex_bubble"].shape[0]
    groups: dict = {}
    for v in range(n):
        groups.setdefault(int(asg["vertex_bubble"][v]), []).append(v)
    bubble_ids = sorted(groups)
    records: list = []

    def rec(left, right, h):
        records.append((left, right, h))
        return n + len(records) - 1

    def linkage_over(handles, M):
        local = dict(enumerate(handles))
        rows, root = [], handles[0]
        for t, (li, ri, h) in enumerate(nn_chain_merges(M)):
            r = rec(local[li], local[ri], h)
            local[len(handles) + t] = r
            rows.append((r, h))
            root = r
        return root, rows

    layer1, group_root = [], {}
    for bid in bubble_ids:
        mem = groups[bid]
        if len(mem) == 1:
            group_root[bid] = mem[0]
            continue
        D = block(o, mem, mem)
        handle = dict(enumerate(mem))
        r = None
        for t, (li, ri, h) in enumerate(nn_chain_merges(D)):
            r = rec(handle[li], handle[ri], h)
            handle[len(mem) + t] = r
            layer1.append((r, h))
        group_root[bid] = r
    layer1.sort(key=lambda x: x[1])

    conv_groups: dict = {}
    for bid in bubble_ids:
        conv_groups.setdefault(int(asg["vertex_converging"][groups[bid][0]]), []).append(bid)
    conv_ids = sorted(conv_groups)
    layer2, conv_root = [], {}
    for c in conv_ids:
        bids = conv_groups[c]
        if len(bids) == 1:
            conv_root[c] = group_root[bids[0]]
            continue
        M = cluster_max_matrix(o, [groups[b] for b in bids])
        root, rows = linkage_over([group_root[b] for b in bids], M)
        conv_root[c] = root
        layer2.extend(rows)
    layer2.sort(key=lambda x: x[1])

    layer3 = []
    if len(conv_ids) > 1:
        members = [sorted(v for b in conv_groups[c] for v in groups[b]) for c in conv_ids]
        M = cluster_max_matrix(o, members)
        _, layer3 = linkage_over([conv_root[c] for c in conv_ids], M)
        layer3.sort(key=lambda x: x[1])

    final, fid, floor = [], {}, -np.inf
    for rows in (layer1, layer2, layer3):
        for handle, _ in rows:
            left, right, h = records[handle - n]
            if h < floor:
                h = floor + HEIGHT_BUMP
            floor = h
            li, ri = fid.get(left, left), fid.get(right, right)
            fid[handle] = n + len(final)
            final.append((min(li, ri), max(li, ri), h))
    return dendrogram_from_merges(n, final)


def cut(d: dict, k: int) -> np.ndarray:
    """linkage.py:151-178."""
    n = d["n_leaves"]
    if not 1 <= k <= n:
        raise ValueError(f"cluster count k={k} out of range 1..{n}")
    parent = list(range(2 * n - 1))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for t in range(n - k):
        for child in (int(d["lefts"][t]), int(d["rights"][t])):
            parent[find(child)] = n + t
    roots, labels = {}, np.empty(n, dtype=np.int64)
    for leaf in range(n):
        r = find(leaf)
        if r not in roots:
            roots[r] = len(roots)
        labels[leaf] = roots[r]
    return labels


def serialize_dendrogram(d: dict) -> str:
    """linkage.py:181-187."""
    lines = [f"{int(a)} {int(b)} {h:.17g} {int(s)}"
             for a, b, h, s in zip(d["lefts"], d["rights"], d["heights"], d["sizes"])]
    return "\n".join(lines) + ("\n" if lines else "")


def dendrogram_digest(d: dict) -> str:
    """pipeline.py:226-227."""
    return hashlib.sha256(serialize_dendrogram(d).encode()).hexdigest()


# ------------------------------------------------------------------ pipeline
def run_stages(S: np.ndarray, k: int, apsp_mode: str = "exact", hub_count=None,
               radius_factor: float = 2.0, keep: bool = False) -> dict:
    """pipeline.py:173-239 (heap variant): sort -> TMFG -> APSP -> DBHT -> cut."""
    import time
    t = {}
    t0 = time.perf_counter()
    order = sort_neighbor_lists(S)
    t["sorting"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    msg = validate_similarity(S)
    if msg is not None:
        raise ValueError(msg)
    graph = build_tmfg_heap(S, order)
    t["tmfg_insertion"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    w = to_weighted(graph, S)
    o = apsp_exact(w) if apsp_mode == "exact" else apsp_hub(w, hub_count, radius_factor)
    t["apsp"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tree = build_bubble_tree(graph)
    dtree = orient_edges(tree, S)
    asg = assign_vertices(graph, dtree, o)
    t["dbht"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    d = build_hierarchy(asg, dtree, o)
    labels = cut(d, k)
    t["linkage"] = time.perf_counter() - t0
    out = dict(digest=dendrogram_digest(d), labels=labels, dendrogram=d, seconds=t,
               num_converging=int(np.unique(asg["vertex_converging"]).size))
    if keep:
        out.update(order=order, graph=graph, weighted=w, oracle=o, tree=tree, dtree=dtree,
                   assignment=asg)
    return out


if __name__ == "__main__":  # pragma: no cover
    build(force=True)
    print("built", _LIB_PATH, "threads", num_threads(), os.cpu_count())
