"""DBHT over a built TMFG on the B200 (drop-in for tmfgclust.dbht).

Mirrors dbht.py:28-61 (BubbleTree, DirectedBubbleTree, BubbleAssignment),
64-122 (build_bubble_tree, orient_edges, converging_bubbles), 143-214
(_next_hops, bubble_sinks, assign_vertices) and 217-339 (_cluster_max_matrix,
build_hierarchy).  All distance work -- layer-1 blocks, the layer-2/3 group-max
matrices (hub min-plus with near-table overrides) and every NN-chain -- runs in
csrc/dbht.cu; the host only arranges group index arrays (vectorised numpy) and
emits the merge records.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .apsp import _oracle_struct, as_oracle
from .linkage import Dendrogram, canonicalize_batch, dendrogram_from_merges, nn_chain_raw_batch
from .tmfg import TraceError

HEIGHT_BUMP = 1e-12


class BubbleTree:
    """Bubbles (4-cliques) of a TMFG linked through shared faces (dbht.py:28-39)."""

    def __init__(self, n, bubbles, links, link_faces, S_device=None, S_host=None):
        self.n = int(n)
        self._b = D.LazyHost(dev=bubbles) if D.is_device(bubbles) else D.LazyHost(host=np.asarray(bubbles))
        self._l = D.LazyHost(dev=links) if D.is_device(links) else D.LazyHost(host=np.asarray(links))
        self._f = D.LazyHost(dev=link_faces) if D.is_device(link_faces) else D.LazyHost(host=np.asarray(link_faces))
        self.S_device = S_device
        self._S_host = S_host

    bubbles = property(lambda self: self._b.host)
    links = property(lambda self: self._l.host)
    link_faces = property(lambda self: self._f.host)

    def dev(self):
        t = D.torch()
        return self._b.device(t.int32), self._l.device(t.int32), self._f.device(t.int32)

    @property
    def num_bubbles(self) -> int:
        return int((self._b.dev if self._b.dev is not None else self._b.host).shape[0])


@dataclass
class DirectedBubbleTree:
    tree: BubbleTree
    sources: np.ndarray
    targets: np.ndarray

    @property
    def num_bubbles(self) -> int:
        return self.tree.num_bubbles

    def out_degrees(self) -> np.ndarray:
        out = np.zeros(self.num_bubbles, dtype=np.int64)
        np.add.at(out, self.sources, 1)
        return out


@dataclass
class BubbleAssignment:
    vertex_bubble: np.ndarray
    vertex_converging: np.ndarray


def _S_for(obj, S):
    return D.chained_device(obj, S)


def build_bubble_tree(graph) -> BubbleTree:
    """One bubble per 4-clique of the insertion trace, linked via host faces (dbht.py:64-89)."""
    t = D.torch()
    n = int(graph.n)
    if hasattr(graph, "device"):
        clique = graph.device("initial_clique")
        trace = graph.device("trace")
    else:
        clique = D.to_device(np.asarray(graph.initial_clique, dtype=np.int32), t.int32)
        trace = D.to_device(np.asarray(graph.trace, dtype=np.int32).reshape(-1, 4), t.int32)
    m = n - 3
    bubbles = D.empty((m, 4), t.int32)
    links = D.empty((max(m - 1, 0), 2), t.int32)
    faces = D.empty((max(m - 1, 0), 3), t.int32)
    bad = np.zeros(1, dtype=np.int64)
    ws = D.Workspace.get(N.size("tg_bubble_tree_workspace_bytes", n))
    code = N.load().tg_bubble_tree(N.ptr(clique), N.ptr(trace), n, N.ptr(bubbles), N.ptr(links), N.ptr(faces),
                                   N.c_p(bad.ctypes.data), N.ptr(ws), ws.numel(), N.stream_ptr())
    if code == N.TG_ERR_TRACE:
        row = np.asarray(graph.trace)[int(bad[0])]
        v, x, y, z = (int(q) for q in row)
        raise TraceError(f"trace inserts {v} into non-live face {tuple(sorted((x, y, z)))}")
    N.check("tg_bubble_tree", code)
    return BubbleTree(n=n, bubbles=bubbles, links=links, link_faces=faces,
                      S_device=getattr(graph, "S_device", None), S_host=getattr(graph, "_S_host", None))


def orient_edges(tree: BubbleTree, S) -> DirectedBubbleTree:
    """Direct every link toward the larger apex gain; ties toward the lower index (dbht.py:100-117)."""
    t = D.torch()
    Sd = _S_for(tree, S)
    b, l, f = tree.dev()
    L = int(l.shape[0])
    src = D.empty((max(L, 1),), t.int64)
    dst = D.empty((max(L, 1),), t.int64)
    N.call("tg_orient_edges", N.ptr(Sd), int(Sd.shape[0]), N.ptr(b), N.ptr(l), N.ptr(f), L, N.ptr(src), N.ptr(dst),
           N.stream_ptr())
    d = DirectedBubbleTree(tree=tree, sources=src[:L].cpu().numpy(), targets=dst[:L].cpu().numpy())
    d._dev = (src[:L], dst[:L])
    d._S_device = Sd
    return d


def converging_bubbles(dtree: DirectedBubbleTree) -> list[int]:
    """Bubbles with no outgoing links, ascending (dbht.py:120-122)."""
    return [int(b) for b in np.flatnonzero(dtree.out_degrees() == 0)]


def _dtree_dev(dtree):
    dv = getattr(dtree, "_dev", None)
    if dv is None:
        t = D.torch()
        dv = (D.to_device(np.asarray(dtree.sources, dtype=np.int64), t.int64),
              D.to_device(np.asarray(dtree.targets, dtype=np.int64), t.int64))
        dtree._dev = dv
    return dv


def bubble_sinks_device(dtree: DirectedBubbleTree, Sd):
    t = D.torch()
    b, _, f = dtree.tree.dev()
    src, dst = _dtree_dev(dtree)
    m = dtree.num_bubbles
    sinks = D.empty((m,), t.int64)
    ws = D.Workspace.get(N.size("tg_bubble_sinks_workspace_bytes", m))
    N.call("tg_bubble_sinks", N.ptr(Sd), int(Sd.shape[0]), N.ptr(b), m, N.ptr(f), N.ptr(src), N.ptr(dst),
           int(src.shape[0]), N.ptr(sinks), N.ptr(ws), ws.numel(), N.stream_ptr())
    return sinks


def bubble_sinks(dtree: DirectedBubbleTree, graph) -> np.ndarray:
    """The converging bubble each bubble's outgoing path ends at (dbht.py:143-175).

    Apex gains are read from S (= the graph's edge weights, tmfg.py:137-143).
    """
    Sd = getattr(dtree, "_S_device", None)
    if Sd is None:
        Sd = getattr(graph, "S_device", None)
    if Sd is None:
        raise ValueError("bubble_sinks needs the similarity matrix on the device (orient_edges provides it)")
    return bubble_sinks_device(dtree, Sd).cpu().numpy()


def assign_vertices(graph, dtree: DirectedBubbleTree, oracle) -> BubbleAssignment:
    """Assign each vertex to its closest containing bubble (dbht.py:178-214)."""
    oracle = as_oracle(oracle)
    t = D.torch()
    Sd = getattr(dtree, "_S_device", None)
    if Sd is None:
        Sd = getattr(graph, "S_device", None)
    sinks = bubble_sinks_device(dtree, Sd)
    b, _, _ = dtree.tree.dev()
    m = dtree.num_bubbles
    n = dtree.tree.n
    vb = D.empty((n,), t.int64)
    vc = D.empty((n,), t.int64)
    s = _oracle_struct(oracle)
    ws = D.Workspace.get(N.size("tg_assign_workspace_bytes", n, m))
    N.call("tg_assign_vertices", s, N.ptr(b), m, N.ptr(sinks), N.ptr(vb), N.ptr(vc), N.ptr(ws), ws.numel(),
           N.stream_ptr())
    a = BubbleAssignment(vertex_bubble=vb.cpu().numpy(), vertex_converging=vc.cpu().numpy())
    return a


# ------------------------------------------------------------------ hierarchy
_SUB_DT = np.dtype([("perm_off", "<i8"), ("len", "<i4"), ("m", "<i4"), ("out_off", "<i8"), ("tile_off", "<i8")])
_TILE_DT = np.dtype([("sub", "<i4"), ("i0", "<i4"), ("j0", "<i4")])


def group_layout(subproblems):
    """Host layout of a batched group-max launch (pure numpy).

    subproblems: list of member lists (each a list of int arrays, one per group),
    vertex-disjoint.  Returns (perm int32, gid int32, subs [_SUB_DT], tiles
    [_TILE_DT], out_len): positions of all sub-problems back to back, the group
    index of every position, one descriptor per sub-problem (its tiles are
    row-major, nt x nt of 64 x 64 positions, starting at tile_off) and the size
    of the concatenated m x m outputs.
    """
    perms, gids, subs, tiles = [], [], [], []
    off = out_off = tile_base = 0
    for p, groups in enumerate(subproblems):
        sizes = np.array([len(g) for g in groups], dtype=np.int64)
        perm = np.concatenate([np.asarray(g, dtype=np.int64) for g in groups]).astype(np.int32)
        L, m = perm.shape[0], len(groups)
        starts = np.arange(0, L, 64, dtype=np.int32)
        ii, jj = np.meshgrid(starts, starts, indexing="ij")
        tl = np.empty(ii.size, dtype=_TILE_DT)
        tl["sub"] = p
        tl["i0"] = ii.reshape(-1)
        tl["j0"] = jj.reshape(-1)
        subs.append((off, L, m, out_off, tile_base))
        perms.append(perm)
        gids.append(np.repeat(np.arange(m, dtype=np.int32), sizes))
        tiles.append(tl)
        tile_base += tl.shape[0]
        off += L
        out_off += m * m
    sub_arr = np.array(subs, dtype=_SUB_DT)
    tile_arr = np.concatenate(tiles) if tiles else np.zeros(0, dtype=_TILE_DT)
    return np.concatenate(perms), np.concatenate(gids), sub_arr, tile_arr, out_off


def group_max_batch(oracle, subproblems):
    """dbht.py:217-230 for several vertex-disjoint sub-problems in one launch.

    Returns the concatenated m x m max matrices (flat CUDA tensor) and the
    sub-problem descriptors (``out_off``, ``m`` ...).
    """
    oracle = as_oracle(oracle)
    t = D.torch()
    perm, gid, sub_arr, tile_arr, out_len = group_layout(subproblems)
    perm_d = D.to_device(perm, t.int32)
    gid_d = D.to_device(gid, t.int32)
    sub_d = D.to_device(np.frombuffer(sub_arr.tobytes(), dtype=np.uint8).copy(), t.uint8)
    tile_d = D.to_device(np.frombuffer(tile_arr.tobytes(), dtype=np.uint8).copy(), t.uint8)
    out = D.empty((max(out_len, 1),), t.float64)
    s = _oracle_struct(oracle)
    ws = D.Workspace.get(N.size("tg_group_max_workspace_bytes", oracle.n, int(tile_arr.shape[0]), int(s.H) if s.mode == 1 else 0))
    N.call("tg_group_max_batch", s, N.ptr(perm_d), N.ptr(gid_d), int(perm.shape[0]), N.ptr(sub_d),
           int(sub_arr.shape[0]), N.ptr(tile_d),
           int(tile_arr.shape[0]), N.ptr(out), out_len, N.ptr(ws), ws.numel(), N.stream_ptr())
    return out, sub_arr


def _cluster_max_matrix(oracle, member_lists) -> np.ndarray:
    """Pairwise max oracle distance between vertex groups (dbht.py:217-230)."""
    out, subs = group_max_batch(oracle, [list(member_lists)])
    m = len(member_lists)
    return out[: m * m].reshape(m, m).cpu().numpy()


def _run_linkages(oracle, mats_dev, sizes: np.ndarray, mat_off: np.ndarray, handles_list, records, n):
    """NN-chain every matrix (GPU), canonicalise, append records; returns (roots, rows) per matrix."""
    le, ri, he, moff = nn_chain_raw_batch(mats_dev, sizes, mat_off)
    a, b, h = canonicalize_batch(le, ri, he, moff, sizes)
    roots, rows_all = [], []
    for k, handles in enumerate(handles_list):
        m = int(sizes[k])
        lo, hi = int(moff[k]), int(moff[k + 1])
        local = list(handles)
        rows = []
        root = handles[0]
        for q in range(lo, hi):
            rec = n + len(records)
            records.append((local[int(a[q])], local[int(b[q])], float(h[q])))
            local.append(rec)
            rows.append((rec, float(h[q])))
            root = rec
        assert len(local) == 2 * m - 1
        roots.append(root)
        rows_all.append(rows)
    return roots, rows_all


def build_hierarchy(assignment: BubbleAssignment, dtree: DirectedBubbleTree, oracle,
                    workers: int | None = None) -> Dendrogram:
    """Assemble the full dendrogram in three complete-linkage layers (dbht.py:233-339).

    Native driver (csrc/hierarchy.cu, ``tg_build_hierarchy``): layer-1 oracle
    blocks, layer-2/3 group maxima and every NN-chain run on the GPU; grouping,
    canonicalisation, records and the height-floor emission are C++ host code.
    """
    t = D.torch()
    oracle = as_oracle(oracle)
    # O(n) upload of the caller's current arrays (no stale device copy if they were edited)
    vb = D.to_device(np.asarray(assignment.vertex_bubble, dtype=np.int64), t.int64)
    vc = D.to_device(np.asarray(assignment.vertex_converging, dtype=np.int64), t.int64)
    n = int(vb.shape[0])
    k = max(n - 1, 0)
    lefts = np.empty(max(k, 1), dtype=np.int64)
    rights = np.empty(max(k, 1), dtype=np.int64)
    heights = np.empty(max(k, 1), dtype=np.float64)
    sizes = np.empty(max(k, 1), dtype=np.int64)
    nm = np.zeros(1, dtype=np.int64)
    s = _oracle_struct(oracle)
    hp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    try:
        N.call("tg_build_hierarchy", s, N.ptr(vb), N.ptr(vc), n, hp(lefts), hp(rights), hp(heights), hp(sizes),
               hp(nm), N.stream_ptr())
    except N.NativeError as e:
        if e.code == N.TG_ERR_NOT_REDUCIBLE:
            raise RuntimeError("NN-chain did not terminate: the distance matrix is not reducible "
                               "(the reference's linkage.py:50-94 loop would not terminate either)") from e
        raise
    m = int(nm[0])
    return Dendrogram(n_leaves=n, lefts=lefts[:m].copy(), rights=rights[:m].copy(), heights=heights[:m].copy(),
                      sizes=sizes[:m].copy())
