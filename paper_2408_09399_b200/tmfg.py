"""TMFG construction on the B200 (drop-in for the heap builder of tmfgclust.tmfg).

Mirrors tmfg.py:34-68 (BuildConfig, TmfgGraph, TraceError), 71-91 (clique,
gain, edge_sum), 208-341 (build_tmfg_exact, build_tmfg_corr) and 344-451
(build_tmfg_heap, build_tmfg).  The heap insertion loop runs as one persistent
CTA cluster (csrc/tmfg.cu), the exact / corr builders as one persistent CTA
(csrc/tmfg_variants.cu); S and the sorted rows never leave HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .simmatrix import DataError, SortedNeighborLists, sort_rows_device, validate_device

GAIN_EPS = 1e-12


@dataclass
class BuildConfig:
    """Builder selection: variant in {exact, corr, heap}, prefix_size >= 1 (tmfg.py:34-45)."""

    variant: str = "heap"
    prefix_size: int = 1

    def __post_init__(self):
        if self.variant not in ("exact", "corr", "heap"):
            raise ValueError(f"unknown TMFG variant {self.variant!r}")
        if self.prefix_size < 1:
            raise ValueError(f"prefix_size must be >= 1, got {self.prefix_size}")


class TraceError(ValueError):
    """An insertion trace references a face that was never live (tmfg.py:67-68)."""


_HOST_FIELDS = {"edges": np.int32, "weights": np.float64, "initial_clique": np.int32, "trace": np.int32,
                "faces": np.int32}


class TmfgGraph:
    """A built TMFG (tmfg.py:48-64): edge list, weights, clique, trace, faces.

    Fields accept host arrays or CUDA tensors; host views are materialised on
    first access, device views (``device(name)``) are reused by later stages.
    ``host_fid`` (the face id each trace row subdivided) is kept on the device.
    """

    def __init__(self, n, edges, weights, initial_clique, trace, faces, variant: str = "",
                 debug_stats: dict | None = None, host_fid=None, S_device=None):
        self.n = int(n)
        self._f = {}
        for name, val in (("edges", edges), ("weights", weights), ("initial_clique", initial_clique),
                          ("trace", trace), ("faces", faces)):
            self._set(name, val)
        self.variant = variant
        self.debug_stats = debug_stats
        self.host_fid = host_fid
        self.S_device = S_device

    def _set(self, name, val):
        dt = _HOST_FIELDS[name]
        if D.is_device(val):
            self._f[name] = D.LazyHost(dev=val, dtype=dt)
        else:
            self._f[name] = D.LazyHost(host=np.asarray(val, dtype=dt))

    def device(self, name: str):
        t = D.torch()
        dt = {np.int32: t.int32, np.float64: t.float64}[_HOST_FIELDS[name]]
        return self._f[name].device(dt).contiguous()

    def __repr__(self) -> str:
        return f"TmfgGraph(n={self.n}, variant={self.variant!r})"


def _make_prop(name):
    def get(self):
        return self._f[name].host

    def set_(self, val):
        self._set(name, val)

    return property(get, set_)


for _name in _HOST_FIELDS:
    setattr(TmfgGraph, _name, _make_prop(_name))


def row_sums_device(Sd):
    """tmfg.py:76 ``S.sum(axis=1) - diag(S)`` in numpy's pairwise order, on device."""
    t = D.torch()
    n = int(Sd.shape[0])
    rowsum = D.empty((n,), t.float64)
    ws = D.Workspace.get(N.size("tg_row_sums_workspace_bytes", n))
    N.call("tg_row_sums_f64", N.ptr(Sd), n, N.ptr(rowsum), N.ptr(ws), ws.numel(), N.stream_ptr())
    return rowsum


def initial_clique_device(Sd, screen=None):
    """tmfg.py:71-79 on device: int32[4] CUDA tensor (ascending).

    With the row sort's ``screen`` only the rows that can reach the top 4 get an
    exact pairwise sum; without it every row does.
    """
    t = D.torch()
    n = int(Sd.shape[0])
    clique = D.empty((4,), t.int32)
    if screen is not None:
        ws = D.Workspace.get(N.size("tg_initial_clique_screened_workspace_bytes", n))
        N.call("tg_initial_clique_screened", N.ptr(Sd), n, N.ptr(screen), N.ptr(clique), N.ptr(ws), ws.numel(),
               N.stream_ptr())
        return clique
    rowsum = row_sums_device(Sd)
    N.call("tg_initial_clique", N.ptr(rowsum), n, N.ptr(clique), N.stream_ptr())
    return clique


def select_initial_clique(S) -> tuple[int, int, int, int]:
    """The 4 vertices with the largest off-diagonal row sums, id-ascending (tmfg.py:71-79)."""
    Sd = D.device_matrix(S)
    c = initial_clique_device(Sd).cpu().numpy()
    return tuple(int(v) for v in c)


def gain(face, v: int, S) -> float:
    """Sum of similarities from v to the three face vertices (tmfg.py:82-85)."""
    a, b, c = sorted(int(x) for x in face)
    if D.is_device(S):
        vals = S[[a, b, c], v].cpu().numpy()
        return float(vals[0] + vals[1] + vals[2])
    return float(S[a, v] + S[b, v] + S[c, v])


def edge_sum(graph: TmfgGraph, S) -> float:
    """Total similarity over the graph's 3n-6 edges (tmfg.py:88-91)."""
    e = graph.edges
    if D.is_device(S):
        w = graph.weights
        return float(np.add.reduce(w))
    return float(S[e[:, 0], e[:, 1]].sum())


def edge_weights_device(Sd, edges_dev):
    t = D.torch()
    m = int(edges_dev.shape[0])
    w = D.empty((m,), t.float64)
    N.call("tg_edge_weights", N.ptr(Sd), int(Sd.shape[0]), N.ptr(edges_dev), m, N.ptr(w), N.stream_ptr())
    return w


def build_tmfg_heap_device(Sd, order_dev, clique_dev, check_invariants: bool = False):
    """Run the persistent heap-insertion kernel; returns device tensors + stats."""
    t = D.torch()
    n = int(Sd.shape[0])
    trace = D.empty((max(n - 4, 0), 4), t.int32)
    host_fid = D.empty((max(n - 4, 0),), t.int32)
    edges = D.empty((3 * n - 6, 2), t.int32)
    faces = D.empty((2 * n - 4, 3), t.int32)
    stats = D.empty((32,), t.int64)
    ws = D.Workspace.get(N.size("tg_tmfg_workspace_bytes", n))
    N.call("tg_tmfg_heap", N.ptr(Sd), N.ptr(order_dev), n, N.ptr(clique_dev), N.ptr(trace), N.ptr(host_fid),
           N.ptr(edges), N.ptr(faces), N.ptr(stats), 1 if check_invariants else 0, N.ptr(ws), ws.numel(),
           N.stream_ptr())
    return dict(trace=trace, host_fid=host_fid, edges=edges, faces=faces, stats=stats)


def _stats_dict(st: np.ndarray, check: bool):
    if int(st[3]) == 2:
        fid = int(st[4])
        g_old = float(np.array([st[5]], dtype=np.int64).view(np.float64)[0])
        g_new = float(np.array([st[6]], dtype=np.int64).view(np.float64)[0])
        raise AssertionError(f"face {fid}: gain rose from {g_old} to {g_new} "
                             "after a refresh of a previously optimal pair")
    if int(st[3]) != 0:
        raise RuntimeError(f"TMFG kernel reported internal status {int(st[3])}")
    if not check:
        return None
    return {"pops": int(st[0]), "refreshes": int(st[1]), "gain_increases": int(st[2])}


def build_tmfg_heap(S, lists: SortedNeighborLists | None = None, config: BuildConfig | None = None,
                    check_invariants: bool = False) -> TmfgGraph:
    """Heap-based builder with lazy refresh (tmfg.py:344-436), on the B200.

    Bit-identical trace / edges / faces / debug_stats to the reference.  With
    ``check_invariants`` the kernel also runs the reference's brute-force
    optimality test and raises the same AssertionError when it fires.
    """
    config = config or BuildConfig(variant="heap")
    shape = tuple(S.shape)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise DataError(f"similarity matrix must be square, got shape {shape}")
    if not D.is_device(S):
        S = np.asarray(S, dtype=np.float64)
    Sd = D.chained_device(lists, S)
    validate_device(Sd)
    n = shape[0]
    # the sort's fused row-sum screen is only valid for the very device S it was computed on
    screen = getattr(lists, "screen_device", None) if getattr(lists, "S_device", None) is Sd else None
    if lists is None:
        order_dev, screen = sort_rows_device(Sd, with_screen=True)
    elif isinstance(lists, SortedNeighborLists):
        order_dev = lists.order_device
    else:
        order_dev = D.to_device(np.asarray(lists.order, dtype=np.int32), D.torch().int32)
    clique = initial_clique_device(Sd, screen)
    out = build_tmfg_heap_device(Sd, order_dev, clique, check_invariants)
    raw = out["stats"].cpu().numpy()
    stats = _stats_dict(raw, check_invariants)
    weights = edge_weights_device(Sd, out["edges"])
    g = TmfgGraph(n=n, edges=out["edges"], weights=weights, initial_clique=clique, trace=out["trace"],
                  faces=out["faces"], variant="heap", debug_stats=stats, host_fid=out["host_fid"],
                  S_device=Sd)
    g._S_host = S
    g._raw_stats = {"pops": int(raw[0]), "refreshes": int(raw[1]), "gain_increases": int(raw[2])}
    g._kernel_profile = {k: int(raw[i]) for i, k in enumerate(
        ["rounds", "refills", "cyc_warp_max", "cyc_probe_max", "cyc_tail_max", "cyc_S_max", "cyc_refill", "pool",
         "cyc_parallel", "cyc_replay", "cyc_merge", "cyc_insert", "cyc_round_tail"], 8)}
    return g


def _variant_device(variant: str, Sd, order_dev, clique_dev, prefix: int):
    """tg_tmfg_exact / tg_tmfg_corr: device trace, edges, faces."""
    t = D.torch()
    n = int(Sd.shape[0])
    trace = D.empty((max(n - 4, 0), 4), t.int32)
    edges = D.empty((3 * n - 6, 2), t.int32)
    faces = D.empty((2 * n - 4, 3), t.int32)
    ws = D.Workspace.get(N.size("tg_tmfg_variant_workspace_bytes", n))
    if variant == "exact":
        N.call("tg_tmfg_exact", N.ptr(Sd), n, N.ptr(clique_dev), int(prefix), N.ptr(trace), N.ptr(edges),
               N.ptr(faces), N.ptr(ws), ws.numel(), N.stream_ptr())
    else:
        N.call("tg_tmfg_corr", N.ptr(Sd), N.ptr(order_dev), n, N.ptr(clique_dev), int(prefix), N.ptr(trace),
               N.ptr(edges), N.ptr(faces), N.ptr(ws), ws.numel(), N.stream_ptr())
    return trace, edges, faces


def _variant_graph(variant: str, S, Sd, order_dev, prefix: int) -> TmfgGraph:
    n = int(Sd.shape[0])
    clique = initial_clique_device(Sd)
    trace, edges, faces = _variant_device(variant, Sd, order_dev, clique, prefix)
    g = TmfgGraph(n=n, edges=edges, weights=edge_weights_device(Sd, edges), initial_clique=clique, trace=trace,
                  faces=faces, variant=variant, S_device=Sd)
    g._S_host = S
    return g


def build_tmfg_exact(S, config: BuildConfig | None = None) -> TmfgGraph:
    """Prefix-based baseline: every live face tracks its true best vertex (tmfg.py:208-263), on the B200.

    Bit-identical trace / edges / faces to the reference for every prefix_size.
    """
    config = config or BuildConfig(variant="exact")
    shape = tuple(S.shape)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise DataError(f"similarity matrix must be square, got shape {shape}")
    if not D.is_device(S):
        S = np.asarray(S, dtype=np.float64)
    Sd = D.device_matrix(S)
    validate_device(Sd)
    return _variant_graph("exact", S, Sd, None, config.prefix_size)


def build_tmfg_corr(S, lists: SortedNeighborLists, config: BuildConfig | None = None) -> TmfgGraph:
    """Correlation-based builder with eager per-round refresh (tmfg.py:280-341), on the B200."""
    config = config or BuildConfig(variant="corr")
    shape = tuple(S.shape)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise DataError(f"similarity matrix must be square, got shape {shape}")
    if not D.is_device(S):
        S = np.asarray(S, dtype=np.float64)
    Sd = D.chained_device(lists, S)
    validate_device(Sd)
    if isinstance(lists, SortedNeighborLists):
        order_dev = lists.order_device
    else:
        order_dev = D.to_device(np.asarray(lists.order, dtype=np.int32), D.torch().int32)
    return _variant_graph("corr", S, Sd, order_dev, config.prefix_size)


def build_tmfg(S, lists: SortedNeighborLists | None, config: BuildConfig) -> TmfgGraph:
    """Dispatch to the configured builder; the exact variant ignores lists (tmfg.py:439-451)."""
    if config.variant == "exact":
        return build_tmfg_exact(S, config)
    if lists is None:
        raise ValueError(f"the {config.variant} builder needs sorted neighbor lists")
    if config.variant == "corr":
        return build_tmfg_corr(S, lists, config)
    return build_tmfg_heap(S, lists, config)


# ------------------------------------------------------------------ trace replay and on-disk format (tmfg.py:454-516)
def replay_trace(graph) -> tuple[set, set]:
    """Re-run the insertion trace: (edge set, final live-face set); TraceError on a non-live host face."""
    clique = [int(x) for x in np.asarray(graph.initial_clique)]
    a, b, c, d = clique
    edges = {(a, b), (a, c), (a, d), (b, c), (b, d), (c, d)}
    live = {(a, b, c), (a, b, d), (a, c, d), (b, c, d)}
    for row in np.asarray(graph.trace).reshape(-1, 4).tolist():
        v, x, y, z = row
        host = tuple(sorted((x, y, z)))
        if host not in live:
            raise TraceError(f"trace inserts {v} into non-live face {host}")
        live.discard(host)
        edges.update((min(q, v), max(q, v)) for q in host)
        live.update(tuple(sorted(t)) for t in ((v, x, y), (v, x, z), (v, y, z)))
    return edges, live


def save_tmfg(graph, edges_path, trace_path) -> None:
    """Edge list ("i j weight", weight as %.17g) and trace file (clique line, then "v a b c" lines)."""
    e = np.asarray(graph.edges).reshape(-1, 2)
    w = np.asarray(graph.weights, dtype=np.float64)
    with open(edges_path, "w") as fh:
        fh.writelines(f"{int(i)} {int(j)} {x:.17g}\n" for (i, j), x in zip(e.tolist(), w.tolist()))
    with open(trace_path, "w") as fh:
        fh.write(" ".join(str(int(v)) for v in np.asarray(graph.initial_clique)) + "\n")
        fh.writelines(" ".join(str(v) for v in row) + "\n" for row in np.asarray(graph.trace).reshape(-1, 4).tolist())


def load_tmfg(edges_path, trace_path) -> TmfgGraph:
    """Rebuild a TmfgGraph from the two files; faces are the replayed live faces, sorted."""
    from pathlib import Path

    erows = [ln.split() for ln in Path(edges_path).read_text().splitlines() if ln.strip()]
    tlines = [ln for ln in Path(trace_path).read_text().splitlines() if ln.strip()]
    clique = np.array([int(x) for x in tlines[0].split()], dtype=np.int32)
    trace = np.array([[int(x) for x in ln.split()] for ln in tlines[1:]], dtype=np.int32).reshape(-1, 4)
    g = TmfgGraph(n=4 + trace.shape[0],
                  edges=np.array([[int(r[0]), int(r[1])] for r in erows], dtype=np.int32).reshape(-1, 2),
                  weights=np.array([float(r[2]) for r in erows], dtype=np.float64),
                  initial_clique=clique, trace=trace, faces=np.zeros((0, 3), dtype=np.int32))
    _, live = replay_trace(g)
    g.faces = np.array(sorted(live), dtype=np.int32).reshape(-1, 3)
    return g


class TmfgState:
    """Scan state of the list-based builders (tmfg.py:147-166): inserted flags, per-vertex
    cursors into the sorted neighbour lists, cached best uninserted neighbours.

    A host-side inspection object with the reference's fields (its tests drive it
    directly); the GPU builders keep the same state in device memory.
    """

    def __init__(self, S, lists):
        self.S = S
        self.n = int(S.shape[0])
        self.order = lists.order
        self.cursors = [0] * self.n
        self.inserted = bytearray(self.n)
        self.max_corrs = [-1] * self.n
        self.rem_count = self.n

    def mark_inserted(self, v: int) -> None:
        self.inserted[v] = 1
        self.rem_count -= 1


def refresh_max_corr(state: TmfgState, v: int) -> int:
    """Advance v's cursor past inserted ids; cache and return the first uninserted one (tmfg.py:169-182)."""
    row = state.order[v]
    ins = state.inserted
    cur = state.cursors[v]
    while ins[int(row[cur])]:
        cur += 1
    state.cursors[v] = cur
    state.max_corrs[v] = int(row[cur])
    return state.max_corrs[v]
