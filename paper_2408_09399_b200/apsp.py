"""Shortest-path distances over the TMFG on the B200 (drop-in for tmfgclust.apsp).

Mirrors apsp.py:23-49 (WeightedTmfg, ApspParams), 52-77 (to_weighted), 80-158
(ExactOracle, HubOracle), 164-235 (apsp_exact, default_hub_count, select_hubs,
apsp_hub, query).  Distances are computed by label-correcting searches in
csrc/apsp.cu and are bit-identical to the reference's binary-heap Dijkstra.
Oracles keep their tables in HBM; the host arrays the reference exposes
(``matrix``, ``hub_dist``, ``near_*`` ...) are materialised on first access.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N


class _Fields:
    """Host/device pairs with lazy host materialisation."""

    def _init_fields(self, spec: dict, values: dict):
        self._f = {}
        for name, dt in spec.items():
            val = values.get(name)
            if val is None:
                self._f[name] = None
            elif D.is_device(val):
                self._f[name] = D.LazyHost(dev=val, dtype=dt)
            else:
                self._f[name] = D.LazyHost(host=np.asarray(val, dtype=dt))

    def dev(self, name: str, dtype):
        f = self._f[name]
        return None if f is None else f.device(dtype).contiguous()


def _lazy(name):
    def get(self):
        f = self._f[name]
        return None if f is None else f.host

    def set_(self, val):
        self._f[name] = D.LazyHost(dev=val) if D.is_device(val) else D.LazyHost(host=np.asarray(val))

    return property(get, set_)


_W_SPEC = {"indptr": np.int64, "neighbors": np.int64, "lengths": np.float64, "strength": np.float64}


class WeightedTmfg(_Fields):
    """CSR adjacency of a TMFG with lengths sqrt(2(1-s)) (apsp.py:23-35)."""

    def __init__(self, n, indptr, neighbors, lengths, strength):
        self.n = int(n)
        self._init_fields(_W_SPEC, dict(indptr=indptr, neighbors=neighbors, lengths=lengths, strength=strength))

    def device_csr(self):
        t = D.torch()
        return self.dev("indptr", t.int64), self.dev("neighbors", t.int32), self.dev("lengths", t.float64)


for _n in _W_SPEC:
    setattr(WeightedTmfg, _n, _lazy(_n))


@dataclass
class ApspParams:
    """Hub-oracle knobs: hub_count defaults to ceil(sqrt(n)) (apsp.py:38-49)."""

    hub_count: int | None = None
    radius_factor: float = 2.0

    def __post_init__(self):
        if self.hub_count is not None and self.hub_count < 1:
            raise ValueError("hub_count must be >= 1")
        if self.radius_factor <= 0:
            raise ValueError("radius_factor must be positive")


def _oracle_struct(o) -> N.TgOracle:
    t = D.torch()
    s = N.TgOracle()
    s.n = o.n
    if o.mode == "exact":
        s.mode = 0
        s.matrix = N.ptr(o.matrix_device).value
        return s
    s.mode = 1
    hd = o.dev("hub_dist", t.float64)
    s.H = int(hd.shape[0])
    s.hub_dist = N.ptr(hd).value
    s.near_indptr = N.ptr(o.dev("near_indptr", t.int64)).value
    s.near_ids = N.ptr(o.dev("near_ids", t.int32)).value
    s.near_dist = N.ptr(o.dev("near_dist", t.float64)).value
    rip, rid, rdd = o.reverse_tables()
    s.rev_indptr = N.ptr(rip).value
    s.rev_ids = N.ptr(rid).value
    s.rev_dist = N.ptr(rdd).value
    return s


def _oracle_block(o, rows, cols, query_semantics: int) -> np.ndarray:
    t = D.torch()
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    cols = np.asarray(cols, dtype=np.int64).reshape(-1)
    out = D.empty((rows.shape[0], cols.shape[0]), t.float64)
    if rows.size and cols.size:
        rd = D.to_device(rows.astype(np.int32), t.int32)
        cd = D.to_device(cols.astype(np.int32), t.int32)
        s = _oracle_struct(o)
        N.call("tg_oracle_block", s, N.ptr(rd), rows.shape[0], N.ptr(cd), cols.shape[0], query_semantics,
               N.ptr(out), N.stream_ptr())
    return out.cpu().numpy()


class ExactOracle:
    """Full n x n shortest-path distance matrix (apsp.py:80-94), kept in HBM."""

    mode = "exact"

    def __init__(self, matrix):
        self._m = D.LazyHost(dev=matrix) if D.is_device(matrix) else D.LazyHost(host=np.asarray(matrix))
        self.n = int(matrix.shape[0])

    @property
    def matrix(self) -> np.ndarray:
        return self._m.host

    @matrix.setter
    def matrix(self, val):
        self._m = D.LazyHost(dev=val) if D.is_device(val) else D.LazyHost(host=np.asarray(val))

    @property
    def matrix_device(self):
        return self._m.device(D.torch().float64)

    def query(self, u: int, v: int) -> float:
        if self._m._host is not None:
            return float(self._m._host[u, v])
        return float(self._m.dev[int(u), int(v)].item())

    def block(self, rows, cols) -> np.ndarray:
        """Dense distance block for the given vertex index arrays."""
        return _oracle_block(self, rows, cols, 0)


_H_SPEC = {"hubs": np.int64, "hub_dist": np.float64, "nearest_hub": np.int64, "nearest_dist": np.float64,
           "radii": np.float64, "near_indptr": np.int64, "near_ids": np.int64, "near_dist": np.float64}


class HubOracle(_Fields):
    """Hub rows plus per-vertex exact neighbourhoods (apsp.py:97-158).

    query(u, v): recorded exact distance when one endpoint lies in the other's
    truncated-search table (smaller id's table first), else min over hubs.
    block(rows, cols): hub estimate, row tables, then column tables win.
    """

    mode = "hub"

    def __init__(self, hubs, hub_dist, nearest_hub, nearest_dist, radii, near_indptr, near_ids, near_dist):
        self._init_fields(_H_SPEC, dict(hubs=hubs, hub_dist=hub_dist, nearest_hub=nearest_hub,
                                        nearest_dist=nearest_dist, radii=radii, near_indptr=near_indptr,
                                        near_ids=near_ids, near_dist=near_dist))
        self.n = int(nearest_hub.shape[0])
        self._rev = None

    def reverse_tables(self):
        """Transposed near table on the device (cached)."""
        if self._rev is None:
            t = D.torch()
            ip = self.dev("near_indptr", t.int64)
            ids = self.dev("near_ids", t.int32)
            dd = self.dev("near_dist", t.float64)
            E = int(ids.shape[0])
            rip = D.empty((self.n + 1,), t.int64)
            rid = D.empty((max(E, 1),), t.int32)
            rdd = D.empty((max(E, 1),), t.float64)
            ws = D.Workspace.get(N.size("tg_near_transpose_workspace_bytes", self.n, E))
            N.call("tg_near_transpose", self.n, N.ptr(ip), N.ptr(ids), N.ptr(dd), N.ptr(rip), N.ptr(rid),
                   N.ptr(rdd), N.ptr(ws), ws.numel(), N.stream_ptr())
            self._rev = (rip, rid, rdd)
        return self._rev

    def _near_lookup(self, u: int, v: int):
        lo, hi = self.near_indptr[u], self.near_indptr[u + 1]
        ids = self.near_ids[lo:hi]
        k = np.searchsorted(ids, v)
        if k < ids.shape[0] and ids[k] == v:
            return float(self.near_dist[lo + k])
        return None

    def query(self, u: int, v: int) -> float:
        return float(_oracle_block(self, [int(u)], [int(v)], 1)[0, 0])

    def block(self, rows, cols) -> np.ndarray:
        return _oracle_block(self, rows, cols, 0)


for _n in _H_SPEC:
    setattr(HubOracle, _n, _lazy(_n))

DistanceOracle = ExactOracle | HubOracle


def to_weighted_device(Sd, edges_dev, n: int):
    """CSR (indptr i64, nbr i32, len f64) + strength f64 as CUDA tensors."""
    t = D.torch()
    m = int(edges_dev.shape[0])
    indptr = D.empty((n + 1,), t.int64)
    nbr = D.empty((max(2 * m, 1),), t.int32)
    lens = D.empty((max(2 * m, 1),), t.float64)
    strength = D.empty((n,), t.float64)
    ws = D.Workspace.get(N.size("tg_weighted_workspace_bytes", n, m))
    N.call("tg_to_weighted", N.ptr(Sd), n, N.ptr(edges_dev), m, N.ptr(indptr), N.ptr(nbr), N.ptr(lens),
           N.ptr(strength), N.ptr(ws), ws.numel(), N.stream_ptr())
    return indptr, nbr[: 2 * m], lens[: 2 * m], strength


def to_weighted(graph, S) -> WeightedTmfg:
    """Attach lengths sqrt(2(1 - S[i,j])) to every TMFG edge (apsp.py:52-77)."""
    n = int(graph.n)
    Sd = D.chained_device(graph, S)
    t = D.torch()
    if hasattr(graph, "device"):
        edges = graph.device("edges")
    else:
        edges = D.to_device(np.asarray(graph.edges, dtype=np.int32), t.int32)
    indptr, nbr, lens, strength = to_weighted_device(Sd, edges, n)
    return WeightedTmfg(n=n, indptr=indptr, neighbors=nbr, lengths=lens, strength=strength)


def as_weighted(g) -> WeightedTmfg:
    """This package's WeightedTmfg for ``g``: passes ours through, converts a foreign one.

    The reference's own ``WeightedTmfg`` (apsp.py:23-35, host arrays, e.g. built by a
    caller or a test) is accepted wherever the reference accepts it; its CSR is
    uploaded on this call.
    """
    if isinstance(g, WeightedTmfg):
        return g
    return WeightedTmfg(n=g.n, indptr=g.indptr, neighbors=g.neighbors, lengths=g.lengths, strength=g.strength)


def as_oracle(o):
    """This package's ExactOracle / HubOracle for ``o`` (a foreign reference oracle is converted).

    The caller keeps the returned object alive while raw device pointers from it are in use.
    """
    if isinstance(o, (ExactOracle, HubOracle)):
        return o
    if getattr(o, "mode", None) == "exact":
        return ExactOracle(np.asarray(o.matrix, dtype=np.float64))
    if getattr(o, "mode", None) == "hub":
        return HubOracle(hubs=o.hubs, hub_dist=o.hub_dist, nearest_hub=o.nearest_hub, nearest_dist=o.nearest_dist,
                         radii=o.radii, near_indptr=o.near_indptr, near_ids=o.near_ids, near_dist=o.near_dist)
    raise TypeError(f"not a distance oracle: {type(o).__name__}")


def sssp_rows_device(w: WeightedTmfg, sources_dev):
    t = D.torch()
    ip, nb, ln = w.device_csr()
    ns = int(sources_dev.shape[0])
    out = D.empty((ns, w.n), t.float64)
    ws = D.Workspace.get(N.size("tg_sssp_workspace_bytes", w.n, ns))
    N.call("tg_sssp_rows", N.ptr(ip), N.ptr(nb), N.ptr(ln), w.n, N.ptr(sources_dev), ns, N.ptr(out), N.ptr(ws),
           ws.numel(), N.stream_ptr())
    return out


def apsp_exact(g: WeightedTmfg, workers: int | None = None) -> ExactOracle:
    """One search per vertex (apsp.py:164-171); ``workers`` is ignored."""
    g = as_weighted(g)
    t = D.torch()
    src = t.arange(g.n, dtype=t.int64, device="cuda")
    return ExactOracle(sssp_rows_device(g, src))


def default_hub_count(n: int) -> int:
    return min(n, math.ceil(math.sqrt(n)))


def select_hubs_device(g: WeightedTmfg, hub_count: int):
    t = D.torch()
    strength = g.dev("strength", t.float64)
    hubs = D.empty((hub_count,), t.int64)
    ws = D.Workspace.get(N.size("tg_select_hubs_workspace_bytes", g.n))
    N.call("tg_select_hubs", N.ptr(strength), g.n, hub_count, N.ptr(hubs), N.ptr(ws), ws.numel(), N.stream_ptr())
    return hubs


def select_hubs(g: WeightedTmfg, hub_count: int) -> np.ndarray:
    """The hub_count vertices of highest strength, (strength desc, id asc) (apsp.py:178-186)."""
    g = as_weighted(g)
    return select_hubs_device(g, hub_count).cpu().numpy().astype(np.int64)


def apsp_hub(g: WeightedTmfg, params: ApspParams | None = None, workers: int | None = None) -> HubOracle:
    """Hub rows, nearest-hub radii and per-vertex truncated searches (apsp.py:189-230)."""
    g = as_weighted(g)
    params = params or ApspParams()
    hub_count = params.hub_count or default_hub_count(g.n)
    if hub_count > g.n:
        raise ValueError(f"hub_count {hub_count} exceeds vertex count {g.n}")
    t = D.torch()
    n = g.n
    hubs = select_hubs_device(g, hub_count)
    hub_dist = sssp_rows_device(g, hubs)
    nh = D.empty((n,), t.int64)
    nd = D.empty((n,), t.float64)
    radii = D.empty((n,), t.float64)
    N.call("tg_nearest_hub", N.ptr(hub_dist), N.ptr(hubs), hub_count, n, float(params.radius_factor), N.ptr(nh),
           N.ptr(nd), N.ptr(radii), N.stream_ptr())
    ip, nb, ln = g.device_csr()
    near_indptr = D.empty((n + 1,), t.int64)
    cap = _truncated_capacity_guess(n)
    total = np.zeros(1, dtype=np.int64)
    for _ in range(2):
        ids = D.empty((max(cap, 1),), t.int32)
        dd = D.empty((max(cap, 1),), t.float64)
        ws = D.Workspace.get(N.size("tg_truncated_workspace_bytes", n) + 12 * cap + 4096)
        lib = N.load()
        code = lib.tg_truncated(N.ptr(ip), N.ptr(nb), N.ptr(ln), n, N.ptr(radii), cap, N.ptr(near_indptr),
                                N.ptr(ids), N.ptr(dd), N.c_p(total.ctypes.data),
                                N.ptr(ws), ws.numel(), N.stream_ptr())
        if code == N.TG_ERR_CAPACITY:
            cap = int(total[0])
            _CAP_HINT[n] = cap
            continue
        N.check("tg_truncated", code)
        break
    E = int(total[0])
    return HubOracle(hubs=hubs, hub_dist=hub_dist, nearest_hub=nh, nearest_dist=nd, radii=radii,
                     near_indptr=near_indptr, near_ids=ids[:E], near_dist=dd[:E])


_CAP_HINT: dict = {}


def _truncated_capacity_guess(n: int) -> int:
    if n in _CAP_HINT:
        return _CAP_HINT[n]
    return int(max(4096, 48 * n * max(1.0, math.log2(max(n, 2)) / 4)))


def query(oracle, u: int, v: int) -> float:
    """Distance between u and v through the given oracle (apsp.py:233-235)."""
    return oracle.query(int(u), int(v))
