"""Complete linkage and dendrograms (drop-in for tmfgclust.linkage's hot functions).

Mirrors linkage.py:11-47 (Dendrogram), 50-116 (_nn_chain, nn_chain_merges),
136-148 (dendrogram_from_merges), 151-178 (cut), 181-187
(serialize_dendrogram).  The NN-chain itself runs on the GPU (one warp per
matrix, csrc/dbht.cu) for whole batches of matrices; canonicalisation
(stable height sort + renumbering) is vectorised host bookkeeping.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N


@dataclass
class Dendrogram:
    """Binary merge tree over n_leaves items (linkage.py:11-47)."""

    n_leaves: int
    lefts: np.ndarray
    rights: np.ndarray
    heights: np.ndarray
    sizes: np.ndarray

    @property
    def n_merges(self) -> int:
        return self.lefts.shape[0]

    def validate(self) -> None:
        n = self.n_leaves
        if self.n_merges != n - 1:
            raise ValueError(f"expected {n - 1} merges, found {self.n_merges}")
        if self.n_merges and np.any(np.diff(self.heights) < 0):
            raise ValueError("merge heights must be nondecreasing")
        used = set()
        sizes = {}
        for t in range(self.n_merges):
            for child in (int(self.lefts[t]), int(self.rights[t])):
                if child in used:
                    raise ValueError(f"cluster {child} merged twice")
                if child >= n + t:
                    raise ValueError(f"merge {t} references later cluster {child}")
                used.add(child)
            size = sum(sizes.get(ch, 1) for ch in (int(self.lefts[t]), int(self.rights[t])))
            if size != int(self.sizes[t]):
                raise ValueError(f"merge {t} size {self.sizes[t]} != {size}")
            sizes[n + t] = size


def nn_chain_raw_batch(blocks_dev, sizes: np.ndarray, mat_off: np.ndarray):
    """Raw NN-chain merges for a batch of matrices already in HBM.

    blocks_dev: flat float64 CUDA tensor (overwritten: it is the working copy).
    Returns host arrays (lefts, rights, heights) concatenated per matrix with
    sizes[b]-1 rows each (discovery order, slot cluster ids).
    """
    t = D.torch()
    sizes = np.asarray(sizes, dtype=np.int64)
    count = sizes.shape[0]
    nm = np.maximum(sizes - 1, 0)
    merge_off = np.zeros(count + 1, dtype=np.int64)
    np.cumsum(nm, out=merge_off[1:])
    aux_off = np.zeros(count + 1, dtype=np.int64)
    np.cumsum(sizes, out=aux_off[1:])
    total = int(merge_off[-1])
    if total == 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy(), np.zeros(0), merge_off
    dv = lambda a, dt: D.to_device(np.ascontiguousarray(a), dt)
    mo, sz, mg, ax = dv(mat_off, t.int64), dv(sizes, t.int64), dv(merge_off, t.int64), dv(aux_off, t.int64)
    lefts = D.empty((total,), t.int64)
    rights = D.empty((total,), t.int64)
    heights = D.empty((total,), t.float64)
    naux = int(aux_off[-1])
    active = D.empty((naux,), t.uint8)
    slot = D.empty((naux,), t.int64)
    chain = D.empty((naux + 1,), t.int64)
    N.call("tg_nn_chain_batch", N.ptr(blocks_dev), N.ptr(mo), N.ptr(sz), count, N.ptr(mg), N.ptr(lefts),
           N.ptr(rights), N.ptr(heights), N.ptr(ax), N.ptr(active), N.ptr(slot), N.ptr(chain), N.stream_ptr())
    h = heights.cpu().numpy()
    bad = h.view(np.int64) == np.int64(0x7ff8dead00000000)
    if bad.any():
        raise RuntimeError("NN-chain did not terminate: the distance matrix is not reducible "
                           "(the reference's linkage.py:50-94 loop would not terminate either)")
    return lefts.cpu().numpy(), rights.cpu().numpy(), h, merge_off


def canonicalize_batch(lefts, rights, heights, merge_off, sizes):
    """linkage.py:97-116 for many matrices at once.

    Per matrix: stable sort of the raw merges by height, renumber cluster id
    m+t -> m+rank(t), rows (min, max, h).  Returns the concatenated canonical
    (a, b, h) arrays (same segmentation as the input).
    """
    sizes = np.asarray(sizes, dtype=np.int64)
    total = lefts.shape[0]
    if total == 0:
        return lefts, rights, heights
    count = sizes.shape[0]
    nm = np.diff(merge_off)
    seg = np.repeat(np.arange(count, dtype=np.int64), nm)
    local_t = np.arange(total, dtype=np.int64) - merge_off[seg]
    order = np.lexsort((local_t, heights, seg))            # stable by height inside each matrix
    rank = np.empty(total, dtype=np.int64)
    rank[order] = np.arange(total, dtype=np.int64) - merge_off[seg[order]]
    m_of = sizes[seg]

    def remap(ids):
        ids = ids.copy()
        big = ids >= m_of
        # cluster id m + t refers to raw merge t of the same matrix
        ids[big] = m_of[big] + rank[merge_off[seg[big]] + (ids[big] - m_of[big])]
        return ids

    a = remap(lefts)[order]
    b = remap(rights)[order]
    h = heights[order]
    return np.minimum(a, b), np.maximum(a, b), h


def nn_chain_merges(D_) -> list[tuple[int, int, float]]:
    """Complete-linkage merges of a distance matrix, canonicalized (linkage.py:97-116)."""
    t = D.torch()
    Dm = np.asarray(D_, dtype=np.float64) if not D.is_device(D_) else D_
    m = int(Dm.shape[0])
    if m < 2:
        return []
    blocks = D.to_device(np.ascontiguousarray(Dm).reshape(-1) if not D.is_device(Dm) else Dm.reshape(-1).clone(),
                         t.float64)
    le, ri, he, mo = nn_chain_raw_batch(blocks, np.array([m]), np.array([0], dtype=np.int64))
    a, b, h = canonicalize_batch(le, ri, he, mo, np.array([m]))
    return [(int(x), int(y), float(z)) for x, y, z in zip(a, b, h)]


def dendrogram_from_merges(n_leaves: int, merges) -> Dendrogram:
    """Assemble a Dendrogram from canonical (left, right, height) rows (linkage.py:136-148)."""
    if isinstance(merges, tuple) and len(merges) == 3 and isinstance(merges[0], np.ndarray):
        lefts, rights, heights = (np.asarray(merges[0], dtype=np.int64), np.asarray(merges[1], dtype=np.int64),
                                  np.asarray(merges[2], dtype=np.float64))
    else:
        lefts = np.array([r[0] for r in merges], dtype=np.int64)
        rights = np.array([r[1] for r in merges], dtype=np.int64)
        heights = np.array([r[2] for r in merges], dtype=np.float64)
    k = lefts.shape[0]
    size_of = np.ones(n_leaves + k, dtype=np.int64)
    sizes = np.empty(k, dtype=np.int64)
    for t in range(k):
        s = size_of[lefts[t]] + size_of[rights[t]]
        size_of[n_leaves + t] = s
        sizes[t] = s
    return Dendrogram(n_leaves=n_leaves, lefts=lefts, rights=rights, heights=heights, sizes=sizes)


def cut(dendrogram: Dendrogram, k: int) -> np.ndarray:
    """Flat labels from undoing the last k-1 merges (linkage.py:151-178).

    The reference's union-find, run by the library's C++ side (``tg_cut_labels``, host
    arrays, O(n)); labels 0..k-1 by ascending smallest member id.
    """
    import ctypes

    n = dendrogram.n_leaves
    if not 1 <= k <= n:
        raise ValueError(f"cluster count k={k} out of range 1..{n}")
    kept = n - k
    lefts = np.ascontiguousarray(np.asarray(dendrogram.lefts)[:kept], dtype=np.int64)
    rights = np.ascontiguousarray(np.asarray(dendrogram.rights)[:kept], dtype=np.int64)
    if lefts.shape[0] < kept or rights.shape[0] < kept:
        raise IndexError("dendrogram has fewer merges than n - k")
    labels = np.empty(n, dtype=np.int64)
    scratch = np.empty(2 * (2 * n - 1), dtype=np.int64)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    rc = N.load(require_cuda=False).tg_cut_labels(vp(lefts), vp(rights), n, k, vp(labels), vp(scratch))
    if rc == N.TG_ERR_ARG:
        raise IndexError("dendrogram child id out of range")
    N.check("tg_cut_labels", rc)
    return labels


def serialize_dendrogram(d: Dendrogram) -> str:
    """Text rows "left right height size", one merge per line (linkage.py:181-187).

    Formatted by the library's C++ side (``tg_serialize_dendrogram``: %.17g is
    Python's "{:.17g}"); the dendrogram digest of the pipeline hashes this text.
    """
    import ctypes

    k = int(d.lefts.shape[0])
    if k == 0:
        return ""
    cols = [np.ascontiguousarray(d.lefts, dtype=np.int64), np.ascontiguousarray(d.rights, dtype=np.int64),
            np.ascontiguousarray(d.heights, dtype=np.float64), np.ascontiguousarray(d.sizes, dtype=np.int64)]
    ptrs = [c.ctypes.data_as(ctypes.c_void_p) for c in cols]
    buf = np.empty(80 * k, dtype=np.uint8)   # no zero fill
    need = ctypes.c_size_t(0)
    lib = N.load(require_cuda=False)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    rc = lib.tg_serialize_dendrogram(*ptrs, k, vp(buf), buf.size, ctypes.byref(need))
    if rc == N.TG_ERR_CAPACITY:
        buf = np.empty(need.value, dtype=np.uint8)
        rc = lib.tg_serialize_dendrogram(*ptrs, k, vp(buf), buf.size, ctypes.byref(need))
    N.check("tg_serialize_dendrogram", rc)
    return buf[: need.value].tobytes().decode()


def save_dendrogram(d: Dendrogram, path) -> None:
    """Write the dendrogram text of serialize_dendrogram (linkage.py:190-191)."""
    from pathlib import Path

    Path(path).write_text(serialize_dendrogram(d))


def load_dendrogram(path) -> Dendrogram:
    """Read "left right height size" rows back (linkage.py:194-208); blank lines ignored."""
    from pathlib import Path

    text = Path(path).read_text()
    rows = [ln.split() for ln in text.splitlines() if ln.strip()]
    k = len(rows)
    lefts = np.fromiter((int(r[0]) for r in rows), dtype=np.int64, count=k)
    rights = np.fromiter((int(r[1]) for r in rows), dtype=np.int64, count=k)
    heights = np.fromiter((float(r[2]) for r in rows), dtype=np.float64, count=k)
    sizes = np.fromiter((int(r[3]) for r in rows), dtype=np.int64, count=k)
    return Dendrogram(n_leaves=k + 1, lefts=lefts, rights=rights, heights=heights, sizes=sizes)


def complete_linkage(items, dist) -> Dendrogram:
    """Complete-linkage HAC over ``items`` with a symmetric callable ``dist`` (linkage.py:119-133).

    The pairwise matrix is filled on the host (dist is arbitrary Python); the NN-chain runs
    on the GPU.  Leaves are item positions 0..len(items)-1.
    """
    items = list(items)
    m = len(items)
    if m < 1:
        raise ValueError("need at least one item")
    Dm = np.zeros((m, m))
    iu, ju = np.triu_indices(m, 1)
    for i, j in zip(iu.tolist(), ju.tolist()):
        Dm[i, j] = Dm[j, i] = float(dist(items[i], items[j]))
    return dendrogram_from_merges(m, nn_chain_merges(Dm))
