"""Similarity matrices and sorted neighbour lists on the B200.

Drop-in for the reference's ``tmfgclust.simmatrix`` hot functions
(simmatrix.py:105-123 pearson_similarity, 126-139 validate_similarity,
205-249 SortedNeighborLists / sort_neighbor_lists): same names, arguments,
return types and exceptions.  The work runs in libtmfg_b200.so; host arrays are
copied to HBM once and results stay device-resident, with host views
materialised lazily on first access.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N


class DataError(ValueError):
    """Raised for malformed input files or invalid matrices (simmatrix.py:18-19)."""


@dataclass
class Dataset:
    """Labeled collection of equal-length series (simmatrix.py:22-54)."""

    labels: np.ndarray
    series: np.ndarray

    def __post_init__(self):
        self.labels = np.asarray(self.labels, dtype=np.int64)
        if not D.is_device(self.series):
            self.series = np.asarray(self.series, dtype=np.float64)
        if self.series.ndim != 2:
            raise DataError("series must be a 2-d array")
        if self.n < 4:
            raise DataError(f"dataset too small: need at least 4 objects, got {self.n}")
        if self.length < 2:
            raise DataError(f"series too short: need length >= 2, got {self.length}")
        if self.labels.shape[0] != self.n:
            raise DataError("labels and series row counts differ")

    @property
    def n(self) -> int:
        return int(self.series.shape[0])

    @property
    def length(self) -> int:
        return int(self.series.shape[1])

    @property
    def num_classes(self) -> int:
        return int(self.labels.max()) + 1 if self.labels.size else 0


def pearson_similarity_device(X, out=None):
    """(n, L) series (host or device) -> (n, n) float64 CUDA tensor S (``out`` if given)."""
    t = D.torch()
    Xd = D.to_device(X, t.float64)
    n, L = (int(s) for s in Xd.shape)
    S = out if out is not None else D.empty((n, n), t.float64)
    ws = D.Workspace.get(N.size("tg_pearson_workspace_bytes", n, L))
    N.call("tg_pearson_f64", N.ptr(Xd), n, L, N.ptr(S), N.ptr(ws), ws.numel(), N.stream_ptr())
    return S


def pearson_similarity_refexact_device(x):
    """(n, L) host series -> the reference's exact S as a CUDA tensor.

    The numpy prologue is the reference's own (simmatrix.py:113-118: mean,
    einsum norm, guarded reciprocal), the O(n^2 L) kernel runs on the GPU in the
    reference's arithmetic order (``tg_pearson_refexact_f64``), so S is
    bit-identical to ``tmfgclust.simmatrix.pearson_similarity`` -- the input the
    bit-exactness contract is stated on.  ``pearson_similarity_device`` (DMMA)
    is the fast path, within 1e-12.
    """
    t = D.torch()
    x = np.asarray(x, dtype=np.float64)
    xc = x - x.mean(axis=1, keepdims=True)
    norm = np.sqrt(np.einsum("ij,ij->i", xc, xc))
    inv = np.zeros_like(norm)
    nz = norm > 0.0
    inv[nz] = 1.0 / norm[nz]
    n, L = xc.shape
    xcd = D.to_device(np.ascontiguousarray(xc), t.float64)
    invd = D.to_device(inv, t.float64)
    S = D.empty((n, n), t.float64)
    N.call("tg_pearson_refexact_f64", N.ptr(xcd), N.ptr(invd), n, L, N.ptr(S), N.stream_ptr())
    return S


def pearson_similarity(data: Dataset, workers: int | None = None):
    """Dense Pearson correlation matrix of the dataset's rows (simmatrix.py:105-123).

    Returns a host ndarray like the reference; when ``data.series`` is a CUDA
    tensor the result stays on the device (a torch tensor).
    ``workers`` is accepted for signature compatibility and ignored.
    """
    S = pearson_similarity_device(data.series)
    if D.is_device(data.series):
        return S
    return S.cpu().numpy()


_FLAG_MESSAGES = (
    (N.TG_BAD_NAN, "similarity matrix contains NaN"),
    (N.TG_BAD_ASYM, "similarity matrix is not symmetric"),
    (N.TG_BAD_DIAG, "similarity matrix diagonal must be exactly 1"),
    (N.TG_BAD_RANGE, "similarity values must lie in [-1, 1]"),
)


def validate_device(Sd) -> None:
    """Run the on-device checks of simmatrix.py:126-139; raise DataError."""
    t = D.torch()
    n = int(Sd.shape[0])
    flags = D.empty((1,), t.int32)
    N.call("tg_validate_f64", N.ptr(Sd), n, N.ptr(flags), N.stream_ptr())
    f = int(flags.item())
    for bit, msg in _FLAG_MESSAGES:
        if f & bit:
            raise DataError(msg)


def validate_similarity(S):
    """Check SimilarityMatrix invariants; returns the validated float64 matrix."""
    shape = tuple(S.shape)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise DataError(f"similarity matrix must be square, got shape {shape}")
    if not D.is_device(S):
        S = np.asarray(S, dtype=np.float64)
    validate_device(D.device_matrix(S))
    return S


class SortedNeighborLists:
    """Per-vertex neighbour ids by (similarity desc, id asc) (simmatrix.py:205-222).

    ``order`` is the (n, n-1) int32 table; on this backend it lives in HBM
    (``order_device``) and the host copy is made on first access.
    """

    def __init__(self, S, order, S_device=None, screen_device=None):
        self.S = S
        self._order = D.LazyHost(dev=order) if D.is_device(order) else D.LazyHost(host=np.asarray(order))
        self.S_device = S_device
        self.screen_device = screen_device   # initial-clique row-sum screen (2n), see sort_rows_device

    @property
    def order(self) -> np.ndarray:
        return self._order.host

    @order.setter
    def order(self, value):
        self._order = D.LazyHost(dev=value) if D.is_device(value) else D.LazyHost(host=np.asarray(value))

    @property
    def order_device(self):
        t = D.torch()
        return self._order.device(t.int32)

    @property
    def n(self) -> int:
        return int(self._order.dev.shape[0] if self._order.dev is not None else self._order.host.shape[0])

    def pairs(self, v: int) -> list[tuple[float, int]]:
        """The (similarity, neighbor) list for vertex v, best first."""
        S = self.S if not D.is_device(self.S) else self.S[v].cpu().numpy()[None, :]
        row = S[v] if not D.is_device(self.S) else S[0]
        return [(float(row[u]), int(u)) for u in self.order[v]]


def sort_rows_device(Sd, with_screen: bool = True, out=None):
    """(order (n, n-1) int32, screen (2n,) float64 or None) as CUDA tensors (``order`` = out if given).

    ``screen[v]`` is row v's off-diagonal sum in the kernel's summation order and
    ``screen[n + v]`` a rigorous bound on its distance to numpy's pairwise sum
    (tmfg.py:76); ``initial_clique_device`` turns it into the exact clique.
    """
    t = D.torch()
    n = int(Sd.shape[0])
    order = out if out is not None else D.empty((n, max(n - 1, 0)), t.int32)
    screen = D.empty((2 * n,), t.float64) if (with_screen and n >= 2) else None
    if n >= 2:
        ws = D.Workspace.get(N.size("tg_row_sort_workspace_bytes", n))
        N.call("tg_row_sort_f64", N.ptr(Sd), n, N.ptr(order), N.ptr(screen), N.ptr(ws), ws.numel(),
               N.stream_ptr())
    return order, screen


def sort_neighbor_lists(S, workers: int | None = None) -> SortedNeighborLists:
    """Sort every vertex's neighbours by (similarity desc, id asc) (simmatrix.py:225-249).

    One fused pass also produces the initial-clique row sums, kept on the
    device for build_tmfg.  ``workers`` is accepted and ignored.
    """
    if not D.is_device(S):
        S = np.asarray(S, dtype=np.float64)
    Sd = D.device_matrix(S)
    order, screen = sort_rows_device(Sd, with_screen=True)
    return SortedNeighborLists(S, order, S_device=Sd, screen_device=screen)


# ------------------------------------------------------------------ on-disk formats (simmatrix.py:55-202)
SYMMETRY_TOL = 1e-9


def _label_codes(raw: list) -> np.ndarray:
    """Map a label alphabet onto 0..k-1: numeric-looking alphabets numerically, else lexicographically."""
    alphabet = sorted(set(raw))
    try:
        alphabet.sort(key=float)
    except ValueError:
        pass
    code = {lab: i for i, lab in enumerate(alphabet)}
    return np.fromiter((code[lab] for lab in raw), dtype=np.int64, count=len(raw))


def load_ucr_dataset(path) -> Dataset:
    """UCR-style text: a label then L values per line, tab / comma (or space) separated (simmatrix.py:72-102)."""
    import re
    from pathlib import Path

    sep = re.compile(r"[\t, ]+")
    labels: list = []
    rows: list = []
    width = None
    path = Path(path)
    with path.open() as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            fields = [f for f in sep.split(line) if f]
            if len(fields) < 3:
                raise DataError(f"{path}:{lineno}: expected a label and at least 2 values")
            if width is None:
                width = len(fields)
            elif len(fields) != width:
                raise DataError(f"{path}:{lineno}: ragged row, expected {width} fields, got {len(fields)}")
            try:
                vals = [float(f) for f in fields[1:]]
            except ValueError as exc:
                raise DataError(f"{path}:{lineno}: non-numeric value") from exc
            if any(v != v for v in vals):
                raise DataError(f"{path}:{lineno}: NaN value in series")
            labels.append(fields[0])
            rows.append(vals)
    if len(rows) < 4:
        raise DataError(f"dataset too small: need at least 4 objects, got {len(rows)}")
    return Dataset(labels=_label_codes(labels), series=np.array(rows, dtype=np.float64))


def write_matrix_binary(path, M) -> None:
    """Square matrix as 8-byte little-endian n, then n*n row-major little-endian float64."""
    if D.is_device(M):
        M = M.cpu().numpy()
    M = np.ascontiguousarray(M, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(np.uint64(M.shape[0]).astype("<u8").tobytes())
        fh.write(memoryview(M).cast("B"))


def read_matrix_binary(path) -> np.ndarray:
    """Inverse of write_matrix_binary; DataError on a truncated or mis-sized file."""
    from pathlib import Path

    raw = Path(path).read_bytes()
    if len(raw) < 8:
        raise DataError(f"{path}: truncated binary matrix")
    n = int(np.frombuffer(raw, dtype="<u8", count=1)[0])
    want = 8 + 8 * n * n
    if len(raw) != want:
        raise DataError(f"{path}: size mismatch, expected {want} bytes for n={n}")
    return np.frombuffer(raw, dtype="<f8", offset=8).reshape(n, n).astype(np.float64)


def save_matrix(path, S) -> None:
    """Validate (on the device) and persist a similarity matrix in the binary format."""
    write_matrix_binary(path, validate_similarity(S))


def _is_binary_matrix(path) -> bool:
    import os

    size = os.path.getsize(path)
    if size < 8:
        return False
    with open(path, "rb") as fh:
        n = int(np.frombuffer(fh.read(8), dtype="<u8")[0])
    return n > 0 and size == 8 + 8 * n * n


def load_matrix(path) -> np.ndarray:
    """Binary or text similarity matrix (simmatrix.py:173-202).

    Asymmetry or a diagonal off 1 by more than SYMMETRY_TOL is a DataError; smaller
    deviations are symmetrised exactly ((S + S.T) / 2, unit diagonal).
    """
    if _is_binary_matrix(path):
        S = read_matrix_binary(path)
    else:
        try:
            S = np.loadtxt(path, delimiter=None)
        except ValueError:
            S = np.loadtxt(path, delimiter=",")
        S = np.atleast_2d(np.asarray(S, dtype=np.float64))
    if S.ndim != 2 or S.shape[0] != S.shape[1]:
        raise DataError(f"{path}: matrix must be square, got shape {S.shape}")
    if np.isnan(S).any():
        raise DataError(f"{path}: matrix contains NaN")
    asym = float(np.abs(S - S.T).max())
    if asym > SYMMETRY_TOL:
        raise DataError(f"{path}: matrix asymmetry {asym:.3e} exceeds {SYMMETRY_TOL}")
    S = (S + S.T) / 2.0
    if np.abs(np.diag(S) - 1.0).max() > SYMMETRY_TOL:
        raise DataError(f"{path}: diagonal entries must equal 1")
    np.fill_diagonal(S, 1.0)
    return validate_similarity(S)
