"""TMFG construction on the B200 (drop-in for tmfgclust.tmfg's heap builder)."""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _native as N


def initial_clique_device(Sd, rowsum=None):
    """tmfg.py:71-79 on device: int32[4] CUDA tensor (ascending)."""
    t = D.torch()
    n = int(Sd.shape[0])
    if rowsum is None:
        rowsum = D.empty((n,), t.float64)
        ws = D.Workspace.get(N.size("tg_row_sums_workspace_bytes", n))
        N.call("tg_row_sums_f64", N.ptr(Sd), n, N.ptr(rowsum), N.ptr(ws), ws.numel(), N.stream_ptr())
    clique = D.empty((4,), t.int32)
    N.call("tg_initial_clique", N.ptr(rowsum), n, N.ptr(clique), N.stream_ptr())
    return clique


def select_initial_clique(S) -> tuple[int, int, int, int]:
    """The 4 vertices with the largest off-diagonal row sums, id-ascending (tmfg.py:71-79)."""
    Sd = D.device_matrix(S)
    c = initial_clique_device(Sd).cpu().numpy()
    return tuple(int(v) for v in c)
