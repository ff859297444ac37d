"""ctypes binding of libtmfg_b200.so (the C ABI declared in include/tmfg_b200.h).

The library holds every kernel of the accelerated path.  There is no CPU
fallback: if the shared library is missing or no CUDA device is present, the
first call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = _LIB_DIR / "libtmfg_b200.so"
if os.environ.get("TG_LIB"):   # developer override (e.g. the TM_PROFILE build used by tools/tmfg_profile.py)
    LIB_PATH = Path(os.environ["TG_LIB"])

TG_OK = 0
TG_ERR_NOT_REDUCIBLE = 7
TG_ERR_ARG = 1
TG_ERR_CUDA = 2
TG_ERR_WORKSPACE = 3
TG_ERR_CAPACITY = 5
TG_ERR_TRACE = 6

TG_BAD_NAN = 1
TG_BAD_ASYM = 2
TG_BAD_DIAG = 4
TG_BAD_RANGE = 8

_ERRNAMES = {TG_ERR_ARG: "invalid argument", TG_ERR_CUDA: "CUDA error", TG_ERR_WORKSPACE: "workspace too small",
             TG_ERR_CAPACITY: "capacity exceeded", TG_ERR_TRACE: "trace error"}


class NativeUnavailable(RuntimeError):
    """libtmfg_b200.so is not built or no CUDA device is visible."""


class NativeError(RuntimeError):
    def __init__(self, fn: str, code: int, detail: str = ""):
        super().__init__(f"{fn} failed: {_ERRNAMES.get(code, code)} {detail}".strip())
        self.code = code


c_p = ctypes.c_void_p
c_i64 = ctypes.c_int64
c_sz = ctypes.c_size_t
c_dbl = ctypes.c_double


class TgOracle(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("n", c_i64), ("matrix", c_p), ("H", c_i64), ("hub_dist", c_p),
                ("near_indptr", c_p), ("near_ids", c_p), ("near_dist", c_p), ("rev_indptr", c_p),
                ("rev_ids", c_p), ("rev_dist", c_p)]


# name -> (restype, argtypes)
_PROTOS = {
    "tg_abi_version": (ctypes.c_int, []),
    "tg_last_error": (ctypes.c_char_p, []),
    "tg_launch_count": (ctypes.c_longlong, []),
    "tg_pearson_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "tg_pearson_f64": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p, c_sz, c_p]),
    "tg_pearson_refexact_f64": (ctypes.c_int, [c_p, c_p, c_i64, c_i64, c_p, c_p]),
    "tg_validate_f64": (ctypes.c_int, [c_p, c_i64, c_p, c_p]),
    "tg_row_sort_workspace_bytes": (c_sz, [c_i64]),
    "tg_row_sort_f64": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_sz, c_p]),
    "tg_row_sums_workspace_bytes": (c_sz, [c_i64]),
    "tg_row_sums_f64": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "tg_initial_clique": (ctypes.c_int, [c_p, c_i64, c_p, c_p]),
    "tg_initial_clique_screened_workspace_bytes": (c_sz, [c_i64]),
    "tg_initial_clique_screened": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_sz, c_p]),
    "tg_tmfg_workspace_bytes": (c_sz, [c_i64]),
    "tg_tmfg_heap": (ctypes.c_int, [c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.c_int32, c_p, c_sz, c_p]),
    "tg_tmfg_variant_workspace_bytes": (c_sz, [c_i64]),
    "tg_tmfg_exact": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_tmfg_corr": (ctypes.c_int, [c_p, c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_edge_weights": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_p, c_p]),
    "tg_weighted_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "tg_to_weighted": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_sssp_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "tg_sssp_rows": (ctypes.c_int, [c_p, c_p, c_p, c_i64, c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "tg_select_hubs_workspace_bytes": (c_sz, [c_i64]),
    "tg_select_hubs": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p, c_sz, c_p]),
    "tg_nearest_hub": (ctypes.c_int, [c_p, c_p, c_i64, c_i64, c_dbl, c_p, c_p, c_p, c_p]),
    "tg_truncated_workspace_bytes": (c_sz, [c_i64]),
    "tg_truncated": (ctypes.c_int, [c_p, c_p, c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_near_transpose_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "tg_near_transpose": (ctypes.c_int, [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_bubble_tree_workspace_bytes": (c_sz, [c_i64]),
    "tg_bubble_tree": (ctypes.c_int, [c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_orient_edges": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_i64, c_p, c_p, c_p]),
    "tg_bubble_sinks_workspace_bytes": (c_sz, [c_i64]),
    "tg_bubble_sinks": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "tg_assign_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "tg_assign_vertices": (ctypes.c_int, [ctypes.POINTER(TgOracle), c_p, c_i64, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "tg_group_blocks": (ctypes.c_int, [ctypes.POINTER(TgOracle), c_p, c_p, c_i64, c_p, c_p, c_p]),
    "tg_oracle_block": (ctypes.c_int, [ctypes.POINTER(TgOracle), c_p, c_i64, c_p, c_i64, ctypes.c_int32, c_p, c_p]),
    "tg_group_max_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64]),
    "tg_group_max_batch": (ctypes.c_int, [ctypes.POINTER(TgOracle), c_p, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p,
                                          c_i64, c_p, c_sz, c_p]),
    "tg_nn_chain_batch": (ctypes.c_int, [c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "tg_serialize_dendrogram": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_i64, c_p, c_sz, ctypes.POINTER(c_sz)]),
    "tg_cut_labels": (ctypes.c_int, [c_p, c_p, c_i64, c_i64, c_p, c_p]),
    "tg_group_tiles_fill": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_p]),
    "tg_release_cached_memory": (ctypes.c_int, []),
    "tg_build_hierarchy": (ctypes.c_int, [ctypes.POINTER(TgOracle), c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p]),
}

EXPORTED = tuple(_PROTOS)

_lib = None
MISSING: tuple = ()


def load(require_cuda: bool = True):
    """Load the library (once) and bind prototypes; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(no CPU fallback exists)")
    lib = ctypes.CDLL(str(LIB_PATH))
    missing = []
    for name, (res, args) in _PROTOS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    global MISSING
    MISSING = tuple(missing)
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible: the B200 path has no CPU fallback")
    _lib = lib
    return lib


def check(fn: str, code: int) -> None:
    if code != TG_OK:
        detail = ""
        try:
            detail = (_lib.tg_last_error() or b"").decode() if code == TG_ERR_CUDA else ""
        except Exception:  # pragma: no cover
            pass
        raise NativeError(fn, code, detail)


def call(fn: str, *args) -> None:
    lib = load()
    if fn in MISSING:
        raise NativeUnavailable(f"{fn} is not in {LIB_PATH}")
    check(fn, getattr(lib, fn)(*args))


def size(fn: str, *args) -> int:
    return int(getattr(load(), fn)(*args))


def ptr(t) -> ctypes.c_void_p:
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return c_p(0)
    return c_p(t.data_ptr())


def stream_ptr(stream=None) -> ctypes.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_p(s.cuda_stream)


def library_loaded_path() -> str | None:
    return str(LIB_PATH) if _lib is not None else None


def host_int64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


__all__ = ["load", "call", "size", "ptr", "stream_ptr", "NativeUnavailable", "NativeError", "TgOracle",
           "EXPORTED", "LIB_PATH", "os"]
