"""Device-memory plumbing: torch owns HBM buffers and streams; kernels live in the .so.

* ``to_device`` moves a host array (or passes a CUDA tensor through).
* ``device_matrix`` keeps a single-slot identity cache of the last host matrix
  uploaded, so the drop-in stage functions called one after another on the same
  numpy ``S`` (as the reference pipeline does, pipeline.py:191-218) copy it to
  HBM once.
* ``Workspace`` hands out reusable scratch for the C ABI's ``ws`` arguments.
* ``LazyHost`` materialises a host numpy view of a device tensor on first use.
"""

from __future__ import annotations

import weakref

import numpy as np


def torch():
    import torch as _t
    return _t


def is_device(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_device(a, dtype=None):
    """Host numpy / torch tensor -> contiguous CUDA tensor of `dtype`."""
    t = torch()
    if isinstance(a, t.Tensor):
        x = a
        if not x.is_cuda:
            x = x.cuda()
        if dtype is not None and x.dtype != dtype:
            x = x.to(dtype)
        return x.contiguous()
    arr = np.ascontiguousarray(a)
    x = t.from_numpy(arr)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.to("cuda", non_blocking=False).contiguous()


def to_host(x) -> np.ndarray:
    t = torch()
    if isinstance(x, t.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _fingerprint(S: np.ndarray) -> tuple:
    flat = S.reshape(-1)
    step = max(1, flat.shape[0] // 4096)
    sample = flat[::step]
    return (S.shape, S.dtype.str, S.__array_interface__["data"][0], float(np.nansum(sample)),
            int(np.isnan(sample).sum()))


class _MatrixCache:
    ref = None
    fp = None
    dev = None


def device_matrix(S):
    """float64 CUDA tensor for S; host arrays are uploaded once per object."""
    t = torch()
    if isinstance(S, t.Tensor):
        return to_device(S, t.float64)
    S = np.asarray(S)
    if _MatrixCache.ref is not None and _MatrixCache.ref() is S and _MatrixCache.fp == _fingerprint(S):
        return _MatrixCache.dev
    dev = to_device(np.ascontiguousarray(S, dtype=np.float64), t.float64)
    try:
        _MatrixCache.ref = weakref.ref(S)
        _MatrixCache.fp = _fingerprint(S)
        _MatrixCache.dev = dev
    except TypeError:  # pragma: no cover - non-weakrefable
        _MatrixCache.ref = None
    return dev


def forget_cached_matrix() -> None:
    _MatrixCache.ref = None
    _MatrixCache.fp = None
    _MatrixCache.dev = None


class Workspace:
    """Grow-only scratch buffer reused by consecutive stream-ordered calls."""

    _buf = None

    @classmethod
    def get(cls, nbytes: int):
        t = torch()
        nbytes = max(int(nbytes), 256)
        if cls._buf is None or cls._buf.numel() < nbytes:
            cls._buf = None
            cls._buf = t.empty(nbytes, dtype=t.uint8, device="cuda")
        return cls._buf


def empty(shape, dtype):
    t = torch()
    return t.empty(shape, dtype=dtype, device="cuda")


class LazyHost:
    """Descriptor-style holder: device tensor now, numpy on first host access."""

    def __init__(self, dev=None, host=None, dtype=None):
        self.dev = dev
        self._host = host
        self.dtype = dtype
        self._conv = {}

    @property
    def host(self) -> np.ndarray:
        if self._host is None:
            h = self.dev.detach().cpu().numpy()
            if self.dtype is not None and h.dtype != self.dtype:
                h = h.astype(self.dtype)
            self._host = h
        return self._host

    def device(self, dtype=None):
        """Device tensor (converted copies are cached so raw pointers stay valid)."""
        if self.dev is None:
            self.dev = to_device(self._host)
        if dtype is not None and self.dev.dtype != dtype:
            if dtype not in self._conv:
                self._conv[dtype] = self.dev.to(dtype).contiguous()
            return self._conv[dtype]
        return self.dev
