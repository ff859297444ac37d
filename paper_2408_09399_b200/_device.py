"""Device-memory plumbing: torch owns HBM buffers and streams; kernels live in the .so.

* ``to_device`` moves a host array (or passes a CUDA tensor through).
* ``device_matrix`` uploads a host matrix (no cross-call cache: an in-place edit
  of S between drop-in stage calls is always seen); ``chained_device`` reuses the
  device S a previous stage result carries only when the caller passes that
  same CUDA tensor.
* ``Workspace`` hands out reusable scratch for the C ABI's ``ws`` arguments,
  one buffer per (device, stream).
* ``LazyHost`` materialises a host numpy view of a device tensor on first use.
"""

from __future__ import annotations

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


def device_matrix(S):
    """float64 CUDA tensor for S.

    A CUDA tensor passes through; a host array is uploaded on every call, so a
    drop-in stage always sees the matrix's current contents (the reference
    re-reads S in every stage; an in-place edit between stage calls must not
    leave a stale device copy).  Stages chained by this package pass the device
    tensor along (``lists.S_device``, ``graph.S_device``) and upload once.
    """
    t = torch()
    if isinstance(S, t.Tensor):
        return to_device(S, t.float64)
    return to_device(np.asarray(S, dtype=np.float64), t.float64)


def chained_device(obj, S):
    """The device S carried by a previous stage's result when it IS the caller's S.

    Only a CUDA tensor identical to the one the chain was built on is reused;
    for a host array the caller's current contents are uploaded again.
    """
    Sd = getattr(obj, "S_device", None) if obj is not None else None
    if Sd is not None and is_device(S) and S is Sd:
        return Sd
    return device_matrix(S)


class Workspace:
    """Grow-only scratch buffers, one per (device, stream).

    Calls on one stream are ordered, so they may share a buffer; calls on
    different streams get different buffers.
    """

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, stream=None):
        t = torch()
        nbytes = max(int(nbytes), 256)
        s = stream if stream is not None else t.cuda.current_stream()
        key = (s.device.index if s.device.index is not None else t.cuda.current_device(), s.cuda_stream)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            cls._bufs.pop(key, None)
            buf = t.empty(nbytes, dtype=t.uint8, device=s.device)
            cls._bufs[key] = buf
        return buf

    @classmethod
    def release(cls) -> None:
        cls._bufs.clear()


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
