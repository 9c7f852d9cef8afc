"""Reused page-locked host staging for the host-memory batch APIs.

Pinning hundreds of MB per call costs more than the asynchronous copies it
enables, so each host thread keeps grow-only pinned buffers (torch's host
allocator) and the calls copy their results out of them before returning."""

from __future__ import annotations

import threading

import numpy as np

_local = threading.local()


def pinned(name: str, n: int, dtype=np.float64) -> np.ndarray:
    """A length-n page-locked array of `dtype`, valid until this thread's next
    request under the same name."""
    dt = np.dtype(dtype)
    key = (name, dt.str)
    bufs = getattr(_local, "bufs", None)
    if bufs is None:
        bufs = _local.bufs = {}
    buf = bufs.get(key)
    if buf is None or len(buf) < n:
        import torch
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
               np.dtype(np.int32): torch.int32}[dt]
        buf = torch.empty(max(int(n), 1 << 20), dtype=tdt).pin_memory().numpy()
        bufs[key] = buf
    return buf[:n]


def widen(src: np.ndarray) -> np.ndarray:
    """float64 copy of a float32 array through libveckm's pooled, streaming
    widening (vkm_widen_f32): the host side of the batch APIs' float64
    results."""
    from . import _lib
    a = np.ascontiguousarray(src, dtype=np.float32)
    out = np.empty(a.shape, dtype=np.float64)
    if a.size:
        _lib.check(_lib.load().vkm_widen_f32(a.ctypes.data, out.ctypes.data, a.size))
    return out


def concat_rows(blocks, dst: np.ndarray) -> None:
    """dst[...] = the row blocks back to back (C-contiguous float64 arrays of
    dst's row width), copied by libveckm's host pool (vkm_concat_rows)."""
    import ctypes as C
    from . import _lib
    arrs = [np.ascontiguousarray(b, dtype=np.float64) for b in blocks]
    ld = dst.shape[1] if dst.ndim == 2 else 1
    ptrs = (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])
    rows = np.array([len(a) for a in arrs], dtype=np.int64)
    assert rows.sum() == len(dst) and all(a.ndim == 2 and a.shape[1] == ld for a in arrs if len(a))
    _lib.check(_lib.load().vkm_concat_rows(ptrs, rows.ctypes.data, len(arrs), ld, dst.ctypes.data))
