"""`FlowEngine`: one libveckm handle (one device, one sensor geometry, one head).

Host-buffer calls go through `vkm_predict_host` / `vkm_encode_host` (the C-ABI
does its own H2D/D2H).  Device calls take torch CUDA tensors; torch is only the
allocator and stream provider here, the work is the C-ABI's kernels.
"""

from __future__ import annotations

import collections
import ctypes as C
import math
import threading
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from .weights import Bases, MlpWeights

_dptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
_fptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731


def _torch():
    import torch
    return torch


class EngineCache:
    """Per-thread, size-bounded cache of `FlowEngine`s keyed by configuration.

    A handle is bound to one device and stream and is not re-entrant, so each
    host thread gets its own handles (distinct handles may run concurrently:
    the ctypes calls release the GIL, as the reference bindings promise,
    pkg/bindings/src/evflow_bindings/__init__.py:10-11).  At most `size`
    handles live per thread; the least recently used one is closed, which
    returns its device scratch and host threads."""

    def __init__(self, size: int = 4):
        self.size = int(size)
        self._tls = threading.local()

    def get(self, key, factory: Callable[[], "FlowEngine"]) -> "FlowEngine":
        lru = getattr(self._tls, "lru", None)
        if lru is None:
            lru = self._tls.lru = collections.OrderedDict()
        eng = lru.get(key)
        if eng is not None:
            lru.move_to_end(key)
            return eng
        eng = lru[key] = factory()
        while len(lru) > self.size:
            _, old = lru.popitem(last=False)
            old.close()
        return eng

    def clear(self) -> None:
        lru = getattr(self._tls, "lru", None)
        while lru:
            _, old = lru.popitem()
            old.close()


class FlowEngine:
    """Device-resident encoder (+ optional flow head) for one sensor geometry.

    Mirrors what `predict_flows` (flow.py:155-197) needs per slice: the weights'
    own bases (flow.py:173-174), the window radii and delta_t.
    """

    def __init__(self, width: int, height: int, delta_x: int, delta_y: int, delta_t: float,
                 bases: Bases, weights: Optional[MlpWeights] = None, device: int = 0,
                 mlp_mode: str = "auto"):
        lib = _lib.load()
        self._lib = lib
        # one handle is not re-entrant: calls from several host
        # threads on the same engine serialise instead of racing on its scratch
        self._lock = threading.RLock()
        self.width, self.height = int(width), int(height)
        self.delta_x, self.delta_y = int(delta_x), int(delta_y)
        self.delta_t = float(delta_t)
        self.device = int(device)
        self.embed_dim = bases.dim
        self.hidden = 0 if weights is None else weights.hidden
        p = _lib.VkmParams(self.width, self.height, self.delta_x, self.delta_y, self.embed_dim,
                           self.hidden, self.delta_t, self.device, _lib.MLP_MODES[mlp_mode])
        T = np.ascontiguousarray(bases.time_freqs, dtype=np.float64)
        X = np.ascontiguousarray(bases.x_freqs, dtype=np.float64)
        Y = np.ascontiguousarray(bases.y_freqs, dtype=np.float64)
        if weights is not None:
            w1 = np.ascontiguousarray(weights.w1, dtype=np.float32)
            b1 = np.ascontiguousarray(weights.b1, dtype=np.float32)
            w2 = np.ascontiguousarray(weights.w2, dtype=np.float32)
            b2 = np.ascontiguousarray(weights.b2, dtype=np.float32)
            wp = [_fptr(w1), _fptr(b1), _fptr(w2), _fptr(b2)]
        else:
            wp = [None, None, None, None]
        h = C.c_void_p()
        _lib.check(lib.vkm_create(C.byref(h), C.byref(p), _dptr(T), _dptr(X), _dptr(Y), *wp))
        self._h = h
        if weights is not None and np.asarray(weights.w1).dtype == np.float64:
            # the reference runs a float64 head for float64 weights (flow.py:98-106);
            # the f64 path keeps them unrounded (the f32 path uses the f32 copy)
            w64 = [np.ascontiguousarray(a, dtype=np.float64) for a in (weights.w1, weights.b1, weights.w2, weights.b2)]
            _lib.check(lib.vkm_set_weights_f64(h, *[_dptr(a) for a in w64]))

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.vkm_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_mlp_mode(self, mode: str) -> None:
        with self._lock: _lib.check(self._lib.vkm_set_mlp_mode(self._h, _lib.MLP_MODES[mode]))

    def set_profiling(self, enable: bool) -> None:
        with self._lock: _lib.check(self._lib.vkm_set_profiling(self._h, int(bool(enable))))

    def last_timings(self):
        """(ms[accumulate, pool, gather+mlp, total], kernel launches) of the last call."""
        ms = (C.c_float * 4)()
        n = C.c_int32()
        with self._lock: _lib.check(self._lib.vkm_last_timings(self._h, ms, C.byref(n)))
        return list(ms), int(n.value)

    # -- host-buffer API ---------------------------------------------------
    def predict_host(self, events: np.ndarray, t_start: float = math.nan, return_counts: bool = False):
        ev = np.ascontiguousarray(events, dtype=np.float64)
        n = len(ev)
        flows = np.empty((n, 2), dtype=np.float32)
        counts = np.empty(n, dtype=np.int32) if return_counts else None
        if n:
            with self._lock: _lib.check(self._lib.vkm_predict_host(self._h, ev.ctypes.data, n, float(t_start),
                                                  flows.ctypes.data,
                                                  counts.ctypes.data if counts is not None else None))
        return (flows, counts) if return_counts else flows

    def predict_host_wide(self, events: np.ndarray, t_start: float = math.nan, return_counts: bool = False):
        """predict_host with (n, 2) float64 flows (vkm_predict_host_wide)."""
        ev = np.ascontiguousarray(events, dtype=np.float64)
        n = len(ev)
        flows = np.empty((n, 2), dtype=np.float64)
        counts = np.empty(n, dtype=np.int32) if return_counts else None
        if n:
            with self._lock: _lib.check(self._lib.vkm_predict_host_wide(self._h, ev.ctypes.data, n, float(t_start), flows.ctypes.data,
                                                       counts.ctypes.data if counts is not None else None))
        return (flows, counts) if return_counts else flows

    def predict_host_checked(self, events: np.ndarray, window: float):
        """vkm_predict_host_checked: one host pass validates and packs the
        (n, 3) f64 rows; for valid, time-sorted rows within `window` returns
        the (n, 2) float64 flows (t_start = first row), else None (nothing
        ran: the caller validates, raises or sorts, and predicts)."""
        from .validation import _EventCheck
        ev = events
        if ev.dtype != np.float64 or ev.ndim != 2 or ev.shape[1] != 3 or not ev.flags.c_contiguous:
            return None
        n = len(ev)
        flows = np.empty((n, 2), dtype=np.float64)
        chk = _EventCheck()
        ran = C.c_int32(0)
        with self._lock: _lib.check(self._lib.vkm_predict_host_checked(self._h, ev.ctypes.data, n, float(window),
                                                                     flows.ctypes.data, C.byref(chk), C.byref(ran)))
        return flows if ran.value else None

    def predict_batch_host(self, events: np.ndarray, offsets: Sequence[int], t_starts=None,
                           flows: Optional[np.ndarray] = None, return_counts: bool = False):
        """Many slices from host memory in one pipelined call (copy-in of slice
        s+1 and copy-out of slice s-1 overlap the kernels of slice s).  Pass
        page-locked `events` / `flows` (e.g. torch pin_memory().numpy()) for
        the copies to run asynchronously."""
        ev = np.ascontiguousarray(events, dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        ns = len(off) - 1
        if flows is None:
            flows = np.empty((len(ev), 2), dtype=np.float32)
        counts = np.empty(len(ev), dtype=np.int32) if return_counts else None
        ts = None
        if t_starts is not None:
            ts_arr = np.ascontiguousarray(t_starts, dtype=np.float64)
            ts = _dptr(ts_arr)
        with self._lock: _lib.check(self._lib.vkm_predict_batch_host(
            self._h, ev.ctypes.data, off.ctypes.data_as(C.POINTER(C.c_int64)), ns, ts, flows.ctypes.data,
            counts.ctypes.data if counts is not None else None))
        return (flows, counts) if return_counts else flows

    def encode_host(self, events: np.ndarray, t_start: float = math.nan, return_counts: bool = False):
        ev = np.ascontiguousarray(events, dtype=np.float64)
        n = len(ev)
        feats = np.empty((n, 2 * self.embed_dim), dtype=np.float32)
        counts = np.empty(n, dtype=np.int32) if return_counts else None
        if n:
            with self._lock: _lib.check(self._lib.vkm_encode_host(self._h, ev.ctypes.data, n, float(t_start),
                                                 feats.ctypes.data,
                                                 counts.ctypes.data if counts is not None else None))
        return (feats, counts) if return_counts else feats

    # -- precision="f64" (complex128 grid, float64 features and head) ----------
    def predict_host_f64(self, events: np.ndarray, t_start: float = math.nan, return_counts: bool = False):
        ev = np.ascontiguousarray(events, dtype=np.float64)
        n = len(ev)
        flows = np.empty((n, 2), dtype=np.float64)
        counts = np.empty(n, dtype=np.int32) if return_counts else None
        if n:
            with self._lock: _lib.check(self._lib.vkm_predict_f64_host(self._h, ev.ctypes.data, n, float(t_start), flows.ctypes.data,
                                                      counts.ctypes.data if counts is not None else None))
        return (flows, counts) if return_counts else flows

    def encode_host_f64(self, events: np.ndarray, t_start: float = math.nan, return_counts: bool = False):
        ev = np.ascontiguousarray(events, dtype=np.float64)
        n = len(ev)
        feats = np.empty((n, 2 * self.embed_dim), dtype=np.float64)
        counts = np.empty(n, dtype=np.int32) if return_counts else None
        if n:
            with self._lock: _lib.check(self._lib.vkm_encode_f64_host(self._h, ev.ctypes.data, n, float(t_start), feats.ctypes.data,
                                                     counts.ctypes.data if counts is not None else None))
        return (feats, counts) if return_counts else feats

    def predict_device_f64(self, events, t_start: float = math.nan, flows=None, counts=None, stream=None):
        torch = _torch()
        self._check_events(events)
        n = events.shape[0]
        if flows is None:
            flows = torch.empty((n, 2), dtype=torch.float64, device=events.device)
        with self._lock: _lib.check(self._lib.vkm_predict_f64(self._h, C.c_void_p(events.data_ptr()), n, float(t_start),
                                             C.c_void_p(flows.data_ptr()),
                                             C.c_void_p(counts.data_ptr()) if counts is not None else None,
                                             self._stream(stream)))
        return flows

    def direct_encode_host(self, events: np.ndarray, queries, return_counts: bool = False):
        """oracle_encode (encoder.py:413-440) on the GPU: f64 direct summation
        over each query's window; `events` time-sorted (n, 3) rows, `queries`
        indices into them.  Returns (nq, D) complex128 (+ int32 counts)."""
        ev = np.ascontiguousarray(events, dtype=np.float64)
        q = np.ascontiguousarray(queries, dtype=np.int64)
        emb = np.empty((len(q), self.embed_dim), dtype=np.complex128)
        counts = np.empty(len(q), dtype=np.int32)
        if len(q):
            with self._lock: _lib.check(self._lib.vkm_direct_encode_host(self._h, ev.ctypes.data, len(ev), q.ctypes.data, len(q),
                                                        emb.ctypes.data, counts.ctypes.data))
        return (emb, counts) if return_counts else emb

    # -- device API (torch tensors) -----------------------------------------
    def _stream(self, stream):
        torch = _torch()
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return C.c_void_p(stream.cuda_stream)

    @staticmethod
    def _check_events(ev):
        if ev.dtype.itemsize != 8 or ev.ndim != 2 or ev.shape[1] != 3 or not ev.is_contiguous() or not ev.is_cuda:
            raise ValueError("device events must be a contiguous CUDA float64 tensor of shape (n, 3)")

    def predict_device(self, events, t_start: float = math.nan, flows=None, counts=None, stream=None):
        torch = _torch()
        self._check_events(events)
        n = events.shape[0]
        if flows is None:
            flows = torch.empty((n, 2), dtype=torch.float32, device=events.device)
        with self._lock: _lib.check(self._lib.vkm_predict(self._h, C.c_void_p(events.data_ptr()), n, float(t_start),
                                         C.c_void_p(flows.data_ptr()),
                                         C.c_void_p(counts.data_ptr()) if counts is not None else None,
                                         self._stream(stream)))
        return flows

    def encode_device(self, events, t_start: float = math.nan, feats=None, counts=None, stream=None):
        torch = _torch()
        self._check_events(events)
        n = events.shape[0]
        if feats is None:
            feats = torch.empty((n, 2 * self.embed_dim), dtype=torch.float32, device=events.device)
        with self._lock: _lib.check(self._lib.vkm_encode(self._h, C.c_void_p(events.data_ptr()), n, float(t_start),
                                        C.c_void_p(feats.data_ptr()),
                                        C.c_void_p(counts.data_ptr()) if counts is not None else None,
                                        self._stream(stream)))
        return feats

    def predict_batch_device(self, events, offsets: Sequence[int], t_starts=None, flows=None, counts=None,
                             stream=None):
        torch = _torch()
        self._check_events(events)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        ns = len(off) - 1
        if flows is None:
            flows = torch.empty((events.shape[0], 2), dtype=torch.float32, device=events.device)
        ts = None
        if t_starts is not None:
            ts_arr = np.ascontiguousarray(t_starts, dtype=np.float64)
            ts = _dptr(ts_arr)
        with self._lock: _lib.check(self._lib.vkm_predict_batch(
            self._h, C.c_void_p(events.data_ptr()), off.ctypes.data_as(C.POINTER(C.c_int64)), ns, ts,
            C.c_void_p(flows.data_ptr()), C.c_void_p(counts.data_ptr()) if counts is not None else None,
            self._stream(stream)))
        return flows

    def pixel_order_device(self, events, t_start: float = math.nan, stream=None):
        """accumulate_grid's stable pixel-major order (encoder.py:255-259):
        ((W*H + 1) int32 run starts, (n) int32 event per slot)."""
        torch = _torch()
        self._check_events(events)
        n = events.shape[0]
        start = torch.empty(self.width * self.height + 1, dtype=torch.int32, device=events.device)
        order = torch.empty(max(n, 1), dtype=torch.int32, device=events.device)
        with self._lock: _lib.check(self._lib.vkm_pixel_order(self._h, C.c_void_p(events.data_ptr()), n,
                                                            float(t_start), C.c_void_p(start.data_ptr()),
                                                            C.c_void_p(order.data_ptr()), self._stream(stream)))
        return start, order[:n]

    def grid_device(self, events, t_start: float = math.nan, pooled: bool = False, stream=None):
        """Per-pixel grid in the reference PixelGrid layout: ((W, H, D) complex64, (W, H) int32)."""
        torch = _torch()
        self._check_events(events)
        W, H, D = self.width, self.height, self.embed_dim
        g = torch.empty((W, H, D, 2), dtype=torch.float32, device=events.device)
        c = torch.empty((W, H), dtype=torch.int32, device=events.device)
        with self._lock: _lib.check(self._lib.vkm_grid(self._h, C.c_void_p(events.data_ptr()), events.shape[0], float(t_start),
                                      int(bool(pooled)), C.c_void_p(g.data_ptr()), C.c_void_p(c.data_ptr()),
                                      self._stream(stream)))
        return torch.view_as_complex(g), c


def predict_multi_host(engines: Sequence["FlowEngine"], events: np.ndarray, offsets: Sequence[int], t_starts=None,
                       flows: Optional[np.ndarray] = None) -> np.ndarray:
    """vkm_predict_multi_host: the slices split into contiguous ranges of
    about equal event counts, one per engine (device), each range pipelined
    through its engine on its own host thread; no collective (SURVEY §8e,
    config 4).  Engines must be distinct handles with the same geometry."""
    if not engines:
        raise ValueError("need at least one engine")
    lib = engines[0]._lib
    ev = np.ascontiguousarray(events, dtype=np.float64)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    if flows is None:
        flows = np.empty((len(ev), 2), dtype=np.float32)
    ts = None
    if t_starts is not None:
        ts_arr = np.ascontiguousarray(t_starts, dtype=np.float64)
        ts = _dptr(ts_arr)
    hs = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
    _lib.check(lib.vkm_predict_multi_host(hs, len(engines), ev.ctypes.data, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                          len(off) - 1, ts, flows.ctypes.data, None))
    return flows
