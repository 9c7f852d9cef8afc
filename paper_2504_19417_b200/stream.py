"""Event streams: loading, slicing into windows, and streaming prediction.

Host-side restatement of the reference's stream ingestion (events.py:66-387):
the EVN1 binary format (12-byte header `EVN1` + u32 width + u32 height, then
packed 17-byte little-endian records f64 t, i32 x, i32 y, i8 polarity), the
CSV format, and `slice_stream`'s windowing semantics (half-open windows
[t0 + i·stride, t0 + i·stride + 2δt), overlapping strides, interior gaps kept
as empty slices, trailing empty windows dropped).  Same checks, messages and
exception types.

`predict_stream` is the B200 streaming path: every window becomes one slice
of one `vkm_predict_batch_host` call (copy-in / kernels / copy-out overlap,
up to 64 windows per launch sequence), with the window start as the slice's
time origin — exactly what `predict_flows` sees for a `slice_stream` slice.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from .errors import EventParseError, GeometryError

BINARY_MAGIC = b"EVN1"
BINARY_RECORD_DTYPE = np.dtype([("t", "<f8"), ("x", "<i4"), ("y", "<i4"), ("p", "<i1")])   # 17 bytes, packed


@dataclass(frozen=True)
class CameraGeometry:
    width: int
    height: int

    def __post_init__(self) -> None:
        if self.width < 1 or self.height < 1:
            raise ValueError(f"geometry must be at least 1x1, got {self.width}x{self.height}")

    def contains(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        return (x >= 0) & (x < self.width) & (y >= 0) & (y < self.height)


@dataclass
class EventStream:
    """Parallel arrays t (f64 s), x, y (int32), optional polarity (int8) (events.py:66-87)."""

    t: np.ndarray
    x: np.ndarray
    y: np.ndarray
    geometry: CameraGeometry
    polarity: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        self.t = np.asarray(self.t, dtype=np.float64)
        self.x = np.asarray(self.x, dtype=np.int32)
        self.y = np.asarray(self.y, dtype=np.int32)
        if self.polarity is not None:
            self.polarity = np.asarray(self.polarity, dtype=np.int8)
            if len(self.polarity) != len(self.t):
                raise ValueError("polarity length mismatch")
        t, x, y = self.t, self.x, self.y
        if not (len(t) == len(x) == len(y)):
            raise ValueError("t, x, y must have equal length")
        if len(t):
            if not np.all(np.isfinite(t)) or np.any(t < 0):
                bad = int(np.flatnonzero(~np.isfinite(t) | (t < 0))[0])
                raise ValueError(f"event {bad}: timestamp {t[bad]} must be finite and non-negative")
            inside = self.geometry.contains(x, y)
            if not np.all(inside):
                bad = int(np.flatnonzero(~inside)[0])
                raise GeometryError(f"event {bad}: ({x[bad]}, {y[bad]}) outside geometry "
                                    f"{self.geometry.width}x{self.geometry.height}")

    def __len__(self) -> int:
        return len(self.t)


@dataclass
class EventSlice:
    """Events of one window [t_start, t_start + window], sorted by t, with the
    reference's construction checks (events.py:90-131: ulp-tolerant window
    bounds, ascending times, geometry)."""

    t: np.ndarray
    x: np.ndarray
    y: np.ndarray
    t_start: float
    window: float
    geometry: Optional[CameraGeometry] = None
    polarity: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        self.t = np.asarray(self.t, dtype=np.float64)
        self.x = np.asarray(self.x, dtype=np.int32)
        self.y = np.asarray(self.y, dtype=np.int32)
        if self.polarity is not None:
            self.polarity = np.asarray(self.polarity, dtype=np.int8)
        if self.window <= 0:
            raise ValueError("window must be positive")
        n = len(self.t)
        if len(self.x) != n or len(self.y) != n:
            raise ValueError("t, x, y must have equal length")
        if n:
            upper = self.t_start + self.window
            slack = 4.0 * np.spacing(max(abs(upper), self.window))   # rebasing rounds edge times
            if self.t[0] < self.t_start - slack or self.t[-1] > upper + slack:
                raise ValueError(f"timestamps [{self.t.min()}, {self.t.max()}] fall outside "
                                 f"window [{self.t_start}, {upper}]")
            if np.any(self.t[1:] < self.t[:-1]):
                raise ValueError("slice events must be sorted ascending by t")
        if self.geometry is not None:
            outside = np.flatnonzero(~self.geometry.contains(self.x, self.y))
            if len(outside):
                bad = int(outside[0])
                raise GeometryError(f"event {bad} at ({self.x[bad]}, {self.y[bad]}) outside geometry")

    def __len__(self) -> int:
        return len(self.t)

    @property
    def n(self) -> int:
        return len(self.t)

    def events(self) -> np.ndarray:
        """(n, 3) float64 [t, x, y] rows, the estimator's input layout."""
        return np.stack([self.t, self.x.astype(np.float64), self.y.astype(np.float64)], axis=1)


StreamSlice = EventSlice   # slice_stream's windows


# ---------------------------------------------------------------------------
# Event files (events.py:177-311).  The formats and the error messages are the
# reference's; the parsing is columnar: fields are converted a column at a
# time by the C-level float/int constructors and checked with numpy, and only
# when something fails is the first offending line re-examined on its own to
# raise the reference's exception for it (line order first, then the check
# order within the line: field count, t/x/y parse, t range, x, y, polarity).
# ---------------------------------------------------------------------------

def _first_bad(values, conv) -> Tuple[Optional[list], int]:
    """(converted column, -1) or (None, index of the first unconvertible field)."""
    try:
        return list(map(conv, values)), -1
    except ValueError:
        for k, v in enumerate(values):
            try:
                conv(v)
            except ValueError:
                return None, k
    raise AssertionError("unreachable")


def _csv_line_error(path: str, lineno: int, fields: List[str], geometry: CameraGeometry) -> Exception:
    """The exception the reference raises for one offending CSV line."""
    if len(fields) not in (3, 4):
        return EventParseError(f"{path}:{lineno}: expected 3 or 4 fields, got {len(fields)}")
    try:
        t, x, y = float(fields[0]), int(fields[1]), int(fields[2])
    except ValueError as exc:
        err = EventParseError(f"{path}:{lineno}: {exc}")
        err.__cause__ = exc
        return err
    if not np.isfinite(t) or t < 0:
        return EventParseError(f"{path}:{lineno}: timestamp {t} not finite and non-negative")
    if not 0 <= x < geometry.width:
        return GeometryError(f"{path}:{lineno}: x={x} violates 0 <= x < {geometry.width}")
    if not 0 <= y < geometry.height:
        return GeometryError(f"{path}:{lineno}: y={y} violates 0 <= y < {geometry.height}")
    if len(fields) == 4:
        try:
            p = int(fields[3])
        except ValueError as exc:
            err = EventParseError(f"{path}:{lineno}: bad polarity {fields[3]!r}")
            err.__cause__ = exc
            return err
        if p not in (0, 1, -1):
            return EventParseError(f"{path}:{lineno}: polarity must be 0, 1 or -1, got {p}")
    raise AssertionError(f"line {lineno} has no error")


def _parse_csv(path: str, geometry: CameraGeometry) -> EventStream:
    """CSV events (events.py:177-236): optional header line (a non-numeric first
    field on line 1), 3 or 4 fields, polarity in {0, 1, -1}; blank lines skipped."""
    with open(path, "r", encoding="utf-8") as fh:
        raw = fh.read().splitlines()
    rows, linenos = [], []
    for k, line in enumerate(raw):
        line = line.strip()
        if line:
            rows.append(line.split(","))
            linenos.append(k + 1)
    if rows and linenos[0] == 1 and _first_bad([rows[0][0]], float)[1] == 0:
        rows, linenos = rows[1:], linenos[1:]          # header
    m = len(rows)
    nf = np.fromiter((len(r) for r in rows), dtype=np.int64, count=m)
    cand = [int(np.flatnonzero((nf != 3) & (nf != 4))[0])] if np.any((nf != 3) & (nf != 4)) else []
    stop = min(cand) if cand else m                    # lines past the first failure never matter
    cols = [[r[c] for r in rows[:stop]] for c in range(3)]
    parsed = []
    for c, conv in enumerate((float, int, int)):
        vals, bad = _first_bad(cols[c], conv)
        if bad >= 0:
            stop = min(stop, bad)
            cand.append(bad)
        parsed.append(vals)
    if any(v is None for v in parsed):                 # re-convert the clean prefix
        parsed = [list(map(conv, cols[c][:stop])) for c, conv in enumerate((float, int, int))]
    t = np.array(parsed[0][:stop], dtype=np.float64)
    x = np.array(parsed[1][:stop], dtype=np.int64)
    y = np.array(parsed[2][:stop], dtype=np.int64)
    value_bad = (~np.isfinite(t)) | (t < 0) | (x < 0) | (x >= geometry.width) | (y < 0) | (y >= geometry.height)
    four = nf[:stop] == 4
    pol = np.zeros(stop, dtype=np.int64)
    if np.any(four):
        idx = np.flatnonzero(four)
        pv, bad = _first_bad([rows[i][3] for i in idx], int)
        if bad >= 0:
            cand.append(int(idx[bad]))
            idx = idx[:bad]
            pv = list(map(int, [rows[i][3] for i in idx]))
        pol[idx] = pv
        value_bad[idx] |= ~np.isin(pol[idx], (0, 1, -1))
    if np.any(value_bad):
        cand.append(int(np.flatnonzero(value_bad)[0]))
    if cand:
        k = min(cand)
        raise _csv_line_error(path, linenos[k], rows[k], geometry)
    return EventStream(t, x.astype(np.int32), y.astype(np.int32), geometry,
                       pol.astype(np.int8) if np.any(four) else None)


def _parse_binary(path: str) -> EventStream:
    """EVN1 (events.py:238-266): `EVN1`, u32 width, u32 height, then packed
    17-byte little-endian records (f64 t, i32 x, i32 y, i8 polarity)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(12)
    if len(head) < 12 or head[:4] != BINARY_MAGIC:
        raise EventParseError(f"{path}: missing {BINARY_MAGIC!r} header")
    width, height = struct.unpack_from("<II", head, 4)
    rec = BINARY_RECORD_DTYPE.itemsize
    if (size - 12) % rec:
        raise EventParseError(f"{path}: truncated record at offset {size} "
                              f"(payload not a multiple of {rec} bytes)")
    geometry = CameraGeometry(width, height)
    records = np.fromfile(path, dtype=BINARY_RECORD_DTYPE, offset=12)
    x, y = records["x"].astype(np.int32), records["y"].astype(np.int32)
    outside = np.flatnonzero(~geometry.contains(x, y))
    if len(outside):
        k = int(outside[0])
        raise GeometryError(f"{path}: record {k} at ({x[k]}, {y[k]}) outside geometry {width}x{height}")
    return EventStream(records["t"].astype(np.float64), x, y, geometry, records["p"].astype(np.int8))


_READERS = {"csv": lambda path, g: _parse_csv(path, g), "binary": lambda path, g: _parse_binary(path)}


def load_events(path: str, fmt: str = "csv", geometry: Optional[CameraGeometry] = None) -> EventStream:
    """Read an event file (events.py:269-291): CSV needs the geometry, EVN1
    carries it (a declared geometry must then match)."""
    if not os.path.exists(path):
        raise EventParseError(f"{path}: no such file")
    if fmt not in _READERS:
        raise ValueError(f"unknown event format {fmt!r}")
    if fmt == "csv" and geometry is None:
        raise ValueError("CSV event files require an explicit geometry")
    stream = _READERS[fmt](path, geometry)
    if fmt == "binary" and geometry is not None and geometry != stream.geometry:
        raise GeometryError(f"{path}: file geometry {stream.geometry.width}x{stream.geometry.height} "
                            f"does not match declared {geometry.width}x{geometry.height}")
    return stream


def write_events_binary(stream: EventStream, path: str) -> None:
    """EVN1 writer (events.py:305-311)."""
    rec = np.zeros(len(stream), dtype=BINARY_RECORD_DTYPE)
    rec["t"], rec["x"], rec["y"] = stream.t, stream.x, stream.y
    if stream.polarity is not None:
        rec["p"] = stream.polarity
    head = BINARY_MAGIC + struct.pack("<II", stream.geometry.width, stream.geometry.height)
    with open(path, "wb") as fh:
        fh.write(head + rec.tobytes())


def write_events_csv(stream: EventStream, path: str) -> None:
    """CSV writer (events.py:294-302): shortest round-trip repr of t, integer x, y[, p]."""
    cols = [map(repr, stream.t.astype(np.float64).tolist()), map(str, stream.x.tolist()), map(str, stream.y.tolist())]
    if stream.polarity is not None:
        cols.append(map(str, stream.polarity.tolist()))
    body = "".join(",".join(f) + "\n" for f in zip(*cols))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(body)


def filter_polarity(stream: EventStream, keep: str) -> EventStream:
    """Keep positive ('pos': p > 0) or non-positive ('neg') events (events.py:314-328)."""
    if keep not in ("pos", "neg"):
        raise ValueError("keep must be 'pos' or 'neg'")
    if stream.polarity is None:
        return stream
    sel = (stream.polarity > 0) == (keep == "pos")
    return EventStream(stream.t[sel], stream.x[sel], stream.y[sel], stream.geometry, stream.polarity[sel])


def window_bounds(t: np.ndarray, delta_t: float, stride: float, t0: float = 0.0) -> List[Tuple[int, int, float]]:
    """(lo, hi, t_start) of every window of slice_stream over sorted times t
    (events.py:331-387): searchsorted with side='left' at both edges, so the
    windows are half-open; trailing empty windows are dropped."""
    if delta_t <= 0:
        raise ValueError("delta_t must be positive")
    if stride <= 0:
        raise ValueError("stride must be positive")
    window = 2.0 * delta_t
    if len(t) == 0:
        return []
    t_last = float(t[-1])
    count = 0
    while t0 + count * stride <= t_last:   # same float sequence as the reference's loop
        count += 1
    starts = np.array([t0 + i * stride for i in range(count)], dtype=np.float64)
    lo = np.searchsorted(t, starts, side="left")
    hi = np.searchsorted(t, starts + window, side="left")
    out = [(int(a), int(b), float(s)) for a, b, s in zip(lo, hi, starts)]
    while out and out[-1][1] == out[-1][0]:
        out.pop()
    return out


def slice_stream(stream: EventStream, delta_t: float, stride: float, t0: float = 0.0) -> List[EventSlice]:
    """Cut a stream into windows of length 2·delta_t (events.py:331-387)."""
    if delta_t <= 0:
        raise ValueError("delta_t must be positive")
    if stride <= 0:
        raise ValueError("stride must be positive")
    if len(stream) == 0:
        return []
    t, x, y, p = stream.t, stream.x, stream.y, stream.polarity
    if np.any(np.diff(t) < 0):
        order = np.argsort(t, kind="stable")
        t, x, y = t[order], x[order], y[order]
        p = p[order] if p is not None else None
    return [EventSlice(t[lo:hi], x[lo:hi], y[lo:hi], start, 2.0 * delta_t, stream.geometry,
                       p[lo:hi] if p is not None else None)
            for lo, hi, start in window_bounds(t, delta_t, stride, t0)]


def _window_starts(t: np.ndarray, stride: float, t0: float) -> np.ndarray:
    """The reference loop's window starts t0 + i·stride while <= t[-1] (events.py:363-368)."""
    t_last = float(t[-1])
    count = 0
    while t0 + count * stride <= t_last:
        count += 1
    return np.array([t0 + i * stride for i in range(count)], dtype=np.float64)


def _predict_stream_device(eng, t, x, y, dt: float, stride: float, t0: float):
    """The windows searched and gathered on the GPU (vkm_window_bounds /
    vkm_predict_windows): the stream crosses PCIe once however much the
    windows overlap."""
    import ctypes as C
    import torch
    from . import _lib
    from ._staging import pinned, widen
    n = len(t)
    dev = torch.device("cuda", eng.device)
    ht = pinned("stream_t", n, np.float64)
    hxy = pinned("stream_xy", 2 * n, np.int32)
    ht[:] = t                                         # plain copies: 16 B/event, no host conversion
    hxy[:n], hxy[n:] = x, y
    td = torch.from_numpy(ht).to(dev, non_blocking=True)
    xyd = torch.from_numpy(hxy).to(dev, non_blocking=True).view(2, n)
    ev = torch.stack([td, xyd[0].double(), xyd[1].double()], 1)   # rows [t, x, y] built on the device
    starts = _window_starts(t, stride, t0)
    nw = len(starts)
    bounds = np.empty((nw, 2), dtype=np.int64)
    torch.cuda.current_stream(eng.device).synchronize()
    _lib.check(eng._lib.vkm_window_bounds(eng._h, C.c_void_p(ev.data_ptr()), n,
                                          starts.ctypes.data_as(C.POINTER(C.c_double)), nw, 2.0 * dt,
                                          bounds.ctypes.data_as(C.POINTER(C.c_int64))))
    while nw and bounds[nw - 1, 1] == bounds[nw - 1, 0]:   # trailing empty windows are dropped
        nw -= 1
    starts, bounds = np.ascontiguousarray(starts[:nw]), np.ascontiguousarray(bounds[:nw])
    sizes = bounds[:, 1] - bounds[:, 0]
    offsets = np.zeros(nw + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    total = int(offsets[-1])
    if total == 0:
        return [(float(s), np.empty((0, 2))) for s in starts]
    flows = torch.empty((total, 2), dtype=torch.float32, device=dev)
    _lib.check(eng._lib.vkm_predict_windows(eng._h, C.c_void_p(ev.data_ptr()), n,
                                            starts.ctypes.data_as(C.POINTER(C.c_double)),
                                            bounds.ctypes.data_as(C.POINTER(C.c_int64)), nw,
                                            C.c_void_p(flows.data_ptr()), None,
                                            C.c_void_p(torch.cuda.current_stream(eng.device).cuda_stream)))
    fh = pinned("flows", 2 * total, np.float32)
    torch.from_numpy(fh).copy_(flows.view(-1))        # pinned D2H
    out = widen(fh).reshape(total, 2)     # one widening pass into the result
    return [(float(s), out[a:b]) for s, a, b in zip(starts, offsets[:-1], offsets[1:])]


def predict_stream(regressor, stream: EventStream, stride: Optional[float] = None, t0: float = 0.0,
                   device_windows: Optional[bool] = None):
    """Per-window normal flow over a whole stream on the B200 path.

    Returns a list of (t_start, flows) with flows (n_window, 2) float64, one
    entry per slice_stream window (empty windows give (0, 2) arrays).  The
    window start is each slice's time origin, like predict_flows on a
    slice_stream slice.  stride defaults to the window (2·delta_t).

    device_windows: search and gather the windows on the GPU (the stream is
    uploaded once, results come back through a pinned buffer); the default
    unless the stream and its windows would take more than
    VKM_STREAM_DEVICE_BYTES (default 16 GiB) of HBM, where the windows go
    through the pipelined host batch instead."""
    from ._staging import pinned, widen
    dt = float(regressor.delta_t)
    if stride is None:
        stride = 2.0 * dt
    g = stream.geometry
    if (g.width, g.height) != (regressor.width, regressor.height):
        raise GeometryError(f"stream geometry {g.width}x{g.height} does not match the estimator's "
                            f"{regressor.width}x{regressor.height}")
    if dt <= 0:
        raise ValueError("delta_t must be positive")
    if stride <= 0:
        raise ValueError("stride must be positive")
    eng = regressor.engine()
    t, x, y = stream.t, stream.x, stream.y
    if len(t) and np.any(np.diff(t) < 0):
        order = np.argsort(t, kind="stable")
        t, x, y = t[order], x[order], y[order]
    if len(t) == 0:
        return []
    if device_windows is None:
        overlap = max(1.0, 2.0 * dt / stride)     # events per window set ≈ overlap · n
        need = len(t) * (24 + overlap * (24 + 8))  # stream + gathered rows + f32 flows
        device_windows = need <= float(os.environ.get("VKM_STREAM_DEVICE_BYTES", 16 << 30))
    if device_windows:
        return _predict_stream_device(eng, t, x, y, dt, stride, t0)
    wins = window_bounds(t, dt, stride, t0)
    if not wins:
        return []
    sizes = np.array([hi - lo for lo, hi, _ in wins], dtype=np.int64)
    offsets = np.zeros(len(wins) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    total = int(offsets[-1])
    if total == 0:
        return [(s, np.empty((0, 2))) for _, _, s in wins]
    ev = pinned("batch_events", 3 * total, np.float64).reshape(total, 3)
    out = pinned("batch_flows", 2 * total, np.float32).reshape(total, 2)
    for (lo, hi, _), o in zip(wins, offsets[:-1]):
        if hi > lo:   # overlapping windows duplicate their shared events
            ev[o:o + hi - lo, 0] = t[lo:hi]
            ev[o:o + hi - lo, 1] = x[lo:hi]
            ev[o:o + hi - lo, 2] = y[lo:hi]
    t_starts = np.array([s for _, _, s in wins], dtype=np.float64)
    eng.predict_batch_host(ev, offsets, t_starts, flows=out)
    res = widen(out)
    return [(s, res[a:b]) for (_, _, s), a, b in zip(wins, offsets[:-1], offsets[1:])]
