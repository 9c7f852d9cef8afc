"""Multi-GPU work division (one process per GPU, torch.distributed plumbing).

Two cases:

* Independent slices (config 4): contiguous slice ranges per rank, no
  data-path collective.  `slice_range` / `shard_slices`.
* One oversized slice (config 5): horizontal row strips balanced by event
  count.  A rank owns the pixels of rows [lo, hi) and receives the events of
  rows [lo - δy, hi + δy) (event-halo duplication): every window of an owned
  pixel then lies inside the rank's sub-grid, so no grid halo exchange is
  needed after the partition, only the partition itself and the gather of the
  owned flows.  The time origin stays the global slice start, so every event's
  phase is bit-identical to the unsplit slice; the spatial modulation tables
  are shift-invariant (modulation and demodulation cancel), so a strip's
  pooled values equal the full slice's up to fp32 rounding.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np


def slice_range(n_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced share of [0, n_items) for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def shard_slices(slices: Sequence, rank: int, world: int) -> List:
    return [slices[i] for i in slice_range(len(slices), rank, world)]


@dataclass(frozen=True)
class Strip:
    """Rows [lo, hi) owned; events of rows [in_lo, in_hi) are this strip's input."""

    lo: int
    hi: int
    in_lo: int
    in_hi: int

    @property
    def height(self) -> int:
        return self.in_hi - self.in_lo


def row_strips(row_counts: np.ndarray, world: int, delta_y: int) -> List[Strip]:
    """Split rows into `world` strips of about equal owned-event count (at least
    one row each), each extended by a δy-row event halo clipped to the image."""
    H = len(row_counts)
    if world < 1 or world > H:
        raise ValueError("need 1 <= world <= number of rows")
    csum = np.concatenate([[0], np.cumsum(np.asarray(row_counts, dtype=np.int64))])
    total = csum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        c = int(np.searchsorted(csum, target, side="left"))
        c = min(max(c, cuts[-1] + 1), H - (world - r))
        cuts.append(c)
    cuts.append(H)
    return [Strip(lo, hi, max(0, lo - delta_y), min(H, hi + delta_y)) for lo, hi in zip(cuts[:-1], cuts[1:])]


@dataclass
class StripEvents:
    """One strip's input: events (shifted to strip-local y) in time order,
    the global index of each, and which of them the strip owns."""

    strip: Strip
    events: np.ndarray      # (m, 3) float64 [t, x, y - in_lo]
    index: np.ndarray       # (m,) int64 global row of each event
    owned: np.ndarray       # (m,) bool


def strip_events(events: np.ndarray, strip: Strip) -> StripEvents:
    """Select the events feeding `strip` from a validated, time-sorted (n, 3)
    slice; the selection keeps time order (so per-pixel sums keep the
    reference's summation order)."""
    y = events[:, 2]
    sel = np.flatnonzero((y >= strip.in_lo) & (y < strip.in_hi))
    sub = events[sel].copy()
    sub[:, 2] -= strip.in_lo
    owned = (events[sel, 2] >= strip.lo) & (events[sel, 2] < strip.hi)
    return StripEvents(strip, sub, sel.astype(np.int64), owned)


def assemble(n: int, parts: Sequence[StripEvents], flows_parts: Sequence[np.ndarray],
             counts_parts: Optional[Sequence[np.ndarray]] = None):
    """Scatter the owned rows of each strip's result into the global order."""
    flows = np.full((n, 2), np.nan, dtype=np.float32)
    counts = np.zeros(n, dtype=np.int32) if counts_parts is not None else None
    seen = np.zeros(n, dtype=np.int32)
    for i, (se, f) in enumerate(zip(parts, flows_parts)):
        flows[se.index[se.owned]] = f[se.owned]
        seen[se.index[se.owned]] += 1
        if counts is not None:
            counts[se.index[se.owned]] = counts_parts[i][se.owned]
    if np.any(seen != 1):
        raise RuntimeError("strip partition does not own every event exactly once")
    return (flows, counts) if counts is not None else flows


def predict_spatial(engine_factory, events: np.ndarray, t_start: float, width: int, height: int, delta_y: int,
                    world: int = 1, rank: int = 0, group=None, return_counts: bool = False):
    """Row-strip split of one slice over `world` ranks (torch.distributed when
    world > 1).  `engine_factory(strip_height)` returns a FlowEngine-like object
    with `predict_host(events, t_start, return_counts=True)`.  Rank 0 returns
    the assembled (n, 2) flows (input row order); other ranks return None."""
    rows = np.bincount(events[:, 2].astype(np.int64), minlength=height)
    strips = row_strips(rows, world, delta_y)
    mine = [r for r in range(len(strips)) if r % world == rank]
    parts, fl, ct = [], [], []
    for r in mine:
        se = strip_events(events, strips[r])
        eng = engine_factory(strips[r].height)
        f, c = eng.predict_host(se.events, t_start, return_counts=True)
        parts.append(se)
        fl.append(f)
        ct.append(c)
    if world > 1:
        import torch.distributed as dist
        payload = [(p.strip, p.index[p.owned], f[p.owned], c[p.owned]) for p, f, c in zip(parts, fl, ct)]
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(payload, gathered, dst=0, group=group)
        if rank != 0:
            return None
        flows = np.full((len(events), 2), np.nan, dtype=np.float32)
        counts = np.zeros(len(events), dtype=np.int32)
        seen = np.zeros(len(events), dtype=np.int32)
        for plist in gathered:
            for _, idx, f, c in plist:
                flows[idx] = f
                counts[idx] = c
                seen[idx] += 1
        if np.any(seen != 1):
            raise RuntimeError("strip partition does not own every event exactly once")
        return (flows, counts) if return_counts else flows
    out = assemble(len(events), parts, fl, ct)
    return out if return_counts else out[0]


def predict_strips_host(make_engine, events: np.ndarray, t_start: float, height: int, delta_y: int,
                        devices: Sequence[int], return_counts: bool = False):
    """One oversized slice over several GPUs from one process
    (vkm_predict_strips_host): row strips of about equal event counts with a
    δy-row event halo, strip i on a handle made by make_engine(strip_height,
    devices[i]) and its own host thread; flows (n, 2) f32 in input order."""
    import ctypes as C
    from . import _lib
    ev = np.ascontiguousarray(events, dtype=np.float64)
    n = len(ev)
    y = ev[:, 2]
    rows = np.bincount(np.clip(y, 0, height - 1).astype(np.int64), minlength=height)[:height] if n else \
        np.zeros(height, dtype=np.int64)
    strips = row_strips(rows, len(devices), delta_y)
    engines = [make_engine(st.in_hi - st.in_lo, d) for st, d in zip(strips, devices)]
    cuts = np.array([st.lo for st in strips] + [strips[-1].hi], dtype=np.int32)
    hs = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
    flows = np.empty((n, 2), dtype=np.float32)
    counts = np.empty(n, dtype=np.int32) if return_counts else None
    _lib.check(engines[0]._lib.vkm_predict_strips_host(hs, len(engines), cuts.ctypes.data, ev.ctypes.data, n,
                                                       float(t_start), flows.ctypes.data,
                                                       counts.ctypes.data if counts is not None else None))
    return (flows, counts) if return_counts else flows


def _is_gloo(group=None) -> bool:
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _send(t, dst, group=None):
    import torch.distributed as dist
    dist.send(t.cpu() if _is_gloo(group) else t, dst, group=group)


def _recv(shape, dtype, src, device, group=None):
    import torch
    import torch.distributed as dist
    if _is_gloo(group):
        buf = torch.empty(shape, dtype=dtype)
        dist.recv(buf, src, group=group)
        return buf.to(device)
    buf = torch.empty(shape, dtype=dtype, device=device)
    dist.recv(buf, src, group=group)
    return buf


def predict_spatial_device(make_engine, events, t_start: float, width: int, height: int, delta_y: int,
                           world: int = 1, rank: int = 0, group=None, device=None):
    """Device-resident row-strip split of one oversized slice (SURVEY.md §8e,
    config 5): the data path never leaves the GPUs.

    Rank 0 holds the slice as a CUDA (n, 3) float64 tensor (other ranks pass
    None).  Rank 0 builds the row histogram on its GPU and the strips on the
    host (a few hundred integers, broadcast); for every rank it selects the
    strip's events plus the δy-row halo with vkm_select_rows (stable, rows
    rebased, owned flags) and sends them over NCCL (NVLink peer-to-peer on an
    NVSwitch box).  Each rank runs its strip through `make_engine(strip_height)`
    (a FlowEngine) on its own GPU with the global t_start, so every phase is
    bit-identical to the unsplit slice; only the flows travel back (rank 0
    kept the indices and owned flags) and vkm_scatter_rows puts the owned
    rows into slice order on GPU 0.  Returns the (n, 2) float32 flows tensor
    on rank 0, None elsewhere.  (gloo groups stage the messages through host
    memory, for CPU-only plumbing tests.)"""
    import ctypes as C
    import torch
    import torch.distributed as dist
    from . import _lib

    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    distributed = world > 1
    if rank == 0:
        n = int(events.shape[0])
        rows = torch.bincount(events[:, 2].to(torch.int64), minlength=height).cpu().numpy()
        strips = row_strips(rows, world, delta_y)
        hdr = [strips, n]
    else:
        hdr = [None, None]
    if distributed:
        dist.broadcast_object_list(hdr, src=0, group=group)
    strips, n = hdr
    mine = strips[rank]
    eng = make_engine(mine.height)
    lib = _lib.load()
    stream = torch.cuda.current_stream(device)

    def select(r):
        s = strips[r]
        m = C.c_int64()
        out = torch.empty((n, 3), dtype=torch.float64, device=device)
        idx = torch.empty(n, dtype=torch.int64, device=device)
        own = torch.empty(n, dtype=torch.uint8, device=device)
        stream.synchronize()
        _lib.check(lib.vkm_select_rows(eng._h, C.c_void_p(events.data_ptr()), n, s.in_lo, s.in_hi, s.lo, s.hi,
                                       C.c_void_p(out.data_ptr()), C.c_void_p(idx.data_ptr()),
                                       C.c_void_p(own.data_ptr()), C.byref(m)))
        k = int(m.value)
        return out[:k].contiguous(), idx[:k], own[:k]

    parts = {}
    if rank == 0:
        for r in range(world):
            ev_r, idx_r, own_r = select(r)
            parts[r] = (idx_r, own_r)
            if r == 0:
                my_ev = ev_r
            else:
                _send(torch.tensor([ev_r.shape[0]], dtype=torch.int64, device=device), r, group)
                if ev_r.shape[0]:
                    _send(ev_r, r, group)
    else:
        k = int(_recv((1,), torch.int64, 0, device, group).item())
        my_ev = _recv((k, 3), torch.float64, 0, device, group) if k else torch.empty((0, 3), dtype=torch.float64,
                                                                                        device=device)
    flows_mine = eng.predict_device(my_ev, t_start) if my_ev.shape[0] else torch.empty((0, 2), dtype=torch.float32,
                                                                                        device=device)
    if rank != 0:
        if flows_mine.shape[0]:
            _send(flows_mine, 0, group)
        return None
    out = torch.full((n, 2), float("nan"), dtype=torch.float32, device=device)
    for r in range(world):
        idx_r, own_r = parts[r]
        f_r = flows_mine if r == 0 else (_recv((idx_r.shape[0], 2), torch.float32, r, device, group)
                                         if idx_r.shape[0] else None)
        if f_r is not None and idx_r.shape[0]:
            _lib.check(lib.vkm_scatter_rows(eng._h, C.c_void_p(f_r.data_ptr()), C.c_void_p(idx_r.data_ptr()),
                                            C.c_void_p(own_r.data_ptr()), idx_r.shape[0], 2,
                                            C.c_void_p(out.data_ptr()), C.c_void_p(stream.cuda_stream)))
    return out
