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
