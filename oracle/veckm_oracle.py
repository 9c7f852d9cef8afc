"""CPU oracle for the VecKM_flow normal-flow hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `evflow` algorithm
(`/root/reference/pkg/src/evflow`, arXiv 2504.19417).  It exists so that the
B200 path can be checked on the GPU box, where the reference itself is not
available.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline / `--impl reference` arm may import it, and only as the checker or as
the timed CPU baseline — never as the product path.  The product
(`paper_2504_19417_b200`) never imports this file and has no CPU fallback.

Parity pinning: `tests/golden/make_golden.py` runs the *real* reference in the
build container and freezes its outputs under `tests/golden/*.npz`;
`tests/test_oracle_golden.py` asserts that this restatement reproduces them
(bit-exact counts, ulp-level floats).

Every function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/evflow/`).  Floating-point operations are performed in
the same order and precision as the reference so the restatement reproduces
its rounding, not just its mathematics.
"""

from __future__ import annotations

import math
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

_REAL = {"f32": np.float32, "f64": np.float64}
_CPLX = {"f32": np.complex64, "f64": np.complex128}

# --------------------------------------------------------------------------
# Pinned RNG: SplitMix64 + Box-Muller                     (rng.py:22-70)
# --------------------------------------------------------------------------

_U64 = np.uint64
_GOLDEN_GAMMA = _U64(0x9E3779B97F4A7C15)


def splitmix64_stream(seed: int, count: int) -> np.ndarray:
    """k-th output = finalizer(seed + (k+1)*gamma) mod 2**64   (rng.py:22-43)."""
    if count < 0:
        raise ValueError("count must be non-negative")
    state = _U64(seed & 0xFFFFFFFFFFFFFFFF) + np.arange(1, count + 1, dtype=np.uint64) * _GOLDEN_GAMMA
    with np.errstate(over="ignore"):
        z = state
        z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
        z = z ^ (z >> _U64(31))
    return z


def box_muller_normals(seed: int, count: int) -> np.ndarray:
    """Pairs (a, b) of stream outputs -> (r cos 2πu2, r sin 2πu2)   (rng.py:46-70)."""
    npairs = (count + 1) // 2
    raw = splitmix64_stream(seed, 2 * npairs)
    u1 = ((raw[0::2] >> _U64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (raw[1::2] >> _U64(11)).astype(np.float64) * 2.0 ** -53
    radius = np.sqrt(-2.0 * np.log(u1))
    both = np.empty(2 * npairs, dtype=np.float64)
    both[0::2] = radius * np.cos(2.0 * np.pi * u2)
    both[1::2] = radius * np.sin(2.0 * np.pi * u2)
    return both[:count]


@dataclass(frozen=True)
class Freqs:
    """The three f64 frequency vectors (encoder.py:87-112)."""

    T: np.ndarray
    X: np.ndarray
    Y: np.ndarray
    sigma2: float = 25.0

    @property
    def dim(self) -> int:
        return len(self.T)


def make_freqs(dim: int, sigma2: float = 25.0, seeds=(0, 1, 2)) -> Freqs:
    """N(0, sigma2) draws from the pinned stream, one seed per axis (encoder.py:115-124)."""
    s = np.sqrt(sigma2)
    return Freqs(
        box_muller_normals(seeds[0], dim) * s,
        box_muller_normals(seeds[1], dim) * s,
        box_muller_normals(seeds[2], dim) * s,
        float(sigma2),
    )


# --------------------------------------------------------------------------
# Phases                                                  (encoder.py:173-226)
# --------------------------------------------------------------------------


def _cis(args: np.ndarray, cdtype) -> np.ndarray:
    """cos + i sin assembled component-wise (encoder.py:211-217)."""
    out = np.empty(args.shape, dtype=cdtype)
    out.real = np.cos(args)
    out.imag = np.sin(args)
    return out


def spatial_table(fr: Freqs, dx: int, dy: int, precision: str = "f32") -> np.ndarray:
    """table[i, j] = e^{i (i-dx)/dx X} * e^{i (j-dy)/dy Y}, f64 then cast (encoder.py:173-179)."""
    ox = np.arange(-dx, dx + 1, dtype=np.float64) / dx
    oy = np.arange(-dy, dy + 1, dtype=np.float64) / dy
    px = _cis(np.outer(ox, fr.X), np.complex128)
    py = _cis(np.outer(oy, fr.Y), np.complex128)
    return (px[:, None, :] * py[None, :, :]).astype(_CPLX[precision])


def temporal_phases(t_rel: np.ndarray, fr: Freqs, delta_t: float,
                    precision: str = "f32", sign: float = 1.0) -> np.ndarray:
    """a = real(t/δt) (f64 divide then cast); arg = a ⊗ real(sign·T); cis   (encoder.py:220-226)."""
    rd = _REAL[precision]
    a = (t_rel / delta_t).astype(rd)
    return _cis(np.multiply.outer(a, (sign * fr.T).astype(rd)), _CPLX[precision])


# --------------------------------------------------------------------------
# Stage 1: per-pixel grid                                 (encoder.py:229-283)
# --------------------------------------------------------------------------


@dataclass
class Grid:
    """Padded [x][y][D] phase sums and int64 counts with a (dx, dy) zero border
    (encoder.py:182-208)."""

    embed_p: np.ndarray
    count_p: np.ndarray
    dx: int
    dy: int
    width: int
    height: int

    @property
    def embed(self) -> np.ndarray:
        return self.embed_p[self.dx:self.dx + self.width, self.dy:self.dy + self.height]

    @property
    def count(self) -> np.ndarray:
        return self.count_p[self.dx:self.dx + self.width, self.dy:self.dy + self.height]


def accumulate(t_rel, x, y, width: int, height: int, dx: int, dy: int, fr: Freqs,
               delta_t: float, precision: str = "f32") -> Grid:
    """Stable sort by padded pixel key, then per-pixel sum in time order
    (encoder.py:229-283; the single-worker branch — the threaded branch is
    bitwise identical by construction, encoder.py:272-282)."""
    stride_x = height + 2 * dy                 # padded column height (encoder.py:248)
    n_cells = (width + 2 * dx) * stride_x
    D = fr.dim
    embed = np.zeros((n_cells, D), dtype=_CPLX[precision])
    count = np.zeros(n_cells, dtype=np.int64)
    n = len(t_rel)
    if n:
        key = (np.asarray(x, np.int64) + dx) * stride_x + (np.asarray(y, np.int64) + dy)
        perm = np.argsort(key, kind="stable")
        ks = key[perm]
        count[:] = np.bincount(key, minlength=n_cells)
        run_start = np.flatnonzero(np.concatenate(([True], ks[1:] != ks[:-1])))
        ph = temporal_phases(np.asarray(t_rel, np.float64)[perm], fr, delta_t, precision)
        embed[ks[run_start]] = np.add.reduceat(ph, run_start, axis=0)
    shape = (width + 2 * dx, stride_x)
    return Grid(embed.reshape(shape + (D,)), count.reshape(shape), dx, dy, width, height)


def accumulate_near(t_rel, x, y, width: int, height: int, dx: int, dy: int, fr: Freqs,
                    delta_t: float, qx, qy, precision: str = "f32", chunk: int = 1 << 18) -> Grid:
    """`accumulate` restricted to the pixels inside the windows of the queries
    (qx, qy), in bounded memory — for at-size checks of large slices on a
    strided query subset.  A pixel's sum depends only on its own events in
    time order (encoder.py:255-267), so every pixel a query window touches
    gets exactly the value `accumulate` gives it; counts are complete
    (np.bincount over all events, encoder.py:259).  Phases are evaluated in
    chunks of whole pixel runs, so np.add.reduceat sees the same runs."""
    stride_x = height + 2 * dy
    n_cells = (width + 2 * dx) * stride_x
    D = fr.dim
    embed = np.zeros((n_cells, D), dtype=_CPLX[precision])
    x = np.asarray(x, np.int64)
    y = np.asarray(y, np.int64)
    key = (x + dx) * stride_x + (y + dy)
    count = np.bincount(key, minlength=n_cells).astype(np.int64)
    need = np.zeros((width + 2 * dx, stride_x), dtype=bool)
    for cx, cy in zip(np.asarray(qx, np.int64), np.asarray(qy, np.int64)):
        need[cx:cx + 2 * dx + 1, cy:cy + 2 * dy + 1] = True
    sel = np.flatnonzero(need.ravel()[key])               # time order kept
    if len(sel):
        ks_all = key[sel]
        perm = np.argsort(ks_all, kind="stable")
        ks = ks_all[perm]
        tr = np.asarray(t_rel, np.float64)[sel][perm]
        run_start = np.flatnonzero(np.concatenate(([True], ks[1:] != ks[:-1])))
        bounds = list(run_start[::max(1, len(run_start) * chunk // max(len(ks), 1))]) + [len(ks)]
        bounds = sorted(set(int(b) for b in bounds))
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            rs = run_start[(run_start >= lo) & (run_start < hi)]
            ph = temporal_phases(tr[lo:hi], fr, delta_t, precision)
            embed[ks[rs]] = np.add.reduceat(ph, rs - lo, axis=0)
    shape = (width + 2 * dx, stride_x)
    return Grid(embed.reshape(shape + (D,)), count.reshape(shape), dx, dy, width, height)


# --------------------------------------------------------------------------
# Stage 2: windowed, phase-weighted pooling + de-phase    (encoder.py:312-346)
# --------------------------------------------------------------------------


def pool(grid: Grid, table: np.ndarray, qt, qx, qy, fr: Freqs, delta_t: float,
         precision: str = "f32") -> Tuple[np.ndarray, np.ndarray]:
    """acc = Σ_i Σ_j G[qx+i, qy+j] ⊙ table[i, j] (i outer, j inner, complex
    product then add, encoder.py:331-336); emb = conj-phase ⊙ acc / max(cnt,1)
    (encoder.py:344-345).  Empty neighbourhoods are returned, not raised
    (`allow_empty=True`, the predict_flows path, flow.py:178-187)."""
    qx = np.asarray(qx, np.int64)
    qy = np.asarray(qy, np.int64)
    nq = len(qx)
    cd = _CPLX[precision]
    acc = np.zeros((nq, fr.dim), dtype=cd)
    cnt = np.zeros(nq, dtype=np.int64)
    prod = np.empty((nq, fr.dim), dtype=cd)
    for i in range(2 * grid.dx + 1):
        col = qx + i
        for j in range(2 * grid.dy + 1):
            row = qy + j
            np.multiply(grid.embed_p[col, row], table[i, j], out=prod)
            acc += prod
            cnt += grid.count_p[col, row]
    back = temporal_phases(np.asarray(qt, np.float64), fr, delta_t, precision, sign=-1.0)
    emb = back * acc / np.maximum(cnt, 1)[:, None].astype(_REAL[precision])
    return emb, cnt


def pool_threaded(grid, table, qt, qx, qy, fr, delta_t, precision="f32", threads=1):
    """Equal query chunks over a thread pool, as the reference's encode()
    does (encoder.py:398-411); results are bitwise equal to `pool`."""
    nq = len(qx)
    if threads <= 1 or nq < 1024:
        return pool(grid, table, qt, qx, qy, fr, delta_t, precision)
    emb = np.empty((nq, fr.dim), dtype=_CPLX[precision])
    cnt = np.empty(nq, dtype=np.int64)
    cuts = np.linspace(0, nq, threads + 1).astype(int)

    def work(lo_hi):
        lo, hi = lo_hi
        e, c = pool(grid, table, qt[lo:hi], qx[lo:hi], qy[lo:hi], fr, delta_t, precision)
        emb[lo:hi] = e
        cnt[lo:hi] = c

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, zip(cuts[:-1], cuts[1:])))
    return emb, cnt


def direct_encode(t_rel, x, y, q: int, dx: int, dy: int, fr: Freqs, delta_t: float):
    """Quadratic f64 summation over the query's window (encoder.py:415-440)."""
    t_rel = np.asarray(t_rel, np.float64)
    x = np.asarray(x, np.int64)
    y = np.asarray(y, np.int64)
    sel = (np.abs(x - x[q]) <= dx) & (np.abs(y - y[q]) <= dy)
    args = (np.outer((t_rel[sel] - t_rel[q]) / delta_t, fr.T)
            + np.outer((x[sel] - x[q]) / dx, fr.X)
            + np.outer((y[sel] - y[q]) / dy, fr.Y))
    return np.exp(1j * args).mean(axis=0), int(sel.sum())


# --------------------------------------------------------------------------
# Flow head                                               (flow.py:92-106)
# --------------------------------------------------------------------------


def to_features(emb: np.ndarray) -> np.ndarray:
    """[Re; Im] along the last axis (flow.py:92-95)."""
    return np.concatenate([emb.real, emb.imag], axis=-1)


def mlp(w1, b1, w2, b2, feats) -> np.ndarray:
    """W2·relu(W1·f + b1) + b2 via BLAS matmuls (flow.py:98-106)."""
    h = np.maximum(feats @ w1.T + b1, 0.0)
    return h @ w2.T + b2


# --------------------------------------------------------------------------
# Host contract: validation and slicing                  (validation.py:10-65)
# --------------------------------------------------------------------------


def validate(X, width: int, height: int):
    """(n,3) [t,x,y] -> (t f64, x i32, y i32) with the reference's checks
    (validation.py:10-37)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] < 3:
        raise ValueError(f"expected an (n, 3) array of [t, x, y], got shape {X.shape}")
    if not np.all(np.isfinite(X[:, :3])):
        raise ValueError("event array contains non-finite values")
    t, xf, yf = X[:, 0], X[:, 1], X[:, 2]
    if np.any(t < 0):
        raise ValueError("timestamps must be non-negative seconds")
    if np.any(xf != np.round(xf)) or np.any(yf != np.round(yf)):
        raise ValueError("pixel coordinates must be integer-valued")
    xi = xf.astype(np.int32)
    yi = yf.astype(np.int32)
    ok = (xi >= 0) & (xi < width) & (yi >= 0) & (yi < height)
    if not np.all(ok):
        b = int(np.flatnonzero(~ok)[0])
        raise ValueError(f"event {b} at ({xi[b]}, {yi[b]}) outside geometry {width}x{height}")
    return t, xi, yi


def make_slice(X, width: int, height: int, window: float):
    """Stable time sort when unsorted; t_start = first; strict f64 span check
    (validation.py:49-65).  Returns (t, x, y, t_start)."""
    t, x, y = validate(X, width, height)
    if len(t) and np.any(np.diff(t) < 0):
        o = np.argsort(t, kind="stable")
        t, x, y = t[o], x[o], y[o]
    t0 = float(t[0]) if len(t) else 0.0
    if len(t) and float(t[-1]) - t0 > window:
        raise ValueError(
            f"events span {float(t[-1]) - t0:.6f}s which exceeds the slice "
            f"window {window:.6f}s; split the stream into slices first")
    return t, x, y, t0


# --------------------------------------------------------------------------
# End-to-end estimator semantics          (estimators.py:89-95, 192-206; flow.py:155-197)
# --------------------------------------------------------------------------


def predict(X, width, height, dx, dy, delta_t, fr: Freqs, w1, b1, w2, b2,
            precision="f32", threads=1, return_counts=False):
    """NormalFlowRegressor.predict: (n,2) float64 in time-sorted order with NaN
    rows for empty neighbourhoods (estimators.py:192-206, flow.py:155-197)."""
    t, x, y, t0 = make_slice(X, width, height, 2.0 * delta_t)
    t_rel = t - t0                                    # rebase_slice (events.py:390-407)
    out = np.full((len(t), 2), np.nan)
    cnt = np.zeros(len(t), dtype=np.int64)
    if len(t):
        tab = spatial_table(fr, dx, dy, precision)
        g = accumulate(t_rel, x, y, width, height, dx, dy, fr, delta_t, precision)
        emb, cnt = pool_threaded(g, tab, t_rel, x, y, fr, delta_t, precision, threads)
        ok = cnt > 0
        if ok.any():
            out[ok] = mlp(w1, b1, w2, b2, to_features(emb[ok]))
    return (out, cnt) if return_counts else out


def encode_features(X, width, height, dx, dy, delta_t, fr: Freqs, precision="f32", threads=1):
    """LocalEventEncoder.transform: (n, 2D) features (estimators.py:89-95).
    Raises on empty neighbourhoods like encode() (encoder.py:337-343)."""
    t, x, y, t0 = make_slice(X, width, height, 2.0 * delta_t)
    t_rel = t - t0
    if len(t) == 0:
        return np.empty((0, 2 * fr.dim), dtype=_REAL[precision])
    tab = spatial_table(fr, dx, dy, precision)
    g = accumulate(t_rel, x, y, width, height, dx, dy, fr, delta_t, precision)
    emb, cnt = pool_threaded(g, tab, t_rel, x, y, fr, delta_t, precision, threads)
    if np.any(cnt == 0):
        raise ValueError("empty neighbourhood")
    return to_features(emb)


def pooled_all_pixels(grid: Grid, table: np.ndarray):
    """Window sums (before de-phasing) at every pixel: the quantity the GPU's
    pool kernel stores.  Restates the acc/cnt loop of encoder.py:331-336 with
    every in-image pixel as a query."""
    xs, ys = np.meshgrid(np.arange(grid.width), np.arange(grid.height), indexing="ij")
    qx, qy = xs.ravel(), ys.ravel()
    cd = grid.embed_p.dtype
    acc = np.zeros((len(qx), grid.embed_p.shape[-1]), dtype=cd)
    cnt = np.zeros(len(qx), dtype=np.int64)
    for i in range(2 * grid.dx + 1):
        for j in range(2 * grid.dy + 1):
            acc += grid.embed_p[qx + i, qy + j] * table[i, j]
            cnt += grid.count_p[qx + i, qy + j]
    shape = (grid.width, grid.height)
    return acc.reshape(shape + (-1,)), cnt.reshape(shape)


def synth_uniform_noise(n: int, width: int, height: int, seed: int = 0, window: float = 0.032):
    """Uniform-noise scene as bench.synth_workload draws it (bench.py:187-190,
    209-213): t~U[0,window), x,y uniform integers, stable-sorted by t."""
    rng = np.random.default_rng(seed)
    t = rng.uniform(0.0, window, size=n)
    x = rng.integers(0, width, size=n)
    y = rng.integers(0, height, size=n)
    o = np.argsort(t, kind="stable")
    return np.stack([t[o], x[o].astype(np.float64), y[o].astype(np.float64)], axis=1)
