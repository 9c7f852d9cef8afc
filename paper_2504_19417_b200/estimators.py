"""Drop-in scikit-learn estimators backed by the B200 kernels.

Same constructor parameters, `fit` / `predict` / `transform` semantics, output
layout and error types as the reference adapters (estimators.py:30-206 under
/root/reference/pkg/src/evflow/); two additive keyword parameters select the
device and the MLP execution mode.  All per-event work runs in libveckm.so;
there is no CPU fallback.
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Union

import numpy as np
from sklearn.base import BaseEstimator, TransformerMixin
from sklearn.exceptions import NotFittedError

from ._staging import concat_rows, pinned, widen
from .engine import EngineCache, FlowEngine, predict_multi_host
from .errors import DimensionMismatchError, EmptyNeighborhoodError
from .validation import block_from_array, check_events
from .weights import MlpWeights, as_weights, generate_bases, load_weights

# LocalEventEncoder handles: per host thread, at most 4 live (EngineCache)
_ENGINES = EngineCache()


def _check_config(delta_t, delta_x, delta_y, embed_dim, sigma2, seeds, precision):
    """EncoderConfig.__post_init__ checks (encoder.py:60-72)."""
    if delta_t <= 0:
        raise ValueError("delta_t must be positive")
    if delta_x < 1 or delta_y < 1:
        raise ValueError("pixel radii must be >= 1")
    if embed_dim < 1:
        raise ValueError("embed_dim must be >= 1")
    if sigma2 <= 0:
        raise ValueError("sigma2 must be positive")
    if precision not in ("f32", "f64"):
        raise ValueError("precision must be one of ['f32', 'f64']")
    if len(tuple(seeds)) != 3:
        raise ValueError("seeds must be a triple (time, x, y)")


def _engine(key, factory) -> FlowEngine:
    return _ENGINES.get(key, factory)


class LocalEventEncoder(TransformerMixin, BaseEstimator):
    """Per-event neighbourhood features [Re; Im] (estimators.py:30-95)."""

    def __init__(self, delta_t: float = 0.016, delta_x: int = 10, delta_y: int = 10, embed_dim: int = 64,
                 sigma2: float = 25.0, seeds: tuple = (0, 1, 2), precision: str = "f32", width: int = 640,
                 height: int = 480, threads: int = 1, device: int = 0):
        self.delta_t = delta_t
        self.delta_x = delta_x
        self.delta_y = delta_y
        self.embed_dim = embed_dim
        self.sigma2 = sigma2
        self.seeds = seeds
        self.precision = precision
        self.width = width
        self.height = height
        self.threads = threads
        self.device = device

    def fit(self, X=None, y=None):
        _check_config(self.delta_t, self.delta_x, self.delta_y, self.embed_dim, self.sigma2, self.seeds,
                      self.precision)
        if X is not None:
            check_events(X, self.width, self.height)
        self.bases_ = generate_bases(self.embed_dim, self.sigma2, tuple(self.seeds))
        return self

    def transform(self, X) -> np.ndarray:
        if not hasattr(self, "bases_"):
            raise NotFittedError("call fit before transform")
        _check_config(self.delta_t, self.delta_x, self.delta_y, self.embed_dim, self.sigma2, self.seeds,
                      self.precision)
        block = block_from_array(X, self.width, self.height, 2.0 * self.delta_t)
        f64 = self.precision == "f64"   # complex128 grid, float64 features (encoder.py:37-38)
        if len(block) == 0:
            return np.empty((0, 2 * self.embed_dim), dtype=np.float64 if f64 else np.float32)
        b = self.bases_
        key = ("enc", self.width, self.height, self.delta_x, self.delta_y, float(self.delta_t), self.device,
               b.time_freqs.tobytes(), b.x_freqs.tobytes(), b.y_freqs.tobytes())
        eng = _engine(key, lambda: FlowEngine(self.width, self.height, self.delta_x, self.delta_y, self.delta_t,
                                              b, None, self.device))
        encode = eng.encode_host_f64 if f64 else eng.encode_host
        feats, counts = encode(block.events, block.t_start, return_counts=True)
        if np.any(counts == 0):  # encoder.py:337-343
            bad = np.flatnonzero(counts == 0)
            raise EmptyNeighborhoodError(f"{len(bad)} queries have empty neighborhoods "
                                         f"(first at batch position {bad[0]})")
        return feats


class NormalFlowRegressor(BaseEstimator):
    """Per-event normal flow (estimators.py:98-206) on the B200 path."""

    def __init__(self, delta_t: float = 0.016, delta_x: int = 10, delta_y: int = 10, embed_dim: int = 64,
                 sigma2: float = 25.0, seeds: tuple = (0, 1, 2), precision: str = "f32", width: int = 640,
                 height: int = 480, threads: int = 1, hidden: int = 128, epochs: int = 300, batch_size: int = 512,
                 learning_rate: float = 1e-3, margin_weight: float = 0.1, random_state: int = 0,
                 weights: Union[MlpWeights, str, None] = None, device: int = 0, mlp_mode: str = "auto"):
        self.delta_t = delta_t
        self.delta_x = delta_x
        self.delta_y = delta_y
        self.embed_dim = embed_dim
        self.sigma2 = sigma2
        self.seeds = seeds
        self.precision = precision
        self.width = width
        self.height = height
        self.threads = threads
        self.hidden = hidden
        self.epochs = epochs
        self.batch_size = batch_size
        self.learning_rate = learning_rate
        self.margin_weight = margin_weight
        self.random_state = random_state
        self.weights = weights
        self.device = device
        self.mlp_mode = mlp_mode

    def __getstate__(self):
        """Picklable / deep-copyable after use, like the reference estimator:
        the libveckm handles (`_engine_cache`, `_device_engines`) hold a CDLL
        and device memory, so they are dropped and rebuilt on the next call."""
        state = dict(super().__getstate__())
        state.pop("_engine_cache", None)
        state.pop("_device_engines", None)
        return state

    def _resolve_pretrained(self) -> Optional[MlpWeights]:
        if self.weights is None:
            return None
        if isinstance(self.weights, str):
            return load_weights(self.weights)
        return as_weights(self.weights)

    def fit(self, X, y):
        pretrained = self._resolve_pretrained()
        if pretrained is not None:
            self.weights_ = pretrained
            return self
        # estimators.py:171-190: train the head on the GPU (training.train_head)
        from .training import TrainConfig, train_head
        from .validation import check_flow_array
        _check_config(self.delta_t, self.delta_x, self.delta_y, self.embed_dim, self.sigma2, self.seeds,
                      self.precision)
        slices = X if isinstance(X, (list, tuple)) else [X]
        targets = y if isinstance(y, (list, tuple)) else [y]
        if len(slices) != len(targets):
            raise ValueError("X and y must pair one flow array per slice")
        dataset = []
        for arr, flows in zip(slices, targets):
            blk = block_from_array(arr, self.width, self.height, 2.0 * self.delta_t)
            dataset.append((arr, check_flow_array(flows, len(blk))))
        tc = TrainConfig(hidden=self.hidden, epochs=self.epochs, batch_size=self.batch_size,
                         learning_rate=self.learning_rate, margin_weight=self.margin_weight, seed=self.random_state)
        bases = generate_bases(self.embed_dim, self.sigma2, tuple(self.seeds))
        self.weights_ = train_head(dataset, self.width, self.height, self.delta_x, self.delta_y, self.delta_t,
                                   self.embed_dim, tc, bases, self.precision, self.device)
        return self

    def _ready(self) -> MlpWeights:
        if not hasattr(self, "weights_"):
            pretrained = self._resolve_pretrained()
            if pretrained is None:
                raise NotFittedError("call fit or supply pretrained weights")
            self.weights_ = pretrained
        _check_config(self.delta_t, self.delta_x, self.delta_y, self.embed_dim, self.sigma2, self.seeds,
                      self.precision)
        w = self.weights_
        if w.embed_dim != self.embed_dim:  # flow.py:167-170
            raise DimensionMismatchError(f"weights expect D={w.embed_dim} but config has D={self.embed_dim}")
        return w

    def engine(self) -> FlowEngine:
        """The cached libveckm handle for this estimator's geometry and head."""
        w = self._ready()
        key = (self.width, self.height, self.delta_x, self.delta_y, float(self.delta_t), self.device,
               self.mlp_mode)
        cached = getattr(self, "_engine_cache", None)
        if cached is not None and cached[0] == key and cached[1] is w:
            return cached[2]
        eng = FlowEngine(self.width, self.height, self.delta_x, self.delta_y, self.delta_t, w.bases, w,
                         self.device, self.mlp_mode)
        self._engine_cache = (key, w, eng)
        return eng

    def predict(self, X) -> np.ndarray:
        """(n, 2) float64 flows in pixels/s; rows in stable time-sorted order
        (input order for sorted input); NaN rows for empty neighbourhoods."""
        eng = self.engine()
        if self.precision == "f32" and isinstance(X, np.ndarray):
            # one host pass validates and packs a sorted, valid slice for the
            # upload (vkm_predict_host_checked); anything else - errors to
            # raise, unsorted rows, small slices - takes the path below
            flows = eng.predict_host_checked(X, 2.0 * self.delta_t)
            if flows is not None:
                return flows
        block = block_from_array(X, self.width, self.height, 2.0 * self.delta_t)
        if len(block) == 0:
            return np.full((0, 2), np.nan)
        if self.precision == "f64":   # f64 grid, features and head (encoder.py:37-38, flow.py:98-106)
            return eng.predict_host_f64(block.events, block.t_start)
        return eng.predict_host_wide(block.events, block.t_start)

    def engines(self, devices: Sequence[int]) -> List[FlowEngine]:
        """One cached libveckm handle per entry of `devices` (a device listed
        twice gets two handles: two pipelines on one GPU)."""
        w = self._ready()
        cache = self.__dict__.setdefault("_device_engines", {})
        out, seen = [], {}
        for d in devices:
            d = int(d)
            k = seen[d] = seen.get(d, -1) + 1
            key = (self.width, self.height, self.delta_x, self.delta_y, float(self.delta_t), d, k, self.mlp_mode)
            hit = cache.get(key)
            if hit is None or hit[0] is not w:
                hit = (w, FlowEngine(self.width, self.height, self.delta_x, self.delta_y, self.delta_t, w.bases, w, d,
                                     self.mlp_mode))
                cache[key] = hit
            out.append(hit[1])
        return out

    def predict_slices(self, slices: Sequence, devices: Optional[Sequence[int]] = None) -> List[np.ndarray]:
        """Additive API: many independent slices, one result
        per slice, each with `predict`'s semantics.  The slices are validated
        on the host, packed into one page-locked buffer and streamed through
        vkm_predict_batch_host, which overlaps the copies of neighbouring
        slices with the kernels.  `devices` (e.g. [0, 1, ..., 7]) shards the
        slices over several GPUs, contiguous ranges of equal event counts, one
        host thread per GPU (vkm_predict_multi_host; no collective)."""
        eng = self.engine()
        if self.precision == "f64":   # one slice per call on the f64 path
            return [self.predict(X) for X in slices]
        blocks = [block_from_array(X, self.width, self.height, 2.0 * self.delta_t) for X in slices]
        sizes = [len(b) for b in blocks]
        total = int(sum(sizes))
        if total == 0:
            return [np.full((0, 2), np.nan) for _ in blocks]
        ev = pinned("batch_events", 3 * total, np.float64).reshape(total, 3)
        out = pinned("batch_flows", 2 * total, np.float32).reshape(total, 2)
        offsets = np.zeros(len(blocks) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        concat_rows([b.events for b in blocks if len(b)], ev)
        t_starts = np.array([b.t_start if len(b) else 0.0 for b in blocks], dtype=np.float64)
        if devices is not None and len(devices) > 1:
            predict_multi_host(self.engines(devices), ev, offsets, t_starts, flows=out)
        else:
            (self.engines(devices)[0] if devices else eng).predict_batch_host(ev, offsets, t_starts, flows=out)
        res = widen(out)   # results leave the reused staging buffer
        return [res[lo:hi] for lo, hi in zip(offsets[:-1], offsets[1:])]


def _stream_predict(self, stream, stride=None, t0: float = 0.0):
    """Per-window flows over an EventStream (stream.slice_stream windows, the
    window start as each slice's time origin), all windows in one pipelined
    host batch.  Returns [(t_start, (n_i, 2) float64)]."""
    from .stream import predict_stream
    return predict_stream(self, stream, stride, t0)


NormalFlowRegressor.predict_stream = _stream_predict
