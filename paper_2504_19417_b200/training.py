"""Head training on the GPU: `train_head` (flow.py:320-402) with the data set's
features encoded by the B200 encoder and the mini-batch Adam steps run by
libveckm (k_train.cu, float64).

The control flow is the reference's, line for line: one numpy
`default_rng(seed)` drives the validation split and the per-epoch
permutations, the margin defaults to 0.05·mean|u|, the weights start from
`init_weights(seed)`, and the weights with the best validation loss are
returned (the initial weights included).  Only the arithmetic moves to the
GPU, so a run follows the reference's trajectory up to float64 summation
order.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import EvflowError
from .weights import Bases, MlpWeights, generate_bases, init_weights

_dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731


def _ref_error(name):
    try:
        import evflow.errors as ref  # type: ignore
        return (getattr(ref, name),)
    except Exception:
        return ()


class TrainingDivergedError(EvflowError, *_ref_error("TrainingDivergedError")):
    """Training produced a non-finite loss (errors.py:28-29 of the reference)."""


@dataclass(frozen=True)
class TrainConfig:
    """flow.py:206-215."""
    hidden: int = 128
    epochs: int = 300
    batch_size: int = 512
    learning_rate: float = 1e-3
    val_fraction: float = 0.2
    margin: Optional[float] = None  # default resolved to 0.05 * mean |u|
    margin_weight: float = 0.1
    constraint_eps: float = 1e-8
    seed: int = 0


class _Trainer:
    def __init__(self, device, feats, u, w: MlpWeights, margin, tc: TrainConfig):
        lib = _lib.load()
        self._lib = lib
        self.F, self.H = feats.shape[1], w.w1.shape[0]
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (feats, u, w.w1, w.b1, w.w2, w.b2)]
        self._keep = arrs
        h = C.c_void_p()
        _lib.check(lib.vkm_train_create(C.byref(h), int(device), _dp(arrs[0]), _dp(arrs[1]), len(feats), self.F,
                                        self.H, *[_dp(a) for a in arrs[2:]], float(margin),
                                        float(tc.margin_weight), float(tc.constraint_eps), float(tc.learning_rate)))
        self._h = h

    def epoch(self, order: np.ndarray, batch_size: int) -> None:
        o = np.ascontiguousarray(order, dtype=np.int64)
        _lib.check(self._lib.vkm_train_epoch(self._h, o.ctypes.data, len(o), int(batch_size)))

    def loss(self, idx: np.ndarray) -> Tuple[float, int]:
        i = np.ascontiguousarray(idx, dtype=np.int64)
        out, bad = C.c_double(), C.c_int64()
        _lib.check(self._lib.vkm_train_loss(self._h, i.ctypes.data, len(i), C.byref(out), C.byref(bad)))
        return float(out.value), int(bad.value)

    def keep(self) -> None:
        _lib.check(self._lib.vkm_train_keep(self._h))

    def weights(self, best: bool):
        w1 = np.empty((self.H, self.F)); b1 = np.empty(self.H); w2 = np.empty((2, self.H)); b2 = np.empty(2)
        _lib.check(self._lib.vkm_train_get(self._h, int(bool(best)), _dp(w1), _dp(b1), _dp(w2), _dp(b2)))
        return w1, b1, w2, b2

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.vkm_train_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def encode_dataset(dataset: Sequence, width: int, height: int, delta_x: int, delta_y: int, delta_t: float,
                   bases: Bases, precision: str = "f32", device: int = 0):
    """_encode_dataset (flow.py:304-331): features of every (slice, flows)
    pair on the GPU encoder, in the configured precision, as float64, and the
    targets.  `dataset` holds (events (n, 3) array, flows (n, 2)) pairs; the
    flows pair with the slice's time-sorted rows (as in the reference's fit)."""
    from .engine import FlowEngine
    from .errors import EmptyNeighborhoodError
    from .validation import block_from_array, check_flow_array
    eng = FlowEngine(width, height, delta_x, delta_y, delta_t, bases, None, device)
    feats, flows = [], []
    for X, u in dataset:
        blk = block_from_array(X, width, height, 2.0 * delta_t)
        u = check_flow_array(u, len(blk))
        if len(blk) == 0:
            continue
        enc = eng.encode_host_f64 if precision == "f64" else eng.encode_host
        f, cnt = enc(blk.events, blk.t_start, return_counts=True)
        if np.any(cnt == 0):   # _pool_batch without allow_empty (encoder.py:337-343)
            bad = np.flatnonzero(cnt == 0)
            raise EmptyNeighborhoodError(f"{len(bad)} queries have empty neighborhoods "
                                         f"(first at batch position {bad[0]})")
        feats.append(f.astype(np.float64))
        flows.append(u)
    if not feats:
        raise ValueError("training dataset is empty")
    eng.close()
    return np.concatenate(feats), np.concatenate(flows)


def train_head(dataset: Sequence, width: int, height: int, delta_x: int = 10, delta_y: int = 10,
               delta_t: float = 0.016, embed_dim: int = 64, train_cfg: TrainConfig = TrainConfig(),
               bases: Optional[Bases] = None, precision: str = "f32", device: int = 0,
               features: Optional[Tuple[np.ndarray, np.ndarray]] = None) -> MlpWeights:
    """train_head (flow.py:334-402) on the GPU.  `features` = precomputed
    (features, targets) skips the encoding (for tests against reference
    features)."""
    if bases is None:
        bases = generate_bases(embed_dim)
    if features is None:
        feats, u = encode_dataset(dataset, width, height, delta_x, delta_y, delta_t, bases, precision, device)
    else:
        feats, u = (np.asarray(a, dtype=np.float64) for a in features)
        if len(feats) == 0:
            raise ValueError("training dataset is empty")
    n = len(feats)
    rng = np.random.default_rng(train_cfg.seed)
    perm = rng.permutation(n)
    n_val = max(1, int(n * train_cfg.val_fraction)) if n > 1 else 0
    val_idx, train_idx = perm[:n_val], perm[n_val:]
    if len(train_idx) == 0:
        train_idx = perm
    margin = train_cfg.margin
    if margin is None:
        margin = 0.05 * float(np.linalg.norm(u, axis=1).mean())
    w = init_weights(bases.dim, train_cfg.hidden, bases, seed=train_cfg.seed)
    tr = _Trainer(device, feats, u, w, margin, train_cfg)
    try:
        vidx = val_idx if len(val_idx) else train_idx
        best, _ = tr.loss(vidx)
        steps_per_epoch = -(-len(train_idx) // train_cfg.batch_size)
        for epoch in range(train_cfg.epochs):
            order = rng.permutation(train_idx)
            tr.epoch(order, train_cfg.batch_size)
            current, bad = tr.loss(vidx)
            if bad >= 0:   # the first mini-batch whose loss was not finite (flow.py:372-376)
                e = (bad - 1) // steps_per_epoch
                batch = min(train_cfg.batch_size, len(train_idx) - ((bad - 1) % steps_per_epoch) * train_cfg.batch_size)
                raise TrainingDivergedError(f"non-finite loss at epoch {e}, step {bad - 1} "
                                            f"(lr={train_cfg.learning_rate}, batch={batch})")
            if not np.isfinite(current):
                raise TrainingDivergedError(f"non-finite validation loss at epoch {epoch}")
            if current < best:
                best = current
                tr.keep()
        w1, b1, w2, b2 = tr.weights(best=True)
    finally:
        tr.close()
    return MlpWeights(w1, b1, w2, b2, bases, w.activation, w.units)
