"""Flow-head weights, frequency bases and the VKMW / VKMB file formats.

Host-side data only (nothing here runs per event).  Semantics follow the
reference: `Bases` (encoder.py:87-112), `generate_bases` with the pinned
SplitMix64 + Box-Muller stream (encoder.py:115-124, rng.py:22-70),
`MlpWeights` (flow.py:48-80), `save_weights` / `load_weights`
(flow.py:117-152, bases block encoder.py:127-145) and `init_weights`
(flow.py:218-231).  Paths are relative to /root/reference/pkg/src/evflow/.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from .errors import DimensionMismatchError, EventParseError

WEIGHTS_MAGIC = b"VKMW"
BASES_MAGIC = b"VKMB"
WEIGHTS_VERSION = 1
ACTIVATIONS = {0: "relu"}
UNITS = {0: "px_per_s"}

_M64 = (1 << 64) - 1


def _splitmix64(seed: int, count: int) -> np.ndarray:
    """Stateless SplitMix64: output k = mix(seed + (k+1)·γ) mod 2^64 (rng.py:22-43)."""
    k = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _M64) + k * np.uint64(0x9E3779B97F4A7C15)
        for shift, mult in ((30, 0xBF58476D1CE4E5B9), (27, 0x94D049BB133111EB)):
            z = (z ^ (z >> np.uint64(shift))) * np.uint64(mult)
        return z ^ (z >> np.uint64(31))


def standard_normals(seed: int, count: int) -> np.ndarray:
    """Box-Muller over consecutive output pairs (rng.py:46-70)."""
    raw = _splitmix64(seed, 2 * ((count + 1) // 2)).reshape(-1, 2)
    u1 = ((raw[:, 0] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (raw[:, 1] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    return np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1).reshape(-1)[:count]


@dataclass(frozen=True)
class Bases:
    """Time / x / y frequency vectors, float64 (encoder.py:87-112)."""

    time_freqs: np.ndarray
    x_freqs: np.ndarray
    y_freqs: np.ndarray
    sigma2: float

    def __post_init__(self) -> None:
        for name in ("time_freqs", "x_freqs", "y_freqs"):
            v = np.ascontiguousarray(getattr(self, name), dtype=np.float64)
            if v.ndim != 1 or not np.all(np.isfinite(v)):
                raise ValueError(f"{name} must be a finite 1-d vector")
            object.__setattr__(self, name, v)
        if not len(self.time_freqs) == len(self.x_freqs) == len(self.y_freqs):
            raise ValueError("frequency vectors must share one length")

    @property
    def dim(self) -> int:
        return len(self.time_freqs)


def generate_bases(embed_dim: int = 64, sigma2: float = 25.0, seeds=(0, 1, 2)) -> Bases:
    """N(0, sigma2) vectors from the pinned stream, one seed per axis."""
    s = float(np.sqrt(sigma2))
    t, x, y = (standard_normals(int(sd), embed_dim) * s for sd in seeds)
    return Bases(t, x, y, float(sigma2))


def bases_to_bytes(b: Bases) -> bytes:
    body = b"".join(v.astype("<f8").tobytes() for v in (b.time_freqs, b.x_freqs, b.y_freqs))
    return BASES_MAGIC + struct.pack("<Id", b.dim, b.sigma2) + body


def bases_from_bytes(buf: bytes, offset: int = 0) -> Tuple[Bases, int]:
    if buf[offset:offset + 4] != BASES_MAGIC:
        raise EventParseError(f"missing {BASES_MAGIC!r} magic at offset {offset}")
    dim, sigma2 = struct.unpack_from("<Id", buf, offset + 4)
    pos = offset + 16
    vecs = np.frombuffer(buf, dtype="<f8", count=3 * dim, offset=pos).reshape(3, dim).copy()
    return Bases(vecs[0], vecs[1], vecs[2], float(sigma2)), pos + 24 * dim


@dataclass
class MlpWeights:
    """Flow head W2·relu(W1·f + b1) + b2 bound to its bases (flow.py:48-80)."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    bases: Bases
    activation: str = "relu"
    units: str = "px_per_s"

    def __post_init__(self) -> None:
        hidden, fin = np.shape(self.w1)
        if fin != 2 * self.bases.dim:
            raise DimensionMismatchError(f"w1 expects {fin} features but bases give {2 * self.bases.dim}")
        if np.shape(self.b1) != (hidden,) or np.shape(self.w2) != (2, hidden) or np.shape(self.b2) != (2,):
            raise DimensionMismatchError("inconsistent weight shapes")
        for a in (self.w1, self.b1, self.w2, self.b2):
            if not np.all(np.isfinite(a)):
                raise ValueError("weights must be finite")
        if self.activation not in ACTIVATIONS.values():
            raise ValueError(f"unsupported activation {self.activation!r}")

    @property
    def embed_dim(self) -> int:
        return self.bases.dim

    @property
    def hidden(self) -> int:
        return int(np.shape(self.w1)[0])


def as_weights(obj) -> MlpWeights:
    """Accept this package's MlpWeights or any duck-typed equivalent (e.g. the
    reference's evflow.MlpWeights)."""
    if isinstance(obj, MlpWeights):
        return obj
    b = obj.bases
    return MlpWeights(np.asarray(obj.w1), np.asarray(obj.b1), np.asarray(obj.w2), np.asarray(obj.b2),
                      Bases(b.time_freqs, b.x_freqs, b.y_freqs, float(b.sigma2)),
                      getattr(obj, "activation", "relu"), getattr(obj, "units", "px_per_s"))


def save_weights(w: MlpWeights, path: str) -> None:
    act = {v: k for k, v in ACTIVATIONS.items()}[w.activation]
    unit = {v: k for k, v in UNITS.items()}[w.units]
    head = WEIGHTS_MAGIC + struct.pack("<IIIBB", WEIGHTS_VERSION, w.embed_dim, w.hidden, act, unit)
    arrays = b"".join(np.ascontiguousarray(a, dtype="<f4").tobytes() for a in (w.w1, w.b1, w.w2, w.b2))
    with open(path, "wb") as fh:
        fh.write(head + bases_to_bytes(w.bases) + arrays)


def load_weights(path: str) -> MlpWeights:
    with open(path, "rb") as fh:
        buf = fh.read()
    if buf[:4] != WEIGHTS_MAGIC:
        raise EventParseError(f"{path}: missing {WEIGHTS_MAGIC!r} magic")
    version, dim, hidden, act, unit = struct.unpack_from("<IIIBB", buf, 4)
    if version != WEIGHTS_VERSION:
        raise EventParseError(f"{path}: unsupported weight version {version}")
    if act not in ACTIVATIONS or unit not in UNITS:
        raise EventParseError(f"{path}: unknown activation/units tags ({act}, {unit})")
    bases, pos = bases_from_bytes(buf, 18)
    if bases.dim != dim:
        raise DimensionMismatchError(f"{path}: header D={dim} but bases carry D={bases.dim}")
    sizes = (hidden * 2 * dim, hidden, 2 * hidden, 2)
    flat = np.frombuffer(buf, dtype="<f4", count=sum(sizes), offset=pos).copy()
    w1, b1, w2, b2 = np.split(flat, np.cumsum(sizes)[:-1])
    return MlpWeights(w1.reshape(hidden, 2 * dim), b1, w2.reshape(2, hidden), b2, bases,
                      ACTIVATIONS[act], UNITS[unit])


def init_weights(embed_dim: int, hidden: int, bases: Bases, seed: int = 0, dtype=np.float64) -> MlpWeights:
    """He-normal W1/W2, zero biases, numpy default_rng(seed) (flow.py:218-231)."""
    g = np.random.default_rng(seed)
    fin = 2 * embed_dim
    w1 = g.normal(0.0, np.sqrt(2.0 / fin), size=(hidden, fin)).astype(dtype)
    w2 = g.normal(0.0, np.sqrt(2.0 / hidden), size=(2, hidden)).astype(dtype)
    return MlpWeights(w1, np.zeros(hidden, dtype), w2, np.zeros(2, dtype), bases)
