"""Freeze golden vectors of the reference's precision="f64" path (complex128
grid, float64 features and head).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_f64.py

Imports `evflow` from /root/reference/pkg/src (read-only, unmodified) and runs
NormalFlowRegressor / LocalEventEncoder with precision="f64" on seeded slices;
writes tests/golden/f64_*.npz (flows, features, neighbourhood counts, the
weights and bases used, numpy version).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import evflow  # noqa: E402
from evflow import (  # noqa: E402
    CameraGeometry, EncoderConfig, LocalEventEncoder, NormalFlowRegressor, QuerySet, SceneParams,
    generate_bases, rebase_slice, synth_workload,
)
from evflow.encoder import encode  # noqa: E402
from evflow.flow import init_weights  # noqa: E402
from evflow.validation import slice_from_array  # noqa: E402


def synth(n, width, height, seed):
    sl, _ = synth_workload(n, CameraGeometry(width, height), "uniform_noise",
                           SceneParams(seed=seed, window=0.032))
    return np.stack([sl.t, sl.x.astype(np.float64), sl.y.astype(np.float64)], axis=1)


def run_case(name, X, width, height, dx, dy, D, hidden, wseed=0, delta_t=0.016, feat_stride=8):
    cfg = EncoderConfig(delta_t=delta_t, delta_x=dx, delta_y=dy, embed_dim=D, precision="f64")
    bases = generate_bases(cfg)
    w = init_weights(D, hidden, bases, seed=wseed, dtype=np.float32)
    reg = NormalFlowRegressor(delta_t=delta_t, delta_x=dx, delta_y=dy, embed_dim=D, precision="f64",
                              width=width, height=height, weights=w)
    flows = reg.predict(X)
    enc = LocalEventEncoder(delta_t=delta_t, delta_x=dx, delta_y=dy, embed_dim=D, precision="f64",
                            width=width, height=height).fit(X)
    feats = enc.transform(X)
    sl = rebase_slice(slice_from_array(X, CameraGeometry(width, height), cfg.window))
    counts = encode(sl, QuerySet.all(len(sl)), cfg, bases).counts
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), X=np.asarray(X, np.float64), width=width, height=height, dx=dx,
        dy=dy, D=D, hidden=hidden, delta_t=delta_t, flows=flows, counts=counts.astype(np.int32),
        feat_idx=np.arange(0, len(feats), feat_stride), feats=feats[::feat_stride],
        w1=w.w1, b1=w.b1, w2=w.w2, b2=w.b2, freqT=bases.time_freqs, freqX=bases.x_freqs, freqY=bases.y_freqs,
        numpy=np.__version__, evflow=evflow.__version__)
    print(f"{name}: n={len(X)} flows {flows.dtype} feats {feats.dtype} {feats.shape}")


def main():
    rng = np.random.default_rng(64)
    run_case("f64_cfg1_6k", synth(6000, 346, 260, seed=11), 346, 260, 10, 10, 64, 128)
    n = 3000
    X = np.stack([np.sort(rng.uniform(0, 0.032, n)), rng.integers(10, 20, n),
                  rng.integers(5, 16, n)], 1).astype(np.float64)
    run_case("f64_dense_asym", X, 40, 30, 3, 6, 64, 128, wseed=4)
    n = 1200
    X = np.stack([1000.0 + np.sort(rng.uniform(0, 0.03, n)), rng.integers(0, 64, n),
                  rng.integers(0, 48, n)], 1).astype(np.float64)
    run_case("f64_d16_offset", X, 64, 48, 4, 4, 16, 8, wseed=2)
    print("done")


if __name__ == "__main__":
    main()
