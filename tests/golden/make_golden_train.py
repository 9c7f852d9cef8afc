"""Freeze a head-training run of the REAL reference (train_head, flow.py:334-402).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_train.py

Two small slices (64x48, D = 16, precision f64) with synthetic ground-truth
flows; the reference encodes them (_encode_dataset) and trains a hidden-16
head for 12 epochs of mini-batch Adam.  Saves the slices, the targets, the
reference's features, the train config and the returned (best) weights.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import evflow  # noqa: E402
from evflow import CameraGeometry, EncoderConfig, QuerySet, generate_bases  # noqa: E402
from evflow.flow import TrainConfig, _encode_dataset, train_head  # noqa: E402
from evflow.validation import slice_from_array  # noqa: E402


def main():
    rng = np.random.default_rng(77)
    W, H = 64, 48
    cfg = EncoderConfig(delta_t=0.016, delta_x=4, delta_y=4, embed_dim=16, precision="f64")
    geom = CameraGeometry(W, H)
    Xs, Us, dataset = [], [], []
    for k in range(2):
        n = 1500
        X = np.stack([np.sort(rng.uniform(0, 0.03, n)), rng.integers(0, W, n), rng.integers(0, H, n)],
                     1).astype(np.float64)
        u = np.array([30.0 - 20 * k, 10.0 + 15 * k]) + rng.normal(0, 3.0, size=(n, 2))
        sl = slice_from_array(X, geom, cfg.window)
        dataset.append((sl, QuerySet.all(len(sl)), u))
        Xs.append(X)
        Us.append(u)
    bases = generate_bases(cfg)
    tc = TrainConfig(hidden=16, epochs=12, batch_size=128, learning_rate=1e-2, seed=3)
    feats, u_all = _encode_dataset(dataset, cfg, bases, 1)
    w = train_head(dataset, cfg, tc, bases=bases)
    np.savez_compressed(os.path.join(HERE, "train_small.npz"), X0=Xs[0], X1=Xs[1], u0=Us[0], u1=Us[1],
                        width=W, height=H, dx=4, dy=4, D=16, delta_t=0.016, hidden=16, epochs=12,
                        batch_size=128, lr=1e-2, seed=3, feats=feats, u=u_all,
                        w1=w.w1, b1=w.b1, w2=w.w2, b2=w.b2, numpy=np.__version__, evflow=evflow.__version__)
    print("train_small:", feats.shape, "w1", w.w1.shape, float(np.abs(w.w1).max()))


if __name__ == "__main__":
    main()
