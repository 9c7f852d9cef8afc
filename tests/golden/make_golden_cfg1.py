"""Freeze the BASELINE configs[0] golden from the REAL reference (build container only).

configs[0] = "single synthetic slice, 346x260 DAVIS sensor, ~100k events,
default delta radius, reference CPU estimator (oracle run)".  This script runs
the unmodified reference (`/root/reference/pkg/src`) on exactly that slice:

    X      = bench.synth_workload(100_000, CameraGeometry(346, 260),
             "uniform_noise", SceneParams(seed=0, window=0.032))   (bench.py:162-214)
    weights = init_weights(64, 128, generate_bases(EncoderConfig(0.016)), seed=0, float32)
    flows  = NormalFlowRegressor(...).predict(X)                     (estimators.py:192-206)
    counts = _pool_batch(..., allow_empty=True) neighbourhood sizes  (encoder.py:312-346)

X itself is not stored (2.4 MB): the oracle's `synth_uniform_noise` draws the
same stream, and the fixture keeps a SHA-256 of the reference's X bytes so the
CPU suite proves the regenerated slice is identical.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cfg1.py
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import evflow  # noqa: E402
from evflow import (  # noqa: E402
    CameraGeometry, EncoderConfig, NormalFlowRegressor, SceneParams, accumulate_grid,
    generate_bases, precompute_spatial_phases, rebase_slice, synth_workload,
)
from evflow.encoder import _pool_batch  # noqa: E402
from evflow.flow import init_weights  # noqa: E402
from evflow.validation import slice_from_array  # noqa: E402

N, W, H, D, HIDDEN, DELTA = 100_000, 346, 260, 64, 128, 10
EMB_STRIDE = 97          # strided embeddings kept (1031 rows)


def main():
    sl, _ = synth_workload(N, CameraGeometry(W, H), "uniform_noise", SceneParams(seed=0, window=0.032))
    X = np.stack([sl.t, sl.x.astype(np.float64), sl.y.astype(np.float64)], axis=1)
    cfg = EncoderConfig(delta_t=0.016, delta_x=DELTA, delta_y=DELTA, embed_dim=D)
    bases = generate_bases(cfg)
    w = init_weights(D, HIDDEN, bases, seed=0, dtype=np.float32)
    reg = NormalFlowRegressor(delta_t=0.016, delta_x=DELTA, delta_y=DELTA, embed_dim=D, width=W, height=H,
                              weights=w)
    t0 = time.perf_counter()
    flows = reg.predict(X)
    t_pred = time.perf_counter() - t0
    s2 = slice_from_array(X, CameraGeometry(W, H), cfg.window)
    rs = rebase_slice(s2)
    grid = accumulate_grid(rs, w.bases, cfg)
    table = precompute_spatial_phases(w.bases, cfg)
    emb, cnt = _pool_batch(grid, table, rs.t, rs.x.astype(np.int64), rs.y.astype(np.int64), w.bases, cfg,
                           allow_empty=True)
    idx = np.arange(0, N, EMB_STRIDE, dtype=np.int64)
    np.savez_compressed(
        os.path.join(HERE, "cfg1_100k.npz"),
        n=N, width=W, height=H, dx=DELTA, dy=DELTA, D=D, hidden=HIDDEN, delta_t=0.016, seed=0,
        X_sha256=hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest(),
        X_head=X[:16], X_tail=X[-16:],
        flows=flows, counts=np.asarray(cnt, np.int32), emb_idx=idx, emb=emb[idx].astype(np.complex64),
        grid_count=grid.count.astype(np.int32),
        w1=np.asarray(w.w1), b1=np.asarray(w.b1), w2=np.asarray(w.w2), b2=np.asarray(w.b2),
        freqT=w.bases.time_freqs, freqX=w.bases.x_freqs, freqY=w.bases.y_freqs, sigma2=np.float64(25.0),
        reference_predict_seconds=np.float64(t_pred), numpy=np.__version__, evflow=evflow.__version__,
    )
    print(f"cfg1_100k: predict {t_pred:.1f} s, finite rows {np.isfinite(flows).all(1).sum()}")


if __name__ == "__main__":
    main()
