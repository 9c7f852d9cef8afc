"""Freeze golden vectors from the REAL reference implementation.

Run in the build container (the reference is importable only here):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `evflow` from /root/reference/pkg/src (read-only, unmodified), runs
its public API on seeded inputs and writes `tests/golden/*.npz` plus one
`.vkmw` weight file.  These fixtures travel to the GPU box; the reference does
not.  numpy / OpenBLAS versions are recorded in every file because the
reference's float results are ulp-sensitive to the numpy build.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import evflow  # noqa: E402
from evflow import (  # noqa: E402
    CameraGeometry, EncoderConfig, EventSlice, LocalEventEncoder, NormalFlowRegressor,
    QuerySet, accumulate_grid, generate_bases, precompute_spatial_phases, rebase_slice,
    synth_workload, SceneParams,
)
from evflow.encoder import _pool_batch  # noqa: E402
from evflow.flow import MlpWeights, init_weights, save_weights  # noqa: E402
from evflow.rng import splitmix64  # noqa: E402
from evflow.validation import slice_from_array  # noqa: E402


def versions():
    return dict(numpy=np.__version__, evflow=evflow.__version__)


def weights_arrays(w):
    return dict(w1=np.asarray(w.w1), b1=np.asarray(w.b1), w2=np.asarray(w.w2), b2=np.asarray(w.b2),
                freqT=w.bases.time_freqs, freqX=w.bases.x_freqs, freqY=w.bases.y_freqs,
                sigma2=np.float64(w.bases.sigma2))


def run_case(name, X, width, height, dx, dy, D, hidden, w=None, feat_stride=1,
             grid_box=None, wseed=0, delta_t=0.016, bias=None):
    cfg = EncoderConfig(delta_t=delta_t, delta_x=dx, delta_y=dy, embed_dim=D)
    bases = generate_bases(cfg)
    if w is None:
        w = init_weights(D, hidden, bases, seed=wseed, dtype=np.float32)
    if bias is not None:
        w = MlpWeights(w1=np.zeros_like(w.w1), b1=np.zeros_like(w.b1), w2=np.zeros_like(w.w2),
                       b2=np.asarray(bias, dtype=np.float32), bases=bases)
    reg = NormalFlowRegressor(delta_t=delta_t, delta_x=dx, delta_y=dy, embed_dim=D,
                              width=width, height=height, weights=w)
    flows = reg.predict(X)
    geom = CameraGeometry(width, height)
    sl = slice_from_array(X, geom, cfg.window)
    rs = rebase_slice(sl)
    grid = accumulate_grid(rs, w.bases, cfg)
    table = precompute_spatial_phases(w.bases, cfg)
    idx = np.arange(0, len(rs), feat_stride, dtype=np.int64)
    emb, cnt_sub = _pool_batch(grid, table, rs.t[idx], rs.x[idx].astype(np.int64),
                               rs.y[idx].astype(np.int64), w.bases, cfg, allow_empty=True)
    _, counts = _pool_batch(grid, table, rs.t, rs.x.astype(np.int64), rs.y.astype(np.int64),
                            w.bases, cfg, allow_empty=True) if feat_stride != 1 else (None, cnt_sub)
    out = dict(
        X=np.asarray(X, np.float64), width=width, height=height, dx=dx, dy=dy, D=D,
        hidden=w.w1.shape[0], delta_t=delta_t,
        flows=flows, counts=np.asarray(counts, np.int32),
        feat_idx=idx, emb=emb.astype(np.complex64),
        grid_count=grid.count.astype(np.int32),
        sorted_t=sl.t, sorted_x=sl.x, sorted_y=sl.y, t_start=np.float64(sl.t_start),
        **weights_arrays(w), **versions(),
    )
    if grid_box is not None:
        x0, x1, y0, y1 = grid_box
        out["grid_box"] = np.array(grid_box)
        out["grid_embed_box"] = grid.embed[x0:x1, y0:y1].astype(np.complex64)
    else:
        out["grid_embed"] = grid.embed.astype(np.complex64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: n={len(X)} flows finite={np.isfinite(flows).all(axis=1).sum()}")
    return w


def synth(n, width, height, seed):
    sl, _ = synth_workload(n, CameraGeometry(width, height), "uniform_noise",
                           SceneParams(seed=seed, window=0.032))
    return np.stack([sl.t, sl.x.astype(np.float64), sl.y.astype(np.float64)], axis=1)


def main():
    rng = np.random.default_rng(20240817)

    # 1. reference-test-sized slice: 64x64, delta 4, D=16, hidden 8.
    n = 1500
    X = np.stack([np.sort(rng.uniform(0, 0.03, n)), rng.integers(0, 64, n),
                  rng.integers(0, 64, n)], 1).astype(np.float64)
    run_case("small_d16", X, 64, 64, 4, 4, 16, 8)

    # 2. config-1 geometry (346x260 DAVIS, delta 10, D=64, hidden 128), 20k events.
    X = synth(20000, 346, 260, seed=0)
    w = run_case("cfg1_20k", X, 346, 260, 10, 10, 64, 128, feat_stride=32,
                 grid_box=(100, 116, 100, 116))
    save_weights(w, os.path.join(HERE, "cfg1_weights.vkmw"))

    # 3. large radius (delta 20) on a 320x180 sensor, 12k events.
    X = synth(12000, 320, 180, seed=3)
    run_case("r20_12k", X, 320, 180, 20, 20, 64, 128, feat_stride=24,
             grid_box=(0, 24, 160, 180))

    # 4. asymmetric radii and a dense pixel cluster (~35 events / px).
    n = 4000
    X = np.stack([np.sort(rng.uniform(0, 0.032, n)), rng.integers(10, 20, n),
                  rng.integers(5, 16, n)], 1).astype(np.float64)
    run_case("dense_asym", X, 40, 30, 3, 6, 64, 128, wseed=4, feat_stride=8)

    # 5. edge cases (tiny slices, delta 4, D=64).
    edge = {
        "single": np.array([[0.0137, 3, 4]]),
        "pair_same_px": np.array([[0.0, 3, 3], [0.016, 3, 3]]),
        "corner": np.stack([np.sort(rng.uniform(0, 0.03, 30)), rng.integers(0, 3, 30),
                            rng.integers(0, 3, 30)], 1),
        "far_corner": np.array([[0.0, 0, 0], [0.001, 7, 7], [0.002, 7, 0], [0.003, 0, 7]]),
        "unsorted_dups": np.array([[0.02, 1, 1], [0.01, 2, 2], [0.01, 2, 2], [0.005, 1, 1],
                                   [0.02, 5, 6], [0.0, 7, 7]]),
        "t_offset": np.stack([1000.0 + np.sort(rng.uniform(0, 0.031, 50)),
                              rng.integers(0, 8, 50), rng.integers(0, 8, 50)], 1),
    }
    for key, X in edge.items():
        run_case(f"edge_{key}", np.asarray(X, np.float64), 8, 8, 4, 4, 64, 128, wseed=1)
    run_case("edge_bias_only", edge["corner"], 8, 8, 4, 4, 64, 128, bias=(2.5, -1.0))

    # 6. known answers for the pinned RNG and the default bases.
    cfg = EncoderConfig(delta_t=0.016)
    b = generate_bases(cfg)
    np.savez_compressed(os.path.join(HERE, "rng_bases.npz"),
                        splitmix_seed0=splitmix64(0, 8), splitmix_seed12345=splitmix64(12345, 8),
                        T=b.time_freqs, X=b.x_freqs, Y=b.y_freqs,
                        T_s789_d48=generate_bases(EncoderConfig(delta_t=0.016, embed_dim=48,
                                                                sigma2=9.0, seeds=(7, 8, 9))).time_freqs,
                        **versions())

    # 7. encoder-only path (LocalEventEncoder.transform), D=64 delta 10.
    X = synth(1000, 96, 64, seed=5)
    enc = LocalEventEncoder(delta_t=0.016, width=96, height=64).fit(X)
    np.savez_compressed(os.path.join(HERE, "encoder_1k.npz"), X=X, width=96, height=64, dx=10,
                        dy=10, D=64, delta_t=0.016, feats=enc.transform(X).astype(np.float32),
                        **versions())
    print("done")


if __name__ == "__main__":
    main()
