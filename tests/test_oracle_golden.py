"""Pin the CPU oracle (oracle/veckm_oracle.py) to golden vectors frozen from
the real reference (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import veckm_oracle as vo


def freqs_of(g):
    return vo.Freqs(g["freqT"], g["freqX"], g["freqY"], float(g["sigma2"]))


def test_splitmix_known_answer():
    # pkg/tests/test_rng.py:25-28 pins the first SplitMix64(0) output.
    assert int(vo.splitmix64_stream(0, 1)[0]) == 0xE220A8397B1DCDAF
    g = load_golden("rng_bases")
    np.testing.assert_array_equal(vo.splitmix64_stream(0, 8), g["splitmix_seed0"])
    np.testing.assert_array_equal(vo.splitmix64_stream(12345, 8), g["splitmix_seed12345"])


def test_default_bases_bitwise():
    g = load_golden("rng_bases")
    fr = vo.make_freqs(64, 25.0, (0, 1, 2))
    np.testing.assert_array_equal(fr.T, g["T"])
    np.testing.assert_array_equal(fr.X, g["X"])
    np.testing.assert_array_equal(fr.Y, g["Y"])
    np.testing.assert_array_equal(vo.make_freqs(48, 9.0, (7, 8, 9)).T, g["T_s789_d48"])


def test_oracle_matches_reference_golden(golden_case):
    g = golden_case
    fr = freqs_of(g)
    W, H, dx, dy = int(g["width"]), int(g["height"]), int(g["dx"]), int(g["dy"])
    dt = float(g["delta_t"])
    flows, counts = vo.predict(g["X"], W, H, dx, dy, dt, fr, g["w1"], g["b1"], g["w2"], g["b2"],
                               return_counts=True)
    # neighbourhood membership: bit-exact
    np.testing.assert_array_equal(counts, g["counts"])
    # flows: same numpy ops in the same order -> ulp-level
    np.testing.assert_allclose(flows, g["flows"], rtol=0, atol=1e-6)

    t, x, y, t0 = vo.make_slice(g["X"], W, H, 2 * dt)
    np.testing.assert_array_equal(t, g["sorted_t"])
    np.testing.assert_array_equal(x, g["sorted_x"])
    assert t0 == float(g["t_start"])
    grid = vo.accumulate(t - t0, x, y, W, H, dx, dy, fr, dt)
    np.testing.assert_array_equal(grid.count, g["grid_count"])
    if "grid_embed" in g:
        np.testing.assert_allclose(grid.embed, g["grid_embed"], rtol=0, atol=1e-6)
    else:
        x0, x1, y0, y1 = g["grid_box"]
        np.testing.assert_allclose(grid.embed[x0:x1, y0:y1], g["grid_embed_box"], rtol=0, atol=1e-6)
    tab = vo.spatial_table(fr, dx, dy)
    idx = g["feat_idx"]
    emb, cnt = vo.pool(grid, tab, (t - t0)[idx], x[idx], y[idx], fr, dt)
    np.testing.assert_allclose(emb, g["emb"], rtol=0, atol=1e-6)


def test_encoder_features_golden():
    g = load_golden("encoder_1k")
    fr = vo.make_freqs(64, 25.0, (0, 1, 2))
    feats = vo.encode_features(g["X"], int(g["width"]), int(g["height"]), int(g["dx"]),
                               int(g["dy"]), float(g["delta_t"]), fr)
    np.testing.assert_allclose(feats, g["feats"], rtol=0, atol=1e-6)


def test_direct_encode_agrees_with_pooled(rng):
    # encoder.py:415-440 vs the pooled path (pkg/tests/test_encoder.py:234-246: f32 rtol 1e-3)
    fr = vo.make_freqs(32, 25.0)
    n = 300
    X = np.stack([np.sort(rng.uniform(0, 0.03, n)), rng.integers(0, 32, n), rng.integers(0, 32, n)], 1)
    t, x, y, t0 = vo.make_slice(X, 32, 32, 0.032)
    g = vo.accumulate(t - t0, x, y, 32, 32, 4, 4, fr, 0.016)
    tab = vo.spatial_table(fr, 4, 4)
    emb, cnt = vo.pool(g, tab, t - t0, x, y, fr, 0.016)
    for q in range(0, n, 37):
        ref, c = vo.direct_encode(t - t0, x, y, q, 4, 4, fr, 0.016)
        assert c == cnt[q]
        np.testing.assert_allclose(emb[q], ref, rtol=1e-3, atol=1e-6)


def test_single_event_self_query_is_all_ones():
    # pkg/tests/test_encoder.py:152-158
    fr = vo.make_freqs(16, 25.0)
    g = vo.accumulate(np.array([0.0]), np.array([3]), np.array([4]), 8, 8, 4, 4, fr, 0.016)
    emb, cnt = vo.pool(g, vo.spatial_table(fr, 4, 4), np.array([0.0]), np.array([3]),
                       np.array([4]), fr, 0.016)
    np.testing.assert_array_equal(emb[0], np.ones(16, np.complex64))
    assert cnt[0] == 1


def test_validation_messages():
    with pytest.raises(ValueError, match="shape"):
        vo.validate(np.zeros(3), 8, 8)
    with pytest.raises(ValueError, match="integer"):
        vo.validate(np.array([[0.0, 1.5, 2.0]]), 8, 8)
    with pytest.raises(ValueError, match="outside geometry"):
        vo.validate(np.array([[0.0, 9, 2.0]]), 8, 8)
    with pytest.raises(ValueError, match="window"):
        vo.make_slice(np.array([[0.0, 1, 1], [0.5, 1, 1]]), 8, 8, 0.032)


def test_vkmw_golden_file_layout():
    # flow.py:117-125: magic, <IIIBB, VKMB bases at byte 18, then f32 arrays.
    p = os.path.join(GOLDEN, "cfg1_weights.vkmw")
    assert os.path.getsize(p) == 18 + (16 + 3 * 64 * 8) + 4 * (128 * 128 + 128 + 256 + 2)
    with open(p, "rb") as fh:
        buf = fh.read()
    assert buf[:4] == b"VKMW" and buf[18:22] == b"VKMB"


F64_CASES = ["f64_cfg1_6k", "f64_dense_asym", "f64_d16_offset"]


@pytest.mark.parametrize("case", F64_CASES)
def test_oracle_f64_matches_reference_golden(case):
    """precision="f64" (complex128 grid, float64 features and head): the oracle
    against the reference's own f64 outputs (tests/golden/make_golden_f64.py)."""
    g = load_golden(case)
    fr = vo.Freqs(g["freqT"], g["freqX"], g["freqY"], 25.0)
    W, H, dx, dy = int(g["width"]), int(g["height"]), int(g["dx"]), int(g["dy"])
    dt = float(g["delta_t"])
    flows, counts = vo.predict(g["X"], W, H, dx, dy, dt, fr, g["w1"], g["b1"], g["w2"], g["b2"],
                               precision="f64", return_counts=True)
    np.testing.assert_array_equal(counts, g["counts"])
    np.testing.assert_allclose(flows, g["flows"], rtol=0, atol=1e-10)
    feats = vo.encode_features(g["X"], W, H, dx, dy, dt, fr, precision="f64")
    assert feats.dtype == np.float64
    np.testing.assert_allclose(feats[g["feat_idx"]], g["feats"], rtol=0, atol=1e-12)


def test_accumulate_near_equals_full_accumulate():
    """The bounded-memory restricted accumulation used by the at-size GPU
    checks gives every pixel a query window touches exactly the full grid's
    value (same runs, same reduceat order); counts are complete."""
    g = load_golden("cfg1_20k")
    fr = freqs_of(g)
    t, x, y = g["sorted_t"] - float(g["t_start"]), g["sorted_x"].astype(np.int64), g["sorted_y"].astype(np.int64)
    full = vo.accumulate(t, x, y, 346, 260, 10, 10, fr, 0.016)
    q = np.arange(0, len(t), 731)
    near = vo.accumulate_near(t, x, y, 346, 260, 10, 10, fr, 0.016, x[q], y[q], chunk=997)
    np.testing.assert_array_equal(near.count_p, full.count_p)
    tab = vo.spatial_table(fr, 10, 10)
    e1, c1 = vo.pool(full, tab, t[q], x[q], y[q], fr, 0.016)
    e2, c2 = vo.pool(near, tab, t[q], x[q], y[q], fr, 0.016)
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_array_equal(e1, e2)


def test_cfg1_100k_golden_regenerates_and_matches_oracle():
    """BASELINE configs[0] (346x260, 100k events, delta 10) frozen from the
    real reference (tests/golden/make_golden_cfg1.py): the oracle's synthetic
    slice is byte-identical to the reference's synth_workload, and the
    oracle reproduces the reference's counts exactly and its flows to ulps
    on a strided subset (the full 100k-query pool is the GPU test's job)."""
    import hashlib
    g = load_golden("cfg1_100k")
    X = vo.synth_uniform_noise(int(g["n"]), 346, 260, seed=0)
    assert hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest() == str(g["X_sha256"])
    fr = freqs_of(g)
    t = X[:, 0] - X[0, 0]
    x, y = X[:, 1].astype(np.int64), X[:, 2].astype(np.int64)
    q = np.arange(0, len(X), 53)
    grid = vo.accumulate_near(t, x, y, 346, 260, 10, 10, fr, 0.016, x[q], y[q])
    np.testing.assert_array_equal(grid.count.astype(np.int32), g["grid_count"])
    emb, cnt = vo.pool(grid, vo.spatial_table(fr, 10, 10), t[q], x[q], y[q], fr, 0.016)
    np.testing.assert_array_equal(cnt, g["counts"][q])
    flows = vo.mlp(g["w1"], g["b1"], g["w2"], g["b2"], vo.to_features(emb))
    np.testing.assert_allclose(flows, g["flows"][q], rtol=0, atol=1e-6)
