"""The array-in/array-out adapter (reference evflow_bindings,
pkg/bindings/tests/test_bindings.py is the model): validation on the host
(CPU), numerics on the GPU against the CPU oracle."""

import numpy as np
import pytest

from conftest import has_cuda
from oracle import veckm_oracle as vo

CONFIG = {
    "delta_t": 0.016, "delta_x": 4, "delta_y": 4, "embed_dim": 16,
    "sigma2": 25.0, "seeds": (0, 1, 2), "precision": "f32",
    "width": 64, "height": 64,
}


def _evb():
    import paper_2504_19417_b200.bindings as evb
    return evb


def random_events(rng, n=80, sorted_t=True):
    t = rng.uniform(0.0, 0.03, n)
    if sorted_t:
        t = np.sort(t)
    return t, rng.integers(0, 64, n).astype(np.int32), rng.integers(0, 64, n).astype(np.int32)


def bias_weights(path, embed_dim=16, b2=(1.5, -0.5)):
    import paper_2504_19417_b200 as pkg
    w = pkg.MlpWeights(np.zeros((4, 2 * embed_dim), np.float32), np.zeros(4, np.float32),
                       np.zeros((2, 4), np.float32), np.array(b2, np.float32), pkg.generate_bases(embed_dim))
    pkg.save_weights(w, str(path))


# ---------------------------------------------------------------- host side
def test_mismatched_lengths_rejected():
    with pytest.raises(ValueError, match="t=2 x=1 y=2"):
        _evb().encode(np.zeros(2), np.zeros(1, int), np.zeros(2, int), np.array([0]), CONFIG)


def test_out_of_range_query_names_index():
    with pytest.raises(IndexError, match="query index 5 at position 1"):
        _evb().encode(np.array([0.0, 0.001]), np.zeros(2, int), np.zeros(2, int), np.array([0, 5]), CONFIG)


def test_queries_must_be_flat():
    with pytest.raises(ValueError, match="flat index array"):
        _evb().encode(np.zeros(2), np.zeros(2, int), np.zeros(2, int), np.zeros((1, 2), int), CONFIG)


def test_span_and_geometry_and_config_errors():
    evb = _evb()
    with pytest.raises(ValueError, match="slice window"):
        evb.encode(np.array([0.0, 0.05]), np.zeros(2, int), np.zeros(2, int), np.array([0]), CONFIG)
    with pytest.raises(ValueError, match="outside geometry"):
        evb.encode(np.array([0.0, 0.01]), np.array([0, 64]), np.zeros(2, int), np.array([0]), CONFIG)
    with pytest.raises(TypeError):
        evb.encode(np.zeros(1), np.zeros(1, int), np.zeros(1, int), np.array([0]), 3)
    with pytest.raises(ValueError, match="precision"):
        evb.encode(np.zeros(1), np.zeros(1, int), np.zeros(1, int), np.array([0]), dict(CONFIG, precision="f16"))


def test_presets():
    evb = _evb()
    p = evb.load_config_preset("640x480_24ms_C64_k10")
    assert (p.geometry.width, p.geometry.height) == (640, 480)
    assert (p.encoder.delta_t, p.encoder.delta_x, p.encoder.embed_dim) == (0.012, 10, 64)
    with pytest.raises(KeyError, match="available"):
        evb.load_config_preset("nope")


# ---------------------------------------------------------------- device
gpu = pytest.mark.gpu


@pytest.fixture
def _need_gpu():
    if not has_cuda():
        pytest.fail("GPU tests need a CUDA device")


@gpu
def test_single_event_self_query(_need_gpu):
    feats = _evb().encode(np.array([0.007]), np.array([10]), np.array([20]), np.array([0]), CONFIG)
    assert feats.dtype == np.float32 and feats.shape == (1, 32)
    # a = 0 -> phase 1; the pre-modulated pooling multiplies by |e^{i theta}|^2 = 1 +- 2^-23
    np.testing.assert_allclose(feats[0, :16], 1.0, rtol=0, atol=3e-7)
    np.testing.assert_allclose(feats[0, 16:], 0.0, rtol=0, atol=3e-7)


@gpu
def test_empty_queries_empty_output(_need_gpu):
    t, x, y = random_events(np.random.default_rng(0))
    assert _evb().encode(t, x, y, np.empty(0, dtype=np.int64), CONFIG).shape == (0, 32)


@gpu
def test_encode_matches_oracle_and_keeps_query_identity(_need_gpu):
    evb = _evb()
    rng = np.random.default_rng(3)
    t, x, y = random_events(rng, n=300, sorted_t=False)
    queries = np.array([0, 17, 41, 299, 17])
    got = evb.encode(t, x, y, queries, CONFIG)
    order = np.argsort(t, kind="stable")
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    np.testing.assert_array_equal(got, evb.encode(t[order], x[order], y[order], inv[queries], CONFIG))
    ts, xs, ys = t[order], x[order].astype(np.int64), y[order].astype(np.int64)
    fr = vo.make_freqs(16, 25.0, (0, 1, 2))
    g = vo.accumulate(ts - ts[0], xs, ys, 64, 64, 4, 4, fr, 0.016)
    q = inv[queries]
    emb, _ = vo.pool(g, vo.spatial_table(fr, 4, 4), ts[q] - ts[0], xs[q], ys[q], fr, 0.016)
    np.testing.assert_allclose(got, vo.to_features(emb), rtol=0, atol=1e-5)


@gpu
def test_preset_config_accepted(_need_gpu):
    evb = _evb()
    feats = evb.encode(np.array([0.0]), np.array([320]), np.array([240]), np.array([0]),
                       evb.load_config_preset("640x480_32ms_C64_k8"))
    assert feats.shape == (1, 128)


@gpu
def test_bias_only_weights_constant_rows(_need_gpu, tmp_path):
    t, x, y = random_events(np.random.default_rng(5), n=12)
    bias_weights(tmp_path / "head.vkmw")
    flows = _evb().predict(t, x, y, np.arange(12), str(tmp_path / "head.vkmw"), CONFIG)
    assert flows.dtype == np.float32
    np.testing.assert_array_equal(flows, np.tile([1.5, -0.5], (12, 1)).astype(np.float32))


@gpu
def test_dim_mismatch_raises(_need_gpu, tmp_path):
    import paper_2504_19417_b200 as pkg
    bias_weights(tmp_path / "head64.vkmw", embed_dim=64)
    t, x, y = random_events(np.random.default_rng(6), n=4)
    with pytest.raises(pkg.DimensionMismatchError):
        _evb().predict(t, x, y, np.arange(4), str(tmp_path / "head64.vkmw"), CONFIG)


@gpu
def test_predict_matches_oracle(_need_gpu, tmp_path):
    import paper_2504_19417_b200 as pkg
    b = pkg.generate_bases(16)
    w = pkg.init_weights(16, 32, b, seed=1, dtype=np.float32)
    pkg.save_weights(w, str(tmp_path / "h.vkmw"))
    rng = np.random.default_rng(9)
    t, x, y = random_events(rng, n=500)
    q = rng.integers(0, 500, 40)
    got = _evb().predict(t, x, y, q, str(tmp_path / "h.vkmw"), CONFIG)
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    want = vo.predict(np.stack([t, x, y], 1), 64, 64, 4, 4, 0.016, fr, w.w1, w.b1, w.w2, w.b2)[q]
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-4)


@gpu
def test_concurrent_calls_on_distinct_inputs(_need_gpu):
    from concurrent.futures import ThreadPoolExecutor
    evb = _evb()
    inputs = [random_events(np.random.default_rng(seed), n=200) for seed in range(8)]
    queries = np.arange(0, 200, 13)
    run = lambda a: evb.encode(*a, queries, CONFIG)  # noqa: E731
    serial = [run(a) for a in inputs]
    with ThreadPoolExecutor(max_workers=4) as pool:
        threaded = list(pool.map(run, inputs))
    for a, b in zip(serial, threaded):
        np.testing.assert_array_equal(a, b)
