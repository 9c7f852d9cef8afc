"""precision="f64" on the GPU (k_f64.cu through vkm_predict_f64 / vkm_encode_f64)
against the reference's own f64 outputs (tests/golden/make_golden_f64.py) and
the CPU oracle in f64.

Bars: neighbourhood counts bit-exact; flows max-abs <= 1e-9 and features
max-abs <= 1e-10 against the reference (the f64 path pools the modulated grid
separably, so its rounding differs from the reference's 441-term direct sum
at the 1e-13 level)."""

import numpy as np
import pytest

from conftest import has_cuda, load_golden
from oracle import veckm_oracle as vo

pytestmark = pytest.mark.gpu

F64_CASES = ["f64_cfg1_6k", "f64_dense_asym", "f64_d16_offset"]
FLOW_TOL64 = 1e-9
FEAT_TOL64 = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("GPU tests need a CUDA device")


def _pkg():
    import paper_2504_19417_b200 as pkg
    return pkg


def _weights(g):
    pkg = _pkg()
    b = pkg.Bases(g["freqT"], g["freqX"], g["freqY"], 25.0)
    return pkg.MlpWeights(g["w1"], g["b1"], g["w2"], g["b2"], b)


@pytest.mark.parametrize("case", F64_CASES)
def test_f64_predict_matches_reference_golden(case):
    pkg = _pkg()
    g = load_golden(case)
    reg = pkg.NormalFlowRegressor(delta_t=float(g["delta_t"]), delta_x=int(g["dx"]), delta_y=int(g["dy"]),
                                  embed_dim=int(g["D"]), width=int(g["width"]), height=int(g["height"]),
                                  precision="f64", weights=_weights(g))
    flows = reg.predict(g["X"])
    assert flows.dtype == np.float64
    np.testing.assert_allclose(flows, g["flows"], rtol=0, atol=FLOW_TOL64)
    blk = pkg.block_from_array(g["X"], int(g["width"]), int(g["height"]), 2 * float(g["delta_t"]))
    _, counts = reg.engine().predict_host_f64(blk.events, blk.t_start, return_counts=True)
    np.testing.assert_array_equal(counts, g["counts"])


@pytest.mark.parametrize("case", F64_CASES)
def test_f64_encoder_matches_reference_golden(case):
    pkg = _pkg()
    g = load_golden(case)
    enc = pkg.LocalEventEncoder(delta_t=float(g["delta_t"]), delta_x=int(g["dx"]), delta_y=int(g["dy"]),
                                embed_dim=int(g["D"]), width=int(g["width"]), height=int(g["height"]),
                                precision="f64").fit(g["X"])
    feats = enc.transform(g["X"])
    assert feats.dtype == np.float64 and feats.shape == (len(g["X"]), 2 * int(g["D"]))
    np.testing.assert_allclose(feats[g["feat_idx"]], g["feats"], rtol=0, atol=FEAT_TOL64)


def test_f64_bindings_dtypes():
    pkg = _pkg()
    g = load_golden("f64_d16_offset")
    X = g["X"]
    cfg = dict(width=int(g["width"]), height=int(g["height"]), delta_t=float(g["delta_t"]), delta_x=int(g["dx"]),
               delta_y=int(g["dy"]), embed_dim=int(g["D"]), precision="f64")
    q = np.arange(0, len(X), 7)
    import paper_2504_19417_b200.bindings as evb
    f = evb.encode(X[:, 0], X[:, 1].astype(int), X[:, 2].astype(int), q, cfg)
    assert f.dtype == np.float64
    np.testing.assert_allclose(f[::1], vo.encode_features(X, cfg["width"], cfg["height"], cfg["delta_x"],
                                                          cfg["delta_y"], cfg["delta_t"],
                                                          vo.Freqs(g["freqT"], g["freqX"], g["freqY"], 25.0),
                                                          precision="f64")[q], rtol=0, atol=FEAT_TOL64)


def test_f64_agrees_with_f32_path_at_config2_size():
    """1M events on 640x480: the f64 and f32 paths give the same counts and
    flows within the f32 bar; the f64 flows match the f64 oracle on a strided
    subset of queries."""
    pkg = _pkg()
    W, H = 640, 480
    X = vo.synth_uniform_noise(1_000_000, W, H, seed=9)
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 10, 10, 0.016, b, w)
    t0 = float(X[0, 0])
    f64, c64 = eng.predict_host_f64(X, t0, return_counts=True)
    f32, c32 = eng.predict_host(X, t0, return_counts=True)
    np.testing.assert_array_equal(c64, c32)
    np.testing.assert_allclose(f64, f32, rtol=0, atol=1e-4)
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    q = np.arange(0, len(X), 997)
    g = vo.accumulate(X[:, 0] - t0, X[:, 1].astype(np.int64), X[:, 2].astype(np.int64), W, H, 10, 10, fr, 0.016,
                      "f64")
    emb, cnt = vo.pool(g, vo.spatial_table(fr, 10, 10, "f64"), X[q, 0] - t0, X[q, 1].astype(np.int64),
                       X[q, 2].astype(np.int64), fr, 0.016, "f64")
    np.testing.assert_array_equal(cnt, c64[q])
    want = vo.mlp(w.w1, w.b1, w.w2, w.b2, vo.to_features(emb))
    np.testing.assert_allclose(f64[q], want, rtol=0, atol=FLOW_TOL64)


def _fuzz_slice(rng, n, width, height, window=0.032):
    """pkg/tests/conftest.py:18-25: sorted uniform times, uniform pixels, t_start = 0."""
    t = np.sort(rng.uniform(0.0, window, size=n))
    return np.stack([t, rng.integers(0, width, size=n), rng.integers(0, height, size=n)], 1).astype(np.float64)


def test_direct_encode_matches_cpu_direct_sum():
    """The GPU oracle_encode against the CPU oracle's direct summation (both f64)."""
    pkg = _pkg()
    rng = np.random.default_rng(3)
    X = _fuzz_slice(rng, 4000, 50, 40)
    b = pkg.generate_bases(64)
    eng = pkg.FlowEngine(50, 40, 8, 6, 0.016, b)
    q = rng.integers(0, len(X), 40)
    emb, cnt = eng.direct_encode_host(X, q, return_counts=True)
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    for i, qi in enumerate(q):
        want, n = vo.direct_encode(X[:, 0], X[:, 1], X[:, 2], int(qi), 8, 6, fr, 0.016)
        assert cnt[i] == n
        np.testing.assert_allclose(emb[i], want, rtol=1e-12, atol=1e-13)


def test_acceptance_oracle_equivalence_fuzz():
    """test_acceptance.py:49-86 on the GPU: 1000 fuzzed slices (n <= 5000,
    geometry <= 64x64, radii 8 and 10, two queries each); the pooled
    embeddings of both precisions against the direct summation: f64 < 1e-6
    and f32 < 1e-3 relative (floors 1e-9 / 1e-6), counts equal."""
    pkg = _pkg()
    rng = np.random.default_rng(7)
    b = pkg.generate_bases(64)
    # one 64x64 handle per radius: pixels beyond a slice's own geometry are empty,
    # so its encodings equal those on its own sensor size
    engines = {r: pkg.FlowEngine(64, 64, r, r, 0.016, b) for r in (8, 10)}
    worst = {"f64": 0.0, "f32": 0.0}
    for i in range(1000):
        r = 8 if i % 2 == 0 else 10
        n = int(rng.integers(1, 5001))
        X = _fuzz_slice(rng, n, int(rng.integers(16, 65)), int(rng.integers(16, 65)))
        q = rng.integers(0, n, size=min(2, n)).astype(np.int64)
        eng = engines[r]
        want, wcnt = eng.direct_encode_host(X, q, return_counts=True)
        for prec, fn, floor in (("f64", eng.encode_host_f64, 1e-9), ("f32", eng.encode_host, 1e-6)):
            feats, cnt = fn(X, 0.0, return_counts=True)
            np.testing.assert_array_equal(cnt[q], wcnt)
            got = feats[q, :64].astype(np.float64) + 1j * feats[q, 64:].astype(np.float64)
            err = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)))
            worst[prec] = max(worst[prec], err)
    print(f"acceptance fuzz: max rel err f64={worst['f64']:.2e} f32={worst['f32']:.2e}")
    assert worst["f64"] < 1e-6 and worst["f32"] < 1e-3, worst


@pytest.mark.parametrize("hidden", [128, 224])
def test_f64_head_keeps_float64_weights(hidden):
    """precision="f64" with float64 weights (what fit returns) runs a float64
    head on those weights, as the reference's mlp_forward does (flow.py:98-106):
    weights that f32 cannot represent must still agree within FLOW_TOL64.
    hidden=128 stages W1ᵀ in shared memory as double (128 KB); at hidden=224
    it does not fit and is read from global memory (same arithmetic)."""
    pkg = _pkg()
    W, H, D = 96, 80, 64
    X = vo.synth_uniform_noise(4000, W, H, seed=11)
    b = pkg.generate_bases(D, 25.0, (0, 1, 2))
    w = pkg.init_weights(D, hidden, b, seed=3, dtype=np.float64)
    g = np.random.default_rng(5)
    w = pkg.MlpWeights(w.w1 * (1 + 1e-3 * g.standard_normal(w.w1.shape)), g.standard_normal(hidden) * 0.1,
                       w.w2, g.standard_normal(2), b)
    assert np.any(w.w1.astype(np.float32).astype(np.float64) != w.w1)
    reg = pkg.NormalFlowRegressor(width=W, height=H, precision="f64", weights=w, hidden=hidden)
    got = reg.predict(X)
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    want = vo.predict(X, W, H, 10, 10, 0.016, fr, w.w1, w.b1, w.w2, w.b2, precision="f64")
    np.testing.assert_allclose(got, want, rtol=0, atol=FLOW_TOL64)
    # the f32-rounded head would miss the bar: the test can see the difference
    w32 = pkg.MlpWeights(*(a.astype(np.float32) for a in (w.w1, w.b1, w.w2, w.b2)), b)
    want32 = vo.predict(X, W, H, 10, 10, 0.016, fr, *(a.astype(np.float64) for a in (w32.w1, w32.b1, w32.w2,
                                                                                        w32.b2)), precision="f64")
    assert np.max(np.abs(want32 - want)) > 10 * FLOW_TOL64
