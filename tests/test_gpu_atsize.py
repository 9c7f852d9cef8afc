"""GPU parity at the BASELINE configs' real sizes (BASELINE.json `configs`).

* configs[0]: 346x260, 100k events, delta 10 — every one of the 100k flows
  and neighbourhood counts against the golden frozen from the REAL reference
  (tests/golden/make_golden_cfg1.py), through the drop-in `predict(X)`.
* configs[2]: 1280x720, 4M events, delta 20 (41-pixel windows, the longest
  sliding-window segments) — counts of all 4M events exact (box sums of the pixel histogram),
  flows of 2000 strided queries against the oracle (vo.accumulate_near: the
  reference's per-pixel order over every pixel a query window touches).
* configs[4] density: the full 1280x720 slice of 32M events (35 ev/px, the
  dense slices' radix-sort path) — all counts exact, 200 strided oracle queries; and a
  1280x96 band at the same density with 2000 queries.
* configs[3]: 125 slices of 200k events (346x260) batched through
  predict_slices — all counts exact per slice against box sums, flows of
  sampled slices against per-slice oracle runs.

Bars: counts bit-exact; flows max-abs <= 1e-4 (FLOW_TOL).  With
VKM_PARITY_OUT=<file>, each test appends its measured max-abs error as one
JSON line (the evidence committed under profiles/).
"""

import json
import os
import time

import numpy as np
import pytest

from conftest import has_cuda, load_golden
from oracle import veckm_oracle as vo

pytestmark = pytest.mark.gpu

FLOW_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("GPU tests need a CUDA device")


def _pkg():
    import paper_2504_19417_b200 as pkg
    return pkg


def _report(case, **vals):
    path = os.environ.get("VKM_PARITY_OUT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(dict(case=case, **vals)) + "\n")


def box_counts(X, W, H, dx, dy):
    """Neighbourhood sizes as exact box sums of the pixel histogram
    (the int64 count loop of encoder.py:331-336)."""
    x, y = X[:, 1].astype(np.int64), X[:, 2].astype(np.int64)
    hist = np.bincount((y + dy) * (W + 2 * dx) + (x + dx),
                       minlength=(H + 2 * dy) * (W + 2 * dx)).reshape(H + 2 * dy, W + 2 * dx)
    ii = np.pad(hist.cumsum(0).cumsum(1), ((1, 0), (1, 0)))
    return (ii[y + 2 * dy + 1, x + 2 * dx + 1] - ii[y, x + 2 * dx + 1] - ii[y + 2 * dy + 1, x] + ii[y, x])


def oracle_flows(X, q, W, H, d, fr, w):
    t0 = float(X[0, 0])
    t = X[:, 0] - t0
    x, y = X[:, 1].astype(np.int64), X[:, 2].astype(np.int64)
    g = vo.accumulate_near(t, x, y, W, H, d, d, fr, 0.016, x[q], y[q])
    emb, c = vo.pool(g, vo.spatial_table(fr, d, d), t[q], x[q], y[q], fr, 0.016)
    return vo.mlp(w.w1, w.b1, w.w2, w.b2, vo.to_features(emb)), c


def default_model(pkg, d):
    fr = vo.make_freqs(64)
    b = pkg.Bases(fr.T, fr.X, fr.Y, 25.0)
    return fr, b, pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)


@pytest.mark.parametrize("mode", ["auto", "fp32"])
def test_config1_full_slice_vs_reference_golden(mode):
    pkg = _pkg()
    g = load_golden("cfg1_100k")
    X = vo.synth_uniform_noise(int(g["n"]), 346, 260, seed=0)
    b = pkg.Bases(g["freqT"], g["freqX"], g["freqY"], 25.0)
    w = pkg.MlpWeights(g["w1"], g["b1"], g["w2"], g["b2"], b)
    reg = pkg.NormalFlowRegressor(delta_t=0.016, delta_x=10, delta_y=10, width=346, height=260, weights=w,
                                  mlp_mode=mode)
    flows = reg.predict(X)                      # the drop-in call, all 100k rows
    assert flows.dtype == np.float64 and flows.shape == (len(X), 2)
    err = float(np.abs(flows - g["flows"]).max())
    _, cnt = reg.engine().predict_host(X, float(X[0, 0]), return_counts=True)
    np.testing.assert_array_equal(cnt, g["counts"])
    _report("cfg1_100k_vs_reference", mode=mode, n=len(X), queries=len(X), max_abs=err)
    assert err <= FLOW_TOL, err


def test_config3_4m_delta20_at_size():
    pkg = _pkg()
    W, H, d, n = 1280, 720, 20, 4_000_000
    X = vo.synth_uniform_noise(n, W, H, seed=0)
    fr, b, w = default_model(pkg, d)
    eng = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    flows, cnt = eng.predict_host(X, float(X[0, 0]), return_counts=True)
    np.testing.assert_array_equal(cnt, box_counts(X, W, H, d, d))
    q = np.arange(0, n, n // 2000)
    want, c = oracle_flows(X, q, W, H, d, fr, w)
    np.testing.assert_array_equal(c, cnt[q])
    err = float(np.abs(flows[q] - want).max())
    _report("cfg3_4M_delta20", n=n, queries=len(q), max_abs=err, counts_checked=n)
    assert err <= FLOW_TOL, err


def test_config5_full_32m_slice_at_size():
    import torch
    pkg = _pkg()
    W, H, d, n = 1280, 720, 10, 32_000_000
    X = vo.synth_uniform_noise(n, W, H, seed=0)
    fr, b, w = default_model(pkg, d)
    eng = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    ev = torch.from_numpy(X).cuda()
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    flows = eng.predict_device(ev, float(X[0, 0]), counts=cnt).cpu().numpy()
    cnt = cnt.cpu().numpy()
    del ev
    np.testing.assert_array_equal(cnt, box_counts(X, W, H, d, d))
    q = np.arange(0, n, n // 200)
    want, c = oracle_flows(X, q, W, H, d, fr, w)
    np.testing.assert_array_equal(c, cnt[q])
    err = float(np.abs(flows[q] - want).max())
    _report("cfg5_32M_full", n=n, queries=len(q), max_abs=err, counts_checked=n)
    assert err <= FLOW_TOL, err


def test_config5_density_band():
    """1280x96 band at configs[4]'s density (35 ev/px, 4.3M events)."""
    pkg = _pkg()
    W, H, d = 1280, 96, 10
    n = int(round(32_000_000 / (1280 * 720) * W * H))
    X = vo.synth_uniform_noise(n, W, H, seed=5)
    fr, b, w = default_model(pkg, d)
    eng = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    flows, cnt = eng.predict_host(X, float(X[0, 0]), return_counts=True)
    np.testing.assert_array_equal(cnt, box_counts(X, W, H, d, d))
    q = np.arange(0, n, n // 2000)
    want, c = oracle_flows(X, q, W, H, d, fr, w)
    np.testing.assert_array_equal(c, cnt[q])
    err = float(np.abs(flows[q] - want).max())
    _report("cfg5_density_band_1280x96", n=n, queries=len(q), max_abs=err, counts_checked=n)
    assert err <= FLOW_TOL, err


def test_config4_125_slices_batched():
    """configs[3]: one rank's share at 8 GPUs (125 of the 1000 slices of 200k
    events, seeds 0..124) through the additive predict_slices API."""
    pkg = _pkg()
    W, H, d, n, ns = 346, 260, 10, 200_000, 125
    fr, b, w = default_model(pkg, d)
    reg = pkg.NormalFlowRegressor(delta_t=0.016, delta_x=d, delta_y=d, width=W, height=H, weights=w)
    slices = [vo.synth_uniform_noise(n, W, H, seed=s) for s in range(ns)]
    t = time.perf_counter()
    outs = reg.predict_slices(slices)
    wall = time.perf_counter() - t
    eng = reg.engine()
    errs = []
    for s, (X, f) in enumerate(zip(slices, outs)):
        assert f.shape == (n, 2) and np.isfinite(f).all()
        if s % 31 == 0:   # counts through the per-slice call, flows vs the oracle
            f1, c1 = eng.predict_host(X, float(X[0, 0]), return_counts=True)
            np.testing.assert_array_equal(c1, box_counts(X, W, H, d, d))
            np.testing.assert_allclose(f, f1, rtol=0, atol=1e-5)
            q = np.arange(s % 7, n, n // 400)
            want, c = oracle_flows(X, q, W, H, d, fr, w)
            np.testing.assert_array_equal(c, c1[q])
            errs.append(float(np.abs(f[q] - want).max()))
    _report("cfg4_125x200k_batched", slices=ns, sampled_slices=len(errs), queries_per_slice=400,
            max_abs=max(errs), wall_s=wall)
    assert max(errs) <= FLOW_TOL, errs
