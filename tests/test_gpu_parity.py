"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
vectors and the CPU oracle.

Bars: pixel counts and neighbourhood counts bit-exact;
flows max-abs <= 1e-4 in the fp32-equivalent modes (FP32, F16X3); BF16 fast
mode: max-abs <= 2e-3 and angular error p99 <= 2 deg, max <= 15 deg over
|flow| >= 1e-2.  Embeddings / features max-abs <= 1e-5 (|emb| <= 1).
"""

import math

import numpy as np
import pytest

from conftest import GOLDEN_CASES, has_cuda, load_golden
from oracle import veckm_oracle as vo

pytestmark = pytest.mark.gpu

FLOW_TOL = 1e-4
EMB_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("GPU tests need a CUDA device")


def _pkg():
    import paper_2504_19417_b200 as pkg
    return pkg


def weights_of(g):
    pkg = _pkg()
    b = pkg.Bases(g["freqT"], g["freqX"], g["freqY"], float(g["sigma2"]))
    return pkg.MlpWeights(g["w1"], g["b1"], g["w2"], g["b2"], b)


def regressor(g, mode="auto"):
    pkg = _pkg()
    return pkg.NormalFlowRegressor(delta_t=float(g["delta_t"]), delta_x=int(g["dx"]), delta_y=int(g["dy"]),
                                   embed_dim=int(g["D"]), width=int(g["width"]), height=int(g["height"]),
                                   weights=weights_of(g), mlp_mode=mode)


def angular_stats(got, want, floor=1e-2):
    sel = np.linalg.norm(want, axis=1) >= floor
    a = np.arctan2(got[sel, 1], got[sel, 0])
    b = np.arctan2(want[sel, 1], want[sel, 0])
    d = np.degrees(np.abs(np.angle(np.exp(1j * (a - b)))))
    return (float(np.percentile(d, 99)), float(d.max())) if len(d) else (0.0, 0.0)


@pytest.mark.parametrize("variant", ["mufu", "poly", "rows"])
@pytest.mark.parametrize("mode", ["fp32", "f16x3", "auto", "bf16"])
@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_predict_matches_reference_golden(case, mode, variant, monkeypatch):
    """Flows vs the reference's (max-abs FLOW_TOL; BF16: 3.5e-3, its angular
    bound is tested below) and neighbourhood counts exact, for every MLP mode,
    both sin/cos flavours of the hot kernels (VKM_SINCOS: special-function
    unit by default, or the polynomials) and both K3 producer layouts
    (one event per lane by default, VKM_K3=rows: one row per warp)."""
    monkeypatch.setenv("VKM_SINCOS", "poly" if variant == "poly" else "mufu")
    if variant == "rows":
        monkeypatch.setenv("VKM_K3", "rows")
    g = load_golden(case)
    reg = regressor(g, mode)
    if mode == "f16x3" and not (int(g["D"]) == 64 and int(g["w1"].shape[0]) == 128):
        pytest.skip("tensor-core head needs D=64, hidden=128")
    if mode == "bf16" and not (int(g["D"]) == 64 and int(g["w1"].shape[0]) == 128):
        pytest.skip("tensor-core head needs D=64, hidden=128")
    flows = reg.predict(g["X"])
    assert flows.dtype == np.float64 and flows.shape == g["flows"].shape
    np.testing.assert_allclose(flows, g["flows"], rtol=0, atol=3.5e-3 if mode == "bf16" else FLOW_TOL)
    blk = _pkg().block_from_array(g["X"], int(g["width"]), int(g["height"]), 2 * float(g["delta_t"]))
    _, counts = reg.engine().predict_host(blk.events, blk.t_start, return_counts=True)
    np.testing.assert_array_equal(counts, g["counts"])


@pytest.mark.parametrize("case", ["cfg1_20k", "r20_12k", "dense_asym"])
def test_bf16_fast_mode_bound(case):
    g = load_golden(case)
    flows = regressor(g, "bf16").predict(g["X"])
    assert np.max(np.abs(flows - g["flows"])) <= 2e-3
    p99, mx = angular_stats(flows, g["flows"])
    assert p99 <= 2.0 and mx <= 15.0, (p99, mx)


def test_bias_only_head_is_exact():
    g = load_golden("edge_bias_only")
    for mode in ("fp32", "f16x3"):
        flows = regressor(g, mode).predict(g["X"])
        np.testing.assert_array_equal(flows, np.tile([2.5, -1.0], (len(flows), 1)))


@pytest.mark.parametrize("case", ["small_d16", "cfg1_20k", "dense_asym", "edge_corner", "edge_t_offset"])
def test_grid_matches_reference_golden(case):
    import torch
    g = load_golden(case)
    pkg = _pkg()
    reg = regressor(g)
    blk = pkg.block_from_array(g["X"], int(g["width"]), int(g["height"]), 2 * float(g["delta_t"]))
    ev = torch.from_numpy(blk.events).cuda()
    grid, cnt = reg.engine().grid_device(ev, blk.t_start, pooled=False)
    np.testing.assert_array_equal(cnt.cpu().numpy(), g["grid_count"])
    grid = grid.cpu().numpy()
    if "grid_embed" in g:
        np.testing.assert_allclose(grid, g["grid_embed"], rtol=0, atol=2e-6 * max(1, g["grid_count"].max()))
    else:
        x0, x1, y0, y1 = g["grid_box"]
        np.testing.assert_allclose(grid[x0:x1, y0:y1], g["grid_embed_box"], rtol=0, atol=1e-5)


@pytest.mark.parametrize("W,H,dx,dy,D,n,seed", [
    (64, 48, 4, 4, 64, 3000, 1),
    (96, 40, 10, 10, 64, 8000, 2),
    (130, 70, 20, 20, 64, 6000, 3),     # strip wider than one CTA at delta 20
    (300, 50, 3, 7, 32, 9000, 4),       # asymmetric radii, D padded to 32
    (40, 300, 12, 5, 16, 5000, 5),      # tall sensor
    (257, 9, 1, 1, 8, 2000, 6),         # radius 1, one-plane grid
])
def test_pooled_grid_matches_oracle(W, H, dx, dy, D, n, seed):
    """K1+K2 against the oracle's window sums at every pixel."""
    import torch
    pkg = _pkg()
    X = vo.synth_uniform_noise(n, W, H, seed=seed)
    fr = vo.make_freqs(D, 25.0, (seed, seed + 1, seed + 2))
    b = pkg.Bases(fr.T, fr.X, fr.Y, 25.0)
    eng = pkg.FlowEngine(W, H, dx, dy, 0.016, b)
    t0 = float(X[0, 0])
    ev = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    q, qc = eng.grid_device(ev, t0, pooled=True)
    g = vo.accumulate(X[:, 0] - t0, X[:, 1].astype(np.int64), X[:, 2].astype(np.int64), W, H, dx, dy, fr, 0.016)
    acc, cnt = vo.pooled_all_pixels(g, vo.spatial_table(fr, dx, dy))
    np.testing.assert_array_equal(qc.cpu().numpy(), cnt)
    scale = np.maximum(cnt, 1)[:, :, None]
    np.testing.assert_allclose(q.cpu().numpy() / scale, acc / scale, rtol=0, atol=EMB_TOL)


def test_encoder_features_golden():
    g = load_golden("encoder_1k")
    pkg = _pkg()
    enc = pkg.LocalEventEncoder(delta_t=float(g["delta_t"]), width=int(g["width"]), height=int(g["height"])).fit(g["X"])
    feats = enc.transform(g["X"])
    assert feats.dtype == np.float32 and feats.shape == g["feats"].shape
    np.testing.assert_allclose(feats, g["feats"], rtol=0, atol=EMB_TOL)


@pytest.mark.parametrize("D", [8, 16, 64])
def test_features_match_oracle_small_dims(D, rng):
    pkg = _pkg()
    W, H = 50, 40
    X = vo.synth_uniform_noise(4000, W, H, seed=D)
    enc = pkg.LocalEventEncoder(delta_t=0.016, delta_x=5, delta_y=3, embed_dim=D, width=W, height=H).fit()
    feats = enc.transform(X)
    fr = vo.make_freqs(D, 25.0)
    want = vo.encode_features(X, W, H, 5, 3, 0.016, fr)
    np.testing.assert_allclose(feats, want, rtol=0, atol=EMB_TOL)


def test_empty_and_tiny_slices():
    pkg = _pkg()
    g = load_golden("edge_single")
    reg = regressor(g)
    assert reg.predict(np.zeros((0, 3))).shape == (0, 2)
    f = reg.predict(g["X"])
    np.testing.assert_allclose(f, g["flows"], atol=FLOW_TOL)


def test_unsorted_input_rows_follow_time_order():
    g = load_golden("edge_unsorted_dups")
    f = regressor(g).predict(g["X"])
    np.testing.assert_allclose(f, g["flows"], atol=FLOW_TOL)


def test_device_api_matches_host_api():
    import torch
    g = load_golden("cfg1_20k")
    reg = regressor(g)
    pkg = _pkg()
    blk = pkg.block_from_array(g["X"], 346, 260, 0.032)
    eng = reg.engine()
    host = eng.predict_host(blk.events, blk.t_start)
    dev = eng.predict_device(torch.from_numpy(blk.events).cuda(), math.nan).cpu().numpy()
    np.testing.assert_allclose(dev, host, rtol=0, atol=1e-6)


def test_batch_matches_single_slices():
    import torch
    pkg = _pkg()
    g = load_golden("cfg1_20k")
    reg = regressor(g)
    eng = reg.engine()
    slices = [vo.synth_uniform_noise(5000 + 1000 * s, 346, 260, seed=10 + s) for s in range(4)]
    ev = torch.from_numpy(np.concatenate(slices)).cuda()
    off = np.cumsum([0] + [len(s) for s in slices])
    out = eng.predict_batch_device(ev, off).cpu().numpy()
    # batched and single launches pick different x-segment widths in
    # k_reduce_x, so the sliding window sums round differently (~1e-7 rel.)
    for s, X in enumerate(slices):
        single = eng.predict_host(X, float(X[0, 0]))
        np.testing.assert_allclose(out[off[s]:off[s + 1]], single, rtol=0, atol=1e-5)


def test_full_size_config2_properties():
    """640x480, 1M events (BASELINE configs[1]): size-independent properties
    plus oracle parity on a strided query subset."""
    import torch
    pkg = _pkg()
    W, H, n = 640, 480, 1_000_000
    X = vo.synth_uniform_noise(n, W, H, seed=0)
    fr = vo.make_freqs(64)
    b = pkg.Bases(fr.T, fr.X, fr.Y, 25.0)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 10, 10, 0.016, b, w)
    ev = torch.from_numpy(X).cuda()
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    flows = eng.predict_device(ev, float(X[0, 0]), counts=cnt).cpu().numpy()
    cnt = cnt.cpu().numpy()
    # neighbourhood counts: exact box sums of the pixel histogram
    hist = np.zeros((H + 20, W + 20), np.int64)
    np.add.at(hist, (X[:, 2].astype(int) + 10, X[:, 1].astype(int) + 10), 1)
    ii = np.pad(hist.cumsum(0).cumsum(1), ((1, 0), (1, 0)))
    yy, xx = X[:, 2].astype(int), X[:, 1].astype(int)
    box = ii[yy + 21, xx + 21] - ii[yy, xx + 21] - ii[yy + 21, xx] + ii[yy, xx]
    np.testing.assert_array_equal(cnt, box)
    assert np.all(np.isfinite(flows))
    # run-to-run: the stable radix sort fixes every summation order -> bit-identical
    flows2 = eng.predict_device(ev, float(X[0, 0])).cpu().numpy()
    np.testing.assert_array_equal(flows, flows2)
    # oracle on 1500 strided queries (pool cost is per query)
    t0 = float(X[0, 0])
    g = vo.accumulate(X[:, 0] - t0, xx, yy, W, H, 10, 10, fr, 0.016)
    q = np.arange(0, n, n // 1500)
    emb, c = vo.pool(g, vo.spatial_table(fr, 10, 10), X[q, 0] - t0, xx[q], yy[q], fr, 0.016)
    np.testing.assert_array_equal(c, cnt[q])
    want = vo.mlp(w.w1, w.b1, w.w2, w.b2, vo.to_features(emb))
    np.testing.assert_allclose(flows[q], want, rtol=0, atol=FLOW_TOL)


def test_spatial_strip_split_matches_unsplit():
    """Config-5 style row-strip split with a δ-row event halo (strips run one
    after another on this GPU): counts bit-exact, flows within fp32 noise."""
    pkg = _pkg()
    from paper_2504_19417_b200 import sharding
    W, H, d, n = 256, 120, 10, 200_000
    X = vo.synth_uniform_noise(n, W, H, seed=11)
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    full = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    f_full, c_full = full.predict_host(X, float(X[0, 0]), return_counts=True)
    for world in (2, 3, 8):
        rows = np.bincount(X[:, 2].astype(np.int64), minlength=H)
        strips = sharding.row_strips(rows, world, d)
        ses = [sharding.strip_events(X, s) for s in strips]
        res = [pkg.FlowEngine(W, s.height, d, d, 0.016, b, w).predict_host(se.events, float(X[0, 0]), True)
               for s, se in zip(strips, ses)]
        flows, counts = sharding.assemble(n, ses, [r[0] for r in res], [r[1] for r in res])
        np.testing.assert_array_equal(counts, c_full)
        np.testing.assert_allclose(flows, f_full, rtol=0, atol=1e-5)


def test_bench_multirank_shared_gpu(tmp_path):
    """The torchrun (N=2) bench path, both ranks on this GPU (gloo plumbing)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VKM_BENCH_SHARED_GPU="1", VKM_BENCH_CFG4_SLICES="6")
    runs = [("cfg1", "slices", 0), ("cfg1", "spatial", 1), ("cfg4", "slices", 2)]
    for wl, split, k in runs:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + k),
               os.path.join(root, "bench.py"), "--gpus", "2", "--workload", wl, "--steps", "3",
               "--warmup", "3", "--no-cpu-baseline", "--split", split]
        if wl == "cfg4":
            cmd.append("--no-e2e")
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=root)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, out.stdout
        rec = json.loads(lines[0])
        assert rec["n_gpus"] == 2 and rec["value"] > 0
        assert rec["scaling"] == ("strong" if (split == "spatial" or wl == "cfg4") else "weak")
        if wl == "cfg4":   # the fixed slice set split over the ranks: 3 slices each
            assert rec["config"]["slices_per_rank_per_step"] == 3
        if split == "spatial":   # e2e: pinned slice -> GPU 0 -> strips -> flows back
            assert rec["e2e"]["value"] > 0 and rec["e2e"]["h2d_bytes_per_step"] == 24 * 100_000


def test_predict_slices_pipelined_host_batch():
    """predict_slices (vkm_predict_batch_host: copy-in / kernels / copy-out on
    three streams) returns, per slice, exactly what predict returns; empty
    slices in the middle and slices of very different sizes included."""
    pkg = _pkg()
    g = load_golden("cfg1_20k")
    reg = regressor(g)
    sizes = [4000, 0, 25000, 1, 9000, 0, 17000]
    slices = [vo.synth_uniform_noise(n, 346, 260, seed=40 + i) if n else np.zeros((0, 3)) for i, n in
              enumerate(sizes)]
    got = reg.predict_slices(slices)
    assert len(got) == len(slices)
    for X, f in zip(slices, got):
        assert f.shape == (len(X), 2) and f.dtype == np.float64
        if len(X):   # batched launches: other x-segment widths -> f32 rounding noise
            np.testing.assert_allclose(f, reg.predict(X), rtol=0, atol=1e-5)
    # counts through the engine call
    eng = reg.engine()
    ev = np.concatenate([s for s in slices if len(s)])
    off = np.cumsum([0] + [len(s) for s in slices if len(s)])
    flows, counts = eng.predict_batch_host(ev, off, [float(s[0, 0]) for s in slices if len(s)], return_counts=True)
    for i, s in enumerate([s for s in slices if len(s)]):
        f1, c1 = eng.predict_host(s, float(s[0, 0]), return_counts=True)
        np.testing.assert_allclose(flows[off[i]:off[i + 1]], f1, rtol=0, atol=1e-5)
        np.testing.assert_array_equal(counts[off[i]:off[i + 1]], c1)


@pytest.mark.parametrize("d", [1, 10, 24, 25])
def test_fused_x_window_matches_split_pooling(d, monkeypatch):
    """k_reduce_x (x window fused into the per-pixel reduction) against the
    raw-grid + two-pass pooling path (VKM_POOL=split) on the same slice:
    counts bit-exact, flows within f32 summation-order noise.  d = 25 is past
    the fused kernel's radius limit, so both handles run the split path."""
    pkg = _pkg()
    W, H, n = 200, 150, 60000
    X = vo.synth_uniform_noise(n, W, H, seed=d)
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    fused = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    monkeypatch.setenv("VKM_POOL", "split")
    split = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    f1, c1 = fused.predict_host(X, float(X[0, 0]), return_counts=True)
    f2, c2 = split.predict_host(X, float(X[0, 0]), return_counts=True)
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_allclose(f1, f2, rtol=0, atol=1e-5)


def test_batched_slices_many_chunks_edge_cases():
    """Batched launch sequences (up to 64 slices stacked as one virtual
    W x (nb·H) sensor with hard slice borders): 70 slices of mixed sizes ->
    more than one chunk; empty slices, a single-event slice, an out-of-sensor
    event (NaN row, count 0), explicit and NaN t_starts.  Each slice must match
    its own single-slice run (counts exact, flows to f32 rounding)."""
    import torch
    pkg = _pkg()
    W, H = 120, 90
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 10, 10, 0.016, b, w)
    rng = np.random.default_rng(5)
    slices = []
    for i in range(70):
        n = int(rng.choice([0, 1, 700, 3000, 9000]))
        X = vo.synth_uniform_noise(n, W, H, seed=100 + i) if n else np.zeros((0, 3))
        if n and i % 9 == 0:
            X[n // 2, 1] = W + 3   # outside the sensor
        slices.append(X)
    off = np.cumsum([0] + [len(s) for s in slices])
    ts = [float(s[0, 0]) if (len(s) and i % 2) else math.nan for i, s in enumerate(slices)]
    ev = torch.from_numpy(np.ascontiguousarray(np.concatenate([s for s in slices if len(s)]))).cuda()
    cnt = torch.empty(len(ev), dtype=torch.int32, device="cuda")
    flows = eng.predict_batch_device(ev, off, ts, counts=cnt).cpu().numpy()
    cnt = cnt.cpu().numpy()
    for i, X in enumerate(slices):
        if not len(X):
            continue
        f1, c1 = eng.predict_host(X, float(X[0, 0]), return_counts=True)
        np.testing.assert_array_equal(cnt[off[i]:off[i + 1]], c1)
        np.testing.assert_allclose(flows[off[i]:off[i + 1]], f1, rtol=0, atol=1e-5)
        if i % 9 == 0:
            assert np.isnan(flows[off[i] + len(X) // 2]).all() and cnt[off[i] + len(X) // 2] == 0


@pytest.mark.parametrize("sort", ["auto", "counting", "rows", "radix"])
@pytest.mark.parametrize("case", ["hot", "hotrow", "dense"])
def test_pixel_order_is_the_stable_argsort(case, sort):
    """K1's event order equals accumulate_grid's np.argsort(flat,
    kind="stable") and bincount run starts (encoder.py:255-259) exactly, on
    both sort paths: the counting scatter + run ordering (k_prep arrival ranks
    -> k_scan -> k_scatter -> k_runsort, long runs sorted in-block) and the
    dense slices' sorts (radix; row-bucket k_rowhist -> k_scan -> k_rowscatter
    -> k_xsort).  "hot": runs of 1, 2..256, 257..4096 and > 4096 events;
    "hotrow": 64 adjacent 300-event runs (more long runs than k_runsort's
    block step sorts together: the rest take the per-thread insertion sort);
    "dense": 35 events per pixel (the config-5 density).  The sort switch (VKM_SORT) is read once
    per process, so each case runs in a fresh interpreter (tests/_order_check.py)."""
    import os, subprocess, sys
    env = dict(os.environ)
    env.pop("VKM_SORT", None)
    if sort != "auto":
        env["VKM_SORT"] = sort
    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, os.path.join(here, "_order_check.py"), case], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, (out.stdout + out.stderr)[-3000:]
    assert "order ok" in out.stdout


def test_host_batch_packing_edge_cases():
    """vkm_predict_batch_host with host packing (VKM_HOST_PACK=1: f32 time
    argument + 16-bit pixel coordinates packed on host threads): out-of-sensor
    and non-integer pixels become NaN rows with count 0, explicit and NaN
    t_starts, and the packed path matches the default f64-row path (fresh
    process) bitwise."""
    import os
    import subprocess
    import sys
    import tempfile
    if os.environ.get("VKM_HOST_PACK") != "1":   # the switch is read once per process: rerun this test packed
        out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                              os.path.abspath(__file__) + "::test_host_batch_packing_edge_cases"],
                             env=dict(os.environ, VKM_HOST_PACK="1"), capture_output=True, text=True, timeout=600,
                             cwd=os.path.dirname(os.path.abspath(__file__)))
        assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
        return
    pkg = _pkg()
    W, H = 200, 120
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 10, 10, 0.016, b, w)
    slices = [vo.synth_uniform_noise(n, W, H, seed=300 + n) for n in (5000, 1, 40000, 7000)]
    slices[2][10, 1] = W          # outside
    slices[2][11, 2] = 3.5        # not an integer pixel
    slices[3][0, 0] += 0.0        # first event defines t0 when t_start is NaN
    ev = np.ascontiguousarray(np.concatenate(slices))
    off = np.cumsum([0] + [len(s) for s in slices])
    ts = [float(slices[0][0, 0]), math.nan, float(slices[2][0, 0]), math.nan]
    flows, counts = eng.predict_batch_host(ev, off, ts, return_counts=True)
    bad = off[2] + np.array([10, 11])
    assert np.isnan(flows[bad]).all() and (counts[bad] == 0).all()
    good = np.setdiff1d(np.arange(len(ev)), bad)
    assert np.isfinite(flows[good]).all() and (counts[good] > 0).all()
    with tempfile.TemporaryDirectory() as td:
        np.save(os.path.join(td, "ev.npy"), ev)
        code = (
            "import sys, math, numpy as np; sys.path.insert(0, %r); import paper_2504_19417_b200 as pkg;"
            "ev = np.load(%r); b = pkg.generate_bases(64); w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32);"
            "e = pkg.FlowEngine(%d, %d, 10, 10, 0.016, b, w);"
            "f, c = e.predict_batch_host(ev, %r, %r, return_counts=True); np.save(%r, f); np.save(%r, c)"
        ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(td, "ev.npy"), W, H,
             [int(v) for v in off], ts, os.path.join(td, "f.npy"), os.path.join(td, "c.npy"))
        code = code.replace("nan", "math.nan")
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, VKM_HOST_PACK="0"),
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        np.testing.assert_array_equal(np.load(os.path.join(td, "c.npy")), counts)
        np.testing.assert_array_equal(np.load(os.path.join(td, "f.npy")), flows)


def _spatial_worker(rank, world, port, W, H, d, path, out_path):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2504_19417_b200 as pkg
    from paper_2504_19417_b200 import sharding
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    X = np.load(path)
    ev = torch.from_numpy(X).cuda() if rank == 0 else None
    out = sharding.predict_spatial_device(lambda h: pkg.FlowEngine(W, h, d, d, 0.016, b, w), ev, float(X[0, 0]),
                                          W, H, d, world, rank)
    if rank == 0:
        np.save(out_path, out.cpu().numpy())
    dist.destroy_process_group()


def test_spatial_split_device_path_two_ranks(tmp_path):
    """Device-resident row-strip split (vkm_select_rows partition, strip runs,
    vkm_scatter_rows gather) with two ranks sharing this GPU (gloo stages the
    messages through host memory): equal to the unsplit slice (flows within
    f32 rounding of the different x/y segmentations)."""
    import socket
    import torch.multiprocessing as mp
    pkg = _pkg()
    W, H, d, n = 200, 160, 10, 120_000
    X = vo.synth_uniform_noise(n, W, H, seed=21)
    path, out_path = str(tmp_path / "X.npy"), str(tmp_path / "f.npy")
    np.save(path, X)
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    mp.spawn(_spatial_worker, args=(2, port, W, H, d, path, out_path), nprocs=2, join=True)
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    full = pkg.FlowEngine(W, H, d, d, 0.016, b, w).predict_host(X, float(X[0, 0]))
    got = np.load(out_path)
    assert np.isfinite(got).all()
    np.testing.assert_allclose(got, full, rtol=0, atol=1e-5)


def test_single_slice_host_packing_and_wide_output():
    """vkm_predict_host on large single slices packs the rows on host threads
    into page-locked staging (n >= VKM_HOST_PACK_SINGLE) and brings the flows
    back in pinned pieces; vkm_predict_host_wide widens them to float64 on the
    host pool.  Both equal the unpacked f64-row path bitwise (fresh process,
    VKM_HOST_PACK_SINGLE=0), out-of-sensor / non-integer pixels included, with
    an explicit and a NaN t_start."""
    import os
    import subprocess
    import sys
    import tempfile
    pkg = _pkg()
    W, H = 320, 240
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 10, 10, 0.016, b, w)
    ev = np.ascontiguousarray(vo.synth_uniform_noise(300_000, W, H, seed=77))
    ev[1000, 1] = W          # outside
    ev[2000, 2] = 7.25       # not an integer pixel
    res = {}
    for ts in (float(ev[0, 0]) - 1e-3, math.nan):
        f, c = eng.predict_host(ev, ts, return_counts=True)
        fw, cw = eng.predict_host_wide(ev, ts, return_counts=True)
        assert fw.dtype == np.float64
        np.testing.assert_array_equal(fw, f.astype(np.float64))
        np.testing.assert_array_equal(cw, c)
        assert np.isnan(f[[1000, 2000]]).all() and (c[[1000, 2000]] == 0).all()
        res[str(ts)] = (f, c)
    small, sc = eng.predict_host_wide(ev[:5000], math.nan, return_counts=True)   # below the packing threshold
    np.testing.assert_array_equal(small, eng.predict_host(ev[:5000], math.nan).astype(np.float64))
    with tempfile.TemporaryDirectory() as td:
        np.save(os.path.join(td, "ev.npy"), ev)
        code = (
            "import sys, math, numpy as np; sys.path.insert(0, %r); import paper_2504_19417_b200 as pkg;"
            "ev = np.load(%r); b = pkg.generate_bases(64); w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32);"
            "e = pkg.FlowEngine(%d, %d, 10, 10, 0.016, b, w);"
            "r = [e.predict_host(ev, t, return_counts=True) for t in (%r, math.nan)];"
            "np.savez(%r, f0=r[0][0], c0=r[0][1], f1=r[1][0], c1=r[1][1])"
        ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(td, "ev.npy"), W, H,
             float(ev[0, 0]) - 1e-3, os.path.join(td, "r.npz"))
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, VKM_HOST_PACK_SINGLE="0"),
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        r = np.load(os.path.join(td, "r.npz"))
        (f0, c0), (f1, c1) = res[str(float(ev[0, 0]) - 1e-3)], res["nan"]
        np.testing.assert_array_equal(r["c0"], c0)
        np.testing.assert_array_equal(r["f0"], f0)
        np.testing.assert_array_equal(r["c1"], c1)
        np.testing.assert_array_equal(r["f1"], f1)


def test_large_host_encodes_match_device_encodes():
    """Feature blocks of large host calls come back through pinned pieces
    copied out by the host pool (vkm_encode_host, vkm_encode_f64_host): equal
    bitwise to the device-pointer calls on the same slice."""
    import torch
    pkg = _pkg()
    W, H = 160, 120
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 6, 6, 0.016, b, w)
    ev = np.ascontiguousarray(vo.synth_uniform_noise(200_000, W, H, seed=91))
    t0 = float(ev[0, 0])
    fh, ch = eng.encode_host(ev, t0, return_counts=True)
    evd = torch.from_numpy(ev).cuda()
    fd = torch.empty((len(ev), 128), dtype=torch.float32, device="cuda")
    cd = torch.empty(len(ev), dtype=torch.int32, device="cuda")
    eng.encode_device(evd, t0, feats=fd, counts=cd)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(fh, fd.cpu().numpy())
    np.testing.assert_array_equal(ch, cd.cpu().numpy())
    import ctypes as C
    m = 150_000
    f64h = eng.encode_host_f64(ev[:m], t0)
    f64d = torch.empty((m, 128), dtype=torch.float64, device="cuda")
    rc = eng._lib.vkm_encode_f64(eng._h, C.c_void_p(evd.data_ptr()), m, t0, C.c_void_p(f64d.data_ptr()), None,
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    np.testing.assert_array_equal(f64h, f64d.cpu().numpy())
    fl64 = eng.predict_host_f64(ev[:m], t0)
    np.testing.assert_array_equal(fl64, eng.predict_device_f64(evd[:m], t0).cpu().numpy())


def test_multi_handle_slice_sharding():
    """vkm_predict_multi_host (config 4's sharding: contiguous slice ranges of
    equal event counts, one handle and host thread each, no collective) with
    several handles on this GPU equals the single-handle batch, empty slices
    and uneven sizes included; duplicate handles are rejected.  Flows within
    1e-6, not bitwise: a handle batches its own slices, and the y pass's
    sliding-window segments depend on how many slices share a launch, which
    moves f32 roundings of the window sums."""
    from paper_2504_19417_b200.engine import predict_multi_host
    pkg = _pkg()
    W, H = 128, 96
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    reg = pkg.NormalFlowRegressor(width=W, height=H, delta_x=5, delta_y=5, weights=w)
    sizes = [3000, 0, 12000, 1, 700, 25000, 0, 4000, 9000]
    slices = [vo.synth_uniform_noise(n, W, H, seed=500 + i) if n else np.zeros((0, 3)) for i, n in enumerate(sizes)]
    ref = reg.predict_slices(slices)
    for devs in ([0, 0], [0, 0, 0]):
        got = reg.predict_slices(slices, devices=devs)
        assert len(got) == len(ref)
        for a, r in zip(got, ref):
            assert a.shape == r.shape
            np.testing.assert_allclose(a, r, rtol=0, atol=1e-6)
    e = reg.engines([0])[0]
    ev = np.ascontiguousarray(np.concatenate([s for s in slices if len(s)]))
    off = np.cumsum([0] + [len(s) for s in slices if len(s)])
    with pytest.raises(ValueError, match="distinct"):
        predict_multi_host([e, e], ev, off)


def test_strips_host_matches_unsplit_slice():
    """vkm_predict_strips_host (config 5's row-strip split from one process,
    one handle per strip, δy event halo, one time origin) against the unsplit
    slice: counts exact, flows within 1e-5 (the strips segment the window
    sums differently); out-of-sensor events stay NaN / 0."""
    from paper_2504_19417_b200.sharding import predict_strips_host
    pkg = _pkg()
    W, H, d = 200, 150, 7
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
    ev = np.ascontiguousarray(vo.synth_uniform_noise(150_000, W, H, seed=17))
    ev[5, 2] = H + 3          # outside every strip
    ev[6, 1] = W              # outside in x, inside a strip's rows
    t0 = float(ev[0, 0])
    f_ref, c_ref = eng.predict_host(ev, t0, return_counts=True)
    for k in (2, 3):
        f, c = predict_strips_host(lambda h, dev: pkg.FlowEngine(W, h, d, d, 0.016, b, w, dev), ev, t0, H, d,
                                   [0] * k, return_counts=True)
        np.testing.assert_array_equal(c, c_ref)
        assert np.isnan(f[[5, 6]]).all() and np.isnan(f_ref[[5, 6]]).all()
        good = np.isfinite(f_ref[:, 0])
        np.testing.assert_allclose(f[good], f_ref[good], rtol=0, atol=1e-5)


def test_checked_fast_path_equals_validated_path():
    """predict(X) on a large sorted slice runs vkm_predict_host_checked (one
    host pass validates and packs); its flows equal the validated path's
    bitwise, and every input the checks reject (NaN, negative time,
    non-integer or outside pixels, span > window) raises the reference's
    error exactly as before; unsorted input falls back to the sorting path."""
    pkg = _pkg()
    W, H = 346, 260
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    reg = pkg.NormalFlowRegressor(width=W, height=H, weights=w)
    X = vo.synth_uniform_noise(300_000, W, H, seed=12)
    eng = reg.engine()
    fast = eng.predict_host_checked(X, 0.032)
    assert fast is not None
    blk = pkg.block_from_array(X, W, H, 0.032)
    np.testing.assert_array_equal(fast, eng.predict_host_wide(blk.events, blk.t_start))
    np.testing.assert_array_equal(reg.predict(X), fast)
    cases = [("nan", lambda Y: Y.__setitem__((5, 0), np.nan), "non-finite"),
             ("neg", lambda Y: Y.__setitem__((0, 0), -1.0), "non-negative"),
             ("frac", lambda Y: Y.__setitem__((9, 1), 3.5), "integer-valued"),
             ("out", lambda Y: Y.__setitem__((200_000, 2), H), "outside geometry"),
             ("span", lambda Y: Y.__setitem__((len(Y) - 1, 0), 1.0), "exceeds the slice window")]
    for name, mutate, msg in cases:
        Y = X.copy()
        mutate(Y)
        assert eng.predict_host_checked(Y, 0.032) is None, name
        with pytest.raises(ValueError, match=msg):
            reg.predict(Y)
    Y = X.copy()
    Y[[10, 11]] = Y[[11, 10]]
    Y[10, 0], Y[11, 0] = X[11, 0] + 1e-9, X[10, 0]        # unsorted pair
    assert eng.predict_host_checked(Y, 0.032) is None
    got = reg.predict(Y)
    order = np.argsort(Y[:, 0], kind="stable")
    np.testing.assert_allclose(got, reg.predict(Y[order]), rtol=0, atol=0)
