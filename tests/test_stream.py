"""Stream ingestion and slicing (events.py:238-387) against fixtures frozen from
the reference (tests/golden/make_golden_stream.py); streaming prediction on
the GPU against per-window predictions."""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, has_cuda
from oracle import veckm_oracle as vo


def _S():
    from paper_2504_19417_b200 import stream as S
    return S


@pytest.mark.parametrize("name", ["overlap", "disjoint", "gap", "edges", "unsorted"])
def test_slice_stream_matches_reference(name):
    S = _S()
    with np.load(os.path.join(GOLDEN, "stream_slices.npz")) as z:
        g = {k: z[k] for k in z.files}
    delta_t, stride, t0 = g[f"{name}_params"]
    st = S.EventStream(g[f"{name}_t"], g[f"{name}_x"], g[f"{name}_y"], S.CameraGeometry(64, 48))
    sl = S.slice_stream(st, float(delta_t), float(stride), float(t0))
    np.testing.assert_array_equal([s.t_start for s in sl], g[f"{name}_starts"])
    np.testing.assert_array_equal([len(s) for s in sl], g[f"{name}_lens"])
    np.testing.assert_array_equal([s.t[0] if len(s) else -1.0 for s in sl], g[f"{name}_first"])
    np.testing.assert_array_equal([int(s.x.sum()) for s in sl], g[f"{name}_xsum"])


def test_slice_stream_errors_and_empty():
    S = _S()
    st = S.EventStream(np.zeros(0), np.zeros(0, int), np.zeros(0, int), S.CameraGeometry(4, 4))
    assert S.slice_stream(st, 0.016, 0.01) == []
    with pytest.raises(ValueError, match="delta_t"):
        S.slice_stream(st, 0.0, 0.01)
    with pytest.raises(ValueError, match="stride"):
        S.slice_stream(st, 0.016, 0.0)


def test_evn1_reads_reference_file_and_round_trips(tmp_path):
    S = _S()
    st = S.load_events(os.path.join(GOLDEN, "events_small.evn1"), "binary")
    with np.load(os.path.join(GOLDEN, "events_small.npz")) as z:
        np.testing.assert_array_equal(st.t, z["t"])
        np.testing.assert_array_equal(st.x, z["x"])
        np.testing.assert_array_equal(st.y, z["y"])
        np.testing.assert_array_equal(st.polarity, z["p"])
    assert (st.geometry.width, st.geometry.height) == (346, 260)
    out = tmp_path / "rt.evn1"
    S.write_events_binary(st, str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, "events_small.evn1"), "rb").read()
    assert len(out.read_bytes()) == 12 + 17 * len(st)   # packed 17-byte records


def test_event_file_errors(tmp_path):
    S = _S()
    from paper_2504_19417_b200.errors import EventParseError, GeometryError
    bad = tmp_path / "bad.evn1"
    bad.write_bytes(b"EVN1" + (4).to_bytes(4, "little") + (4).to_bytes(4, "little") + b"\x00" * 5)
    with pytest.raises(EventParseError, match="truncated"):
        S.load_events(str(bad), "binary")
    with pytest.raises(EventParseError, match="header"):
        (tmp_path / "nohdr.evn1").write_bytes(b"XXXX")
        S.load_events(str(tmp_path / "nohdr.evn1"), "binary")
    csv = tmp_path / "ev.csv"
    csv.write_text("t,x,y\n0.001,1,2\n0.002,3,1,1\n")
    st = S.load_events(str(csv), "csv", S.CameraGeometry(4, 4))
    assert len(st) == 2 and st.polarity is not None
    csv.write_text("0.001,9,2\n")
    with pytest.raises(GeometryError, match="x=9"):
        S.load_events(str(csv), "csv", S.CameraGeometry(4, 4))
    with pytest.raises(ValueError, match="explicit geometry"):
        S.load_events(str(csv), "csv")


@pytest.mark.gpu
def test_predict_stream_matches_per_window_predictions():
    """Overlapping windows (stride < window) through one pipelined host batch:
    each window equals its own single-slice run with the window start as time
    origin (counts exact, flows to f32 rounding), and one window matches the
    CPU oracle."""
    if not has_cuda():
        pytest.fail("GPU test needs a CUDA device")
    import paper_2504_19417_b200 as pkg
    S = _S()
    W, H = 120, 90
    rng = np.random.default_rng(12)
    n = 60000
    st = S.EventStream(np.sort(rng.uniform(0.0, 0.4, n)), rng.integers(0, W, n), rng.integers(0, H, n),
                       S.CameraGeometry(W, H))
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    reg = pkg.NormalFlowRegressor(width=W, height=H, weights=w)
    res = S.predict_stream(reg, st, stride=0.01, t0=0.0)
    sl = S.slice_stream(st, 0.016, 0.01, 0.0)
    assert len(res) == len(sl)
    eng = reg.engine()
    for (t_start, flows), s in zip(res, sl):
        assert t_start == s.t_start and flows.shape == (len(s), 2)
        if len(s):
            np.testing.assert_allclose(flows, eng.predict_host(s.events(), s.t_start), rtol=0, atol=1e-5)
    s = sl[7]
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    ev = s.events()
    g = vo.accumulate(ev[:, 0] - s.t_start, s.x.astype(np.int64), s.y.astype(np.int64), W, H, 10, 10, fr, 0.016)
    q = np.arange(0, len(s), 37)
    emb, _ = vo.pool(g, vo.spatial_table(fr, 10, 10), ev[q, 0] - s.t_start, s.x[q].astype(np.int64),
                     s.y[q].astype(np.int64), fr, 0.016)
    np.testing.assert_allclose(res[7][1][q], vo.mlp(w.w1, w.b1, w.w2, w.b2, vo.to_features(emb)), rtol=0, atol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("stride,chunk", [(0.004, 0), (0.004, 3000), (0.01, 0), (0.032, 0), (0.05, 0)])
def test_device_windowing_matches_host_windowing(stride, chunk, monkeypatch):
    """vkm_window_bounds / vkm_predict_windows (windows searched and gathered on
    the GPU from one upload of the stream) equal the host-windowed batch: same
    windows and starts, flows within 1e-6 (the two paths group the windows
    into different launch batches, and the y pass's sliding-window segments
    depend on how many slices share a launch, which moves f32 roundings).
    chunk > 0: the windows are gathered and predicted in chunks of at most
    that many events (VKM_WINDOW_CHUNK_EVENTS; default 32M), one window alone
    may exceed it."""
    if chunk:
        monkeypatch.setenv("VKM_WINDOW_CHUNK_EVENTS", str(chunk))
    if not has_cuda():
        pytest.fail("GPU test needs a CUDA device")
    import paper_2504_19417_b200 as pkg
    S = _S()
    W, H = 100, 80
    rng = np.random.default_rng(31)
    n = 40000
    t = np.sort(np.concatenate([rng.uniform(0.0, 0.15, n // 2), rng.uniform(0.25, 0.4, n - n // 2)]))  # a gap
    st = S.EventStream(t, rng.integers(0, W, n), rng.integers(0, H, n), S.CameraGeometry(W, H))
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    reg = pkg.NormalFlowRegressor(width=W, height=H, weights=w)
    dev = S.predict_stream(reg, st, stride=stride, t0=0.0, device_windows=True)
    host = S.predict_stream(reg, st, stride=stride, t0=0.0, device_windows=False)
    ref = S.slice_stream(st, 0.016, stride, 0.0)
    assert len(dev) == len(host) == len(ref)
    for (sd, fd), (sh, fh), r in zip(dev, host, ref):
        assert sd == sh == r.t_start and fd.shape == fh.shape == (len(r), 2)
        np.testing.assert_allclose(fd, fh, rtol=0, atol=1e-6)


def test_device_window_starts_follow_the_reference_loop():
    """The starts uploaded for device windowing are the reference loop's
    float sequence (events.py:363-368), the same as the host windowing's,
    before trailing empty windows are dropped."""
    S = _S()
    from paper_2504_19417_b200.stream import _window_starts
    rng = np.random.default_rng(3)
    for stride in (0.004, 0.01, 0.032, 0.1 / 3):
        t = np.sort(rng.uniform(0.0, 0.4, 5000))
        starts = _window_starts(t, stride, 0.0)
        wins = S.window_bounds(t, 0.016, stride, 0.0)
        assert [s for _, _, s in wins] == list(starts[:len(wins)])
        assert starts[-1] <= t[-1] < starts[-1] + stride


def test_csv_parser_matches_reference_outcomes(tmp_path):
    """The columnar CSV reader against the reference's own outcomes
    (tests/golden/make_golden_csv.py): parsed columns bit-exact, or the same
    exception type and message (first offending line, then the check order
    within the line)."""
    import json
    S = _S()
    from paper_2504_19417_b200 import errors as E
    with open(os.path.join(GOLDEN, "csv_cases.json")) as fh:
        cases = json.load(fh)
    g = S.CameraGeometry(16, 12)
    for name, c in cases.items():
        path = tmp_path / f"{name}.csv"
        path.write_text(c["text"], encoding="utf-8")
        if c["ok"]:
            st = S.load_events(str(path), "csv", g)
            assert [repr(v) for v in st.t.tolist()] == c["t"], name
            assert st.x.tolist() == c["x"] and st.y.tolist() == c["y"], name
            assert (None if st.polarity is None else st.polarity.tolist()) == c["p"], name
        else:
            with pytest.raises(getattr(E, c["type"])) as ei:
                S.load_events(str(path), "csv", g)
            assert str(ei.value).replace(str(path), "<path>") == c["message"], name


def test_csv_writer_round_trips(tmp_path):
    S = _S()
    rng = np.random.default_rng(9)
    st = S.EventStream(np.sort(rng.uniform(0, 1, 500)), rng.integers(0, 16, 500), rng.integers(0, 12, 500),
                       S.CameraGeometry(16, 12), rng.choice([0, 1, -1], 500))
    S.write_events_csv(st, str(tmp_path / "a.csv"))
    lines = (tmp_path / "a.csv").read_text().splitlines()
    assert lines[3] == f"{float(st.t[3])!r},{st.x[3]},{st.y[3]},{st.polarity[3]}"   # events.py:294-302 format
    back = S.load_events(str(tmp_path / "a.csv"), "csv", S.CameraGeometry(16, 12))
    np.testing.assert_array_equal(back.t, st.t)
    np.testing.assert_array_equal(back.polarity, st.polarity)
    pos = S.filter_polarity(st, "pos")
    assert (pos.polarity > 0).all() and len(pos) + len(S.filter_polarity(st, "neg")) == len(st)


def test_event_slice_checks():
    """EventSlice construction checks (events.py:106-131)."""
    S = _S()
    from paper_2504_19417_b200.errors import GeometryError
    g = S.CameraGeometry(8, 8)
    s = S.EventSlice([0.0, 0.01], [1, 2], [3, 4], 0.0, 0.032, g)
    assert s.n == 2 and s.events().shape == (2, 3)
    with pytest.raises(ValueError, match="window must be positive"):
        S.EventSlice([0.0], [1], [1], 0.0, 0.0, g)
    with pytest.raises(ValueError, match="fall outside"):
        S.EventSlice([0.0, 0.05], [1, 2], [3, 4], 0.0, 0.032, g)
    with pytest.raises(ValueError, match="sorted ascending"):
        S.EventSlice([0.01, 0.0], [1, 2], [3, 4], 0.0, 0.032, g)
    with pytest.raises(GeometryError, match="outside geometry"):
        S.EventSlice([0.0], [9], [1], 0.0, 0.032, g)
    S.EventSlice([0.032 + 1e-18], [1], [1], 0.0, 0.032, g)   # ulp slack at the upper edge
