"""CPU tests of the host side: input contract, weight formats, estimator API
semantics, and the C-ABI library's exports.  No kernel is launched here."""

import ctypes
import os

import numpy as np
import pytest
from sklearn.base import clone
from sklearn.exceptions import NotFittedError

from conftest import GOLDEN, load_golden
import paper_2504_19417_b200 as pkg
from paper_2504_19417_b200 import _lib
from paper_2504_19417_b200.validation import block_from_array, check_events
from paper_2504_19417_b200.weights import bases_from_bytes, bases_to_bytes


def make_events(rng, n=50, width=64, height=64, window=0.03):
    t = np.sort(rng.uniform(0, window, n))
    return np.stack([t, rng.integers(0, width, n), rng.integers(0, height, n)], axis=1)


# ---------------------------------------------------------------- C-ABI ----

def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _lib.declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES)


def test_library_version_and_no_cpu_fallback():
    lib = _lib.load()
    assert lib.vkm_version() == 1
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    # without a device the create call must fail loudly (no CPU path)
    p = _lib.VkmParams(8, 8, 2, 2, 8, 0, 0.016, 0, 0)
    h = ctypes.c_void_p()
    T = np.zeros(8)
    ptr = T.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    rc = lib.vkm_create(ctypes.byref(h), ctypes.byref(p), ptr, ptr, ptr, None, None, None, None)
    assert rc != 0
    with pytest.raises(RuntimeError):
        _lib.check(rc)


def test_create_rejects_bad_params_before_touching_the_device():
    lib = _lib.load()
    T = np.zeros(8)
    ptr = T.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    h = ctypes.c_void_p()
    for bad, exc in [((0, 8, 2, 2, 8, 0, 0.016), ValueError), ((8, 8, 0, 2, 8, 0, 0.016), ValueError),
                     ((8, 8, 2, 2, 8, 0, 0.0), ValueError), ((8, 8, 2, 2, 65, 0, 0.016), NotImplementedError),
                     ((8, 8, 2, 2, 8, 4, 0.016), ValueError)]:
        p = _lib.VkmParams(*bad, 0, 0)
        rc = lib.vkm_create(ctypes.byref(h), ctypes.byref(p), ptr, ptr, ptr, None, None, None, None)
        with pytest.raises(exc):
            _lib.check(rc)


# ------------------------------------------------------- input contract ----

def test_check_event_array_types(rng):
    X = make_events(rng, n=5)
    X3, x, y = check_events(X, 64, 64)
    assert X3.dtype == np.float64 and x.dtype == np.int32


@pytest.mark.parametrize("X,match", [
    (np.zeros((3,)), "shape"),
    (np.array([[0.0, 1.5, 2.0]]), "integer"),
    (np.array([[np.nan, 1.0, 2.0]]), "non-finite"),
    (np.array([[-1.0, 1.0, 2.0]]), "non-negative"),
    (np.array([[0.0, 9.0, 2.0]]), "outside geometry"),
])
def test_validation_messages(X, match):
    with pytest.raises(ValueError, match=match):
        check_events(X, 8, 8)


def test_slice_sorts_stably_and_checks_span():
    X = np.array([[0.02, 1, 1], [0.01, 2, 2], [0.01, 3, 3]])
    b = block_from_array(X, 8, 8, 0.032)
    assert b.events[:, 0].tolist() == [0.01, 0.01, 0.02]
    assert b.events[:, 1].tolist() == [2, 3, 1]
    assert b.t_start == 0.01
    with pytest.raises(ValueError, match="window"):
        block_from_array(np.array([[0.0, 1, 1], [0.5, 1, 1]]), 8, 8, 0.032)
    # strict f64 span check (validation.py:59-64)
    with pytest.raises(ValueError, match="window"):
        block_from_array(np.array([[5.0, 1, 1], [5.032, 1, 1]]), 8, 8, 0.032)


def test_slice_matches_golden_sorting(golden_case):
    g = golden_case
    b = block_from_array(g["X"], int(g["width"]), int(g["height"]), 2 * float(g["delta_t"]))
    np.testing.assert_array_equal(b.events[:, 0], g["sorted_t"])
    np.testing.assert_array_equal(b.events[:, 1].astype(np.int32), g["sorted_x"])
    np.testing.assert_array_equal(b.events[:, 2].astype(np.int32), g["sorted_y"])
    assert b.t_start == float(g["t_start"])


# --------------------------------------------------------------- weights ----

def test_generate_bases_matches_reference_golden():
    g = load_golden("rng_bases")
    b = pkg.generate_bases(64, 25.0, (0, 1, 2))
    np.testing.assert_array_equal(b.time_freqs, g["T"])
    np.testing.assert_array_equal(b.x_freqs, g["X"])
    np.testing.assert_array_equal(b.y_freqs, g["Y"])
    np.testing.assert_array_equal(pkg.generate_bases(48, 9.0, (7, 8, 9)).time_freqs, g["T_s789_d48"])


def test_load_reference_weight_file_and_roundtrip(tmp_path):
    w = pkg.load_weights(os.path.join(GOLDEN, "cfg1_weights.vkmw"))
    g = load_golden("cfg1_20k")
    np.testing.assert_array_equal(w.w1, g["w1"])
    np.testing.assert_array_equal(w.b2, g["b2"])
    np.testing.assert_array_equal(w.bases.time_freqs, g["freqT"])
    out = tmp_path / "rt.vkmw"
    pkg.save_weights(w, str(out))
    with open(out, "rb") as a, open(os.path.join(GOLDEN, "cfg1_weights.vkmw"), "rb") as b:
        assert a.read() == b.read()


def test_bases_block_roundtrip():
    b = pkg.generate_bases(48, 9.0, (4, 5, 6))
    buf = bases_to_bytes(b)
    assert len(buf) == 16 + 3 * 48 * 8
    b2, pos = bases_from_bytes(buf)
    assert pos == len(buf) and b2.sigma2 == 9.0
    np.testing.assert_array_equal(b2.y_freqs, b.y_freqs)


def test_bad_weight_files(tmp_path):
    p = tmp_path / "bad.vkmw"
    p.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(pkg.EventParseError):
        pkg.load_weights(str(p))


def test_init_weights_matches_golden():
    g = load_golden("cfg1_20k")
    b = pkg.Bases(g["freqT"], g["freqX"], g["freqY"], 25.0)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    np.testing.assert_array_equal(w.w1, g["w1"])
    np.testing.assert_array_equal(w.w2, g["w2"])


def test_weights_shape_checks():
    b = pkg.generate_bases(4)
    with pytest.raises(pkg.DimensionMismatchError):
        pkg.MlpWeights(np.zeros((3, 6)), np.zeros(3), np.zeros((2, 3)), np.zeros(2), b)
    with pytest.raises(ValueError):
        pkg.MlpWeights(np.full((3, 8), np.nan), np.zeros(3), np.zeros((2, 3)), np.zeros(2), b)


# ------------------------------------------------------------ estimators ----

def test_estimator_params_clone():
    reg = pkg.NormalFlowRegressor(delta_x=4, width=64, height=64)
    assert reg.get_params()["delta_x"] == 4
    c = clone(reg)
    assert c.get_params() == reg.get_params()
    enc = pkg.LocalEventEncoder(embed_dim=16)
    enc.set_params(embed_dim=8)
    assert enc.get_params()["embed_dim"] == 8


def test_estimator_errors_raised_before_the_device(rng):
    with pytest.raises(NotFittedError):
        pkg.NormalFlowRegressor().predict(make_events(rng))
    with pytest.raises(NotFittedError):
        pkg.LocalEventEncoder().transform(make_events(rng))
    b = pkg.generate_bases(16)
    w = pkg.init_weights(16, 8, b, dtype=np.float32)
    with pytest.raises(pkg.DimensionMismatchError):
        pkg.NormalFlowRegressor(embed_dim=64, weights=w).predict(make_events(rng))
    with pytest.raises(ValueError, match="precision"):
        pkg.NormalFlowRegressor(embed_dim=16, precision="f16", weights=w).predict(make_events(rng))
    # training (GPU) validates its targets on the host first (estimators.py:171-181)
    with pytest.raises(ValueError, match="flow targets"):
        pkg.NormalFlowRegressor(embed_dim=16).fit(make_events(rng), np.zeros((3, 2)))
    with pytest.raises(ValueError, match="pair one flow array"):
        pkg.NormalFlowRegressor(embed_dim=16).fit([make_events(rng)], [np.zeros((3, 2)), np.zeros((3, 2))])
    # pretrained weights: fit only stores them (estimators.py:166-170)
    reg = pkg.NormalFlowRegressor(embed_dim=16, weights=w).fit(None, None)
    assert reg.weights_ is w
    with pytest.raises(ValueError, match="outside geometry"):
        pkg.LocalEventEncoder(width=8, height=8).fit(np.array([[0.0, 9.0, 1.0]]))


def test_reference_weights_object_is_accepted():
    class Duck:
        pass
    b = pkg.generate_bases(8)
    d = Duck()
    d.w1, d.b1, d.w2, d.b2 = np.zeros((4, 16)), np.zeros(4), np.zeros((2, 4)), np.ones(2)
    d.bases = b
    reg = pkg.NormalFlowRegressor(embed_dim=8, weights=d)
    assert reg._resolve_pretrained().hidden == 4


def test_native_event_check_matches_numpy_semantics():
    """vkm_check_events (one pass, AVX-512 body + scalar tail) against the
    numpy predicates of validation.py:10-37 on adversarial arrays."""
    import ctypes
    from paper_2504_19417_b200 import _lib, validation as v
    lib = _lib.load()
    rng = np.random.default_rng(11)
    W, H = 40, 30
    for trial in range(300):
        n = int(rng.integers(0, 70))
        cols = 3 if trial % 3 else 4                       # (n, 4) rows: the strided scalar path
        X = np.stack([np.sort(rng.uniform(0, 0.03, n)), rng.integers(-2, W + 2, n), rng.integers(-2, H + 2, n)]
                     + ([rng.uniform(size=n)] if cols == 4 else []), 1).astype(np.float64)
        for _ in range(int(rng.integers(0, 3))):           # sprinkle defects
            if n == 0:
                break
            i, kind = int(rng.integers(0, n)), int(rng.integers(0, 7))
            if kind == 0:
                X[i, int(rng.integers(0, 3))] = np.nan
            elif kind == 1:
                X[i, int(rng.integers(0, 3))] = -np.inf
            elif kind == 2:
                X[i, 0] = -1e-3
            elif kind == 3:
                X[i, 1 + int(rng.integers(0, 2))] += 0.5
            elif kind == 4:
                X[i, 1] = 3e9                              # out of int32 range
            elif kind == 5:
                X[i, 0] = 0.05 * rng.uniform()             # breaks the order
            else:
                X[i, 2] = 2.0 ** 60                        # huge but integer-valued
        _assert_check_matches(lib, X, W, H)


def _assert_check_matches(lib, X, W, H):
    import ctypes
    from paper_2504_19417_b200 import validation as v
    n, cols = X.shape
    c = v._EventCheck()
    assert lib.vkm_check_events(X.ctypes.data, n, cols, W, H, ctypes.byref(c)) == 0
    X3 = X[:, :3]
    t, x, y = X3[:, 0], X3[:, 1], X3[:, 2]
    fin = np.isfinite(X3).all(axis=1)
    assert bool(c.nonfinite) == (not fin.all())
    assert bool(c.negative_t) == bool(np.any(t < 0))
    with np.errstate(invalid="ignore"):
        nonint = bool(np.any(fin & ((x != np.round(x)) | (y != np.round(y)))))
        xi, yi = x.astype(np.int32), y.astype(np.int32)
    assert bool(c.nonint) == nonint
    with np.errstate(invalid="ignore"):
        assert bool(c.sorted) == (not np.any(np.diff(t) < 0))
    outside = fin & ~((xi >= 0) & (xi < W) & (yi >= 0) & (yi < H))
    if outside.any():
        k = int(np.flatnonzero(outside)[0])
        assert (c.first_outside, c.outside_x, c.outside_y) == (k, xi[k], yi[k])
    else:
        assert c.first_outside == -1
    if n:
        assert (c.t_first, c.t_last) == (X[0, 0], X[-1, 0]) or np.isnan(X[[0, -1], 0]).any()


def test_native_event_check_parallel_parts():
    """Large inputs are checked in contiguous parts on the host pool and
    merged: defects placed on and around part boundaries (order breaks
    across a boundary, the first outside pixel in a late part while an
    earlier part is clean) give the serial pass's answer."""
    from paper_2504_19417_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(12)
    W, H = 64, 48
    for trial in range(12):
        n = int(rng.integers(1 << 18, 1 << 20))
        X = np.stack([np.sort(rng.uniform(0, 0.03, n)), rng.integers(0, W, n), rng.integers(0, H, n)],
                     1).astype(np.float64)
        cuts = [n * k // 16 for k in range(1, 16)] + [n * k // 64 for k in range(1, 64, 7)]
        for _ in range(int(rng.integers(0, 4))):
            i = int(np.clip(rng.choice(cuts) + int(rng.integers(-2, 2)), 1, n - 1))
            kind = int(rng.integers(0, 5))
            if kind == 0:
                X[i, 0] = X[i - 1, 0] - 1e-9                # order break at / near a boundary
            elif kind == 1:
                X[i, 1] = W + int(rng.integers(0, 3))       # outside
            elif kind == 2:
                X[i, 2] = np.nan
            elif kind == 3:
                X[i, 1] += 0.25
            else:
                X[i, 0] = -1.0
        _assert_check_matches(lib, X, W, H)


def test_fused_check_pack_matches_check_and_records():
    """vkm_host::check_pack (the drop-in call's one pass: checks + 8-byte
    records, AVX-512 body between a scalar head and tail) gives
    vkm_check_events' answer and the records k_prep would build: f32 bits of
    (t - t0)/dt and x | y << 16, or 0xFFFFFFFF for rows outside the image or
    not integral; records written at every alignment of the output."""
    import ctypes
    from paper_2504_19417_b200 import _lib, validation as v
    lib = _lib.load()
    fn = lib.vkm_debug_check_pack
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                   ctypes.c_void_p, ctypes.c_void_p]
    rng = np.random.default_rng(21)
    W, H = 40, 30
    for trial in range(200):
        n = int(rng.integers(0, 400)) if trial % 4 else int(rng.integers(1000, 5000))
        X = np.stack([np.sort(rng.uniform(0, 0.03, n)), rng.integers(-2, W + 2, n), rng.integers(-2, H + 2, n)],
                     1).astype(np.float64)
        for _ in range(int(rng.integers(0, 4))):
            if n == 0:
                break
            i, kind = int(rng.integers(0, n)), int(rng.integers(0, 7))
            if kind == 0:
                X[i, 1 + int(rng.integers(0, 2))] = np.nan
            elif kind == 1:
                X[i, 1] = -np.inf
            elif kind == 2:
                X[i, 0] = -1e-3
            elif kind == 3:
                X[i, 1 + int(rng.integers(0, 2))] += 0.5
            elif kind == 4:
                X[i, 1] = 3e9
            elif kind == 5:
                X[i, 0] = 0.05 * rng.uniform()
            else:
                X[i, 2] = -0.0
        t0, dt = (X[0, 0] if n else 0.0), 1e-3
        shift = trial % 4                                  # record alignment: 8-byte steps inside a 32-byte line
        buf = np.zeros(2 * (n + 8), dtype=np.uint32)
        out = buf[2 * shift: 2 * (shift + n)]
        c = v._EventCheck()
        assert fn(X.ctypes.data, n, t0, dt, W, H, out.ctypes.data, ctypes.byref(c)) == 0
        ref = v._EventCheck()
        assert lib.vkm_check_events(X.ctypes.data, n, 3, W, H, ctypes.byref(ref)) == 0
        for f in ("nonfinite", "negative_t", "nonint", "sorted", "first_outside", "outside_x", "outside_y"):
            assert getattr(c, f) == getattr(ref, f), (trial, f)
        if n:
            assert (c.t_first, c.t_last) == (ref.t_first, ref.t_last)
        rec = out.reshape(-1, 2)
        with np.errstate(invalid="ignore"):
            a = ((X[:, 0] - t0) / dt).astype(np.float32).view(np.uint32)
            x, y = X[:, 1], X[:, 2]
            ok = (x >= 0) & (x < W) & (y >= 0) & (y < H) & (x == np.floor(x)) & (y == np.floor(y))
            xy = np.where(ok, np.nan_to_num(x).astype(np.int64) | (np.nan_to_num(y).astype(np.int64) << 16),
                          0xFFFFFFFF).astype(np.uint32)
        assert np.array_equal(rec[:, 0], a), trial
        assert np.array_equal(rec[:, 1], xy), trial


def test_product_path_does_not_import_the_oracle():
    """oracle/ is test infrastructure only: importing the package and building
    an estimator pulls in nothing from it (run in a fresh interpreter)."""
    import subprocess, sys, os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); import paper_2504_19417_b200 as p; "
            "import paper_2504_19417_b200.bindings, paper_2504_19417_b200.stream, paper_2504_19417_b200.sharding, "
            "paper_2504_19417_b200.training; p.NormalFlowRegressor(); "
            "bad = [m for m in sys.modules if m == 'oracle' or m.startswith('oracle.')]; "
            "assert not bad, bad") % root
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]


def test_native_widening_matches_astype():
    """vkm_widen_f32 (pooled, streaming stores, scalar head until the
    destination is 64-byte aligned) equals numpy's astype(float64), NaN and
    infinities included, for sizes around the pool threshold and misaligned
    destinations."""
    import ctypes
    from paper_2504_19417_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(4)
    for n in (0, 1, 7, 8, 9, 1000, (1 << 19) - 3, (1 << 19) + 5, 3_000_001):
        src = rng.standard_normal(n).astype(np.float32)
        if n > 10:
            src[[1, 5, n - 1]] = [np.nan, np.inf, -np.inf]
        buf = np.empty(n + 3, dtype=np.float64)
        for off in (0, 1, 3):
            dst = buf[off:off + n]
            assert lib.vkm_widen_f32(src.ctypes.data, dst.ctypes.data, n) == 0
            np.testing.assert_array_equal(dst, src.astype(np.float64))


def test_native_concat_rows_matches_numpy():
    """vkm_concat_rows (pooled copy of row blocks into one buffer, parts that
    straddle block borders) equals np.concatenate, empty blocks included."""
    from paper_2504_19417_b200._staging import concat_rows
    rng = np.random.default_rng(6)
    for sizes in ([0], [5], [3, 0, 7], [200_000, 1, 0, 150_000, 33], [1] * 1000, [300_001, 299_999]):
        blocks = [rng.standard_normal((n, 3)) for n in sizes]
        dst = np.empty((sum(sizes), 3))
        concat_rows(blocks, dst)
        np.testing.assert_array_equal(dst, np.concatenate(blocks) if sizes else dst)


def test_estimator_pickles_after_use():
    """Handles are dropped on pickling / deepcopy (rebuilt lazily), so a used
    estimator stays picklable like the reference's."""
    import copy
    import pickle
    import paper_2504_19417_b200 as pkg
    b = pkg.generate_bases(8, 25.0, (0, 1, 2))
    w = pkg.init_weights(8, 16, b, seed=0)
    reg = pkg.NormalFlowRegressor(embed_dim=8, hidden=16, weights=w)
    reg.weights_ = w
    reg._engine_cache = (("k",), w, object())        # stand-ins for libveckm handles
    reg._device_engines = {("k", 0): (w, object())}
    back = pickle.loads(pickle.dumps(reg))
    assert not hasattr(back, "_engine_cache") and not hasattr(back, "_device_engines")
    np.testing.assert_array_equal(back.weights_.w1, w.w1)
    assert copy.deepcopy(reg).get_params()["embed_dim"] == 8


def test_engine_cache_is_per_thread_and_bounded():
    import threading
    from paper_2504_19417_b200.engine import EngineCache

    class Fake:
        closed = 0

        def close(self):
            Fake.closed += 1
    cache = EngineCache(size=2)
    a = cache.get("a", Fake)
    assert cache.get("a", Fake) is a
    cache.get("b", Fake)
    cache.get("c", Fake)                 # evicts "a" (least recently used)
    assert Fake.closed == 1
    assert cache.get("a", Fake) is not a
    other = []
    th = threading.Thread(target=lambda: other.append(cache.get("b", Fake)))
    th.start()
    th.join()
    assert other[0] is not cache.get("b", Fake)   # another thread, another handle


def test_encoder_fit_checks_precision():
    import paper_2504_19417_b200 as pkg
    with pytest.raises(ValueError, match="precision"):
        pkg.LocalEventEncoder(precision="f16").fit()


def test_reference_signature_helpers():
    """check_event_array(X, geometry) / slice_from_array(X, geometry, window)
    keep the reference's signatures and return types (validation.py:10-65)."""
    import paper_2504_19417_b200 as pkg
    g = pkg.CameraGeometry(8, 6)
    X = np.array([[0.02, 1, 2], [0.01, 3, 4], [0.01, 5, 5]])
    t, x, y = pkg.check_event_array(X, g)
    assert t.dtype == np.float64 and x.dtype == np.int32 and y.dtype == np.int32
    np.testing.assert_array_equal(x, [1, 3, 5])
    sl = pkg.slice_from_array(X, g, 0.032)
    assert isinstance(sl, pkg.EventSlice) and sl.geometry == g and sl.window == 0.032
    np.testing.assert_array_equal(sl.t, [0.01, 0.01, 0.02])          # stable time sort
    np.testing.assert_array_equal(sl.x, [3, 5, 1])
    assert sl.t_start == 0.01
    with pytest.raises(ValueError, match="outside geometry 8x6"):
        pkg.check_event_array(np.array([[0.0, 8, 0]]), g)
    with pytest.raises(ValueError, match="exceeds the slice window"):
        pkg.slice_from_array(np.array([[0.0, 1, 1], [0.5, 1, 1]]), g, 0.032)

    class RefGeometry:   # duck-typed (e.g. evflow.CameraGeometry)
        width, height = 8, 6
    assert len(pkg.slice_from_array(X, RefGeometry(), 0.032)) == 3


def test_bench_reference_arm_line_matches_b200_config():
    """`bench.py --impl reference` prints the contract's line with the same
    `config` as the b200 arm (so the driver can pair the two arms)."""
    import json
    import subprocess
    import sys
    import argparse
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--workload", "cfg1",
                          "--steps", "1", "--warmup", "0", "--ref-budget", "2"], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "flows/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    sys.path.insert(0, root)
    import bench
    args = argparse.Namespace(workload="cfg1", slices=0, split="slices", mlp_mode="auto")
    assert line["config"] == bench.bench_config(args, 1)
    a4 = argparse.Namespace(workload="cfg4", slices=0, split="slices", mlp_mode="auto")
    c4 = bench.bench_config(a4, 8)   # config 4: the 1000 slices split over 8 ranks
    assert c4["slices_total_per_step"] == 1000 and c4["slices_per_rank_per_step"] == 125
