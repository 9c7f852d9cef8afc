"""Wall time of predict_slices and of predict_stream over an overlapping-window stream: windows
searched and gathered on the GPU (one upload) vs windowed on the host (each
window's rows copied)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2504_19417_b200 as pkg
from paper_2504_19417_b200 import stream as S

W, H, n, dur = 640, 480, 8_000_000, 1.0
rng = np.random.default_rng(0)
t = np.sort(rng.uniform(0.0, dur, n))
st = S.EventStream(t, rng.integers(0, W, n), rng.integers(0, H, n), S.CameraGeometry(W, H))
reg = pkg.NormalFlowRegressor(width=W, height=H, weights=pkg.init_weights(64, 128, pkg.generate_bases(64), seed=0,
                                                                           dtype=np.float32))
out = {"events": n, "duration_s": dur, "window_s": 0.032}
for stride in (0.032, 0.008):
    for dev in (False, True):
        S.predict_stream(reg, st, stride=stride, device_windows=dev)
        ts = []
        for _ in range(3):
            a = time.perf_counter()
            r = S.predict_stream(reg, st, stride=stride, device_windows=dev)
            ts.append(time.perf_counter() - a)
        rows = sum(len(f) for _, f in r)
        out[f"stride{stride}_{'device' if dev else 'host'}"] = {"s": min(ts), "windows": len(r), "flows": rows,
                                                                "flows_per_s": rows / min(ts)}
# predict_slices: 64 cfg-4-shaped slices (346x260, 2e5 events each) through the pipelined host batch
W4, H4 = 346, 260
reg4 = pkg.NormalFlowRegressor(width=W4, height=H4, weights=reg.weights_ if hasattr(reg, "weights_") else
                               pkg.init_weights(64, 128, pkg.generate_bases(64), seed=0, dtype=np.float32))
sl = []
for i in range(64):
    r = np.random.default_rng(i)
    tt = np.sort(r.uniform(0, 0.032, 200_000))
    sl.append(np.stack([tt, r.integers(0, W4, len(tt)), r.integers(0, H4, len(tt))], 1).astype(np.float64))
reg4.predict_slices(sl)
ts = []
for _ in range(3):
    a = time.perf_counter()
    reg4.predict_slices(sl)
    ts.append(time.perf_counter() - a)
out["predict_slices_64x2e5"] = {"s": min(ts), "flows_per_s": 64 * 200_000 / min(ts)}
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
S.predict_stream(reg, st, stride=0.008, device_windows=True)
pr.disable(); b = io.StringIO(); pstats.Stats(pr, stream=b).sort_stats("tottime").print_stats(8)
out["profile_device_stride0.008"] = b.getvalue().splitlines()[-14:]
print(json.dumps(out))
