"""Wall time of predict_stream over an overlapping-window stream: windows
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
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
S.predict_stream(reg, st, stride=0.008, device_windows=True)
pr.disable(); b = io.StringIO(); pstats.Stats(pr, stream=b).sort_stats("tottime").print_stats(8)
out["profile_device_stride0.008"] = b.getvalue().splitlines()[-14:]
print(json.dumps(out))
