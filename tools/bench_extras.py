"""Throughput of the non-headline paths on one GPU (device-timed, CUDA events):
precision="f64" predict at config 2, and the GPU head trainer (samples/s).
Prints one JSON line."""
import json, os, sys, time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_19417_b200 as pkg  # noqa: E402
from oracle import veckm_oracle as vo  # noqa: E402  (synthetic input generator only)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


W, H, n = 640, 480, 1_000_000
X = vo.synth_uniform_noise(n, W, H, seed=0)
b = pkg.generate_bases(64)
w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
eng = pkg.FlowEngine(W, H, 10, 10, 0.016, b, w)
ev = torch.from_numpy(X).cuda()
t0 = float(X[0, 0])
f32 = torch.empty((n, 2), dtype=torch.float32, device="cuda")
f64 = torch.empty((n, 2), dtype=torch.float64, device="cuda")
ms32 = timed(lambda: eng.predict_device(ev, t0, flows=f32), 20)
ms64 = timed(lambda: eng.predict_device_f64(ev, t0, flows=f64), 5)

# the drop-in call: NormalFlowRegressor.predict(X) on a pageable numpy slice
# (host validation, copies, kernels, float64 result), wall clock
reg = pkg.NormalFlowRegressor(width=W, height=H, weights=w)
reg.predict(X)
t = time.perf_counter()
for _ in range(5):
    reg.predict(X)
predict_ms = (time.perf_counter() - t) / 5 * 1e3
t = time.perf_counter()
for _ in range(5):
    pkg.block_from_array(X, W, H, 0.032)
validate_ms = (time.perf_counter() - t) / 5 * 1e3

# trainer: 200k samples, D = 64 (128 features), hidden 128, batch 512
m = 200_000
rng = np.random.default_rng(0)
feats = rng.uniform(-1, 1, size=(m, 128))
u = rng.normal(0, 10, size=(m, 2))
tc = pkg.TrainConfig(hidden=128, epochs=5, batch_size=512, learning_rate=1e-3, seed=0)
torch.cuda.synchronize()
t = time.perf_counter()
pkg.train_head(None, W, H, 10, 10, 0.016, 64, tc, b, features=(feats, u))
torch.cuda.synchronize()
tr_s = time.perf_counter() - t
train_samples = 5 * (m - int(m * 0.2))
print(json.dumps({"cfg2_f32_flows_per_s": n / (ms32 / 1e3), "cfg2_f64_flows_per_s": n / (ms64 / 1e3),
                  "dropin_predict_ms_1M": predict_ms, "dropin_validate_ms_1M": validate_ms,
                  "f64_ms": ms64, "f32_ms": ms32,
                  "train_samples_per_s": train_samples / tr_s, "train_wall_s": tr_s,
                  "train_config": "200k samples (160k train), 128 features, hidden 128, batch 512, 5 epochs, wall clock incl. per-epoch validation"}))
