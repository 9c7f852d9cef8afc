import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2504_19417_b200 as pkg
from paper_2504_19417_b200.validation import block_from_array
W, H = 640, 480
reg = pkg.NormalFlowRegressor(width=W, height=H, weights=pkg.init_weights(64, 128, pkg.generate_bases(64), seed=0, dtype=np.float32))
r = np.random.default_rng(0); n = 1_000_000
t = np.sort(r.uniform(0, 0.032, n))
X = np.stack([t, r.integers(0, W, n), r.integers(0, H, n)], 1).astype(np.float64)
for _ in range(3): reg.predict(X)
eng = reg.engine()
def tm(f, k=10):
    ts = []
    for _ in range(k):
        a = time.perf_counter(); f(); ts.append(time.perf_counter() - a)
    return round(min(ts) * 1e3, 3), round(float(np.median(ts)) * 1e3, 3)
blk = block_from_array(X, W, H, 0.032)
fl = eng.predict_host(blk.events, blk.t_start)
print("predict(X) ms", tm(lambda: reg.predict(X)))
print("block_from_array", tm(lambda: block_from_array(X, W, H, 0.032)))
print("predict_host", tm(lambda: eng.predict_host(blk.events, blk.t_start)))
print("astype", tm(lambda: fl.astype(np.float64)))
print("predict_host_wide", tm(lambda: eng.predict_host_wide(blk.events, blk.t_start)))
print("events contiguous?", blk.events.flags.c_contiguous, blk.events.dtype, blk.events is X)
import os
print("VKM_HOST_PACK_SINGLE", os.environ.get("VKM_HOST_PACK_SINGLE"))
print("encode_host", tm(lambda: eng.encode_host(blk.events, blk.t_start), 5))
print("predict_host_f64", tm(lambda: eng.predict_host_f64(blk.events, blk.t_start), 5))
print("encode_host_f64", tm(lambda: eng.encode_host_f64(blk.events, blk.t_start), 3))
