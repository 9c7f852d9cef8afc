import sys, os, time, numpy as np
sys.path.insert(0, ".")
import paper_2504_19417_b200 as pkg
W, H = 640, 480
reg = pkg.NormalFlowRegressor(width=W, height=H, weights=pkg.init_weights(64, 128, pkg.generate_bases(64), seed=0, dtype=np.float32))
r = np.random.default_rng(0); n = 1_000_000
t = np.sort(r.uniform(0, 0.032, n))
X = np.stack([t, r.integers(0, W, n), r.integers(0, H, n)], 1).astype(np.float64)
for _ in range(5): reg.predict(X)
ts=[]
for _ in range(10):
    a=time.perf_counter(); reg.predict(X); ts.append(time.perf_counter()-a)
print("predict(X) ms min/med", min(ts)*1e3, np.median(ts)*1e3, file=sys.stderr)
