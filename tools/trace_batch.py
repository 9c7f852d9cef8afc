"""VKM_TRACE timeline of one vkm_predict_batch_host call (32 cfg2 slices, pinned host buffers)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2504_19417_b200 as pkg
W, H, n, K = 640, 480, 1_000_000, 32
reg = pkg.NormalFlowRegressor(width=W, height=H, weights=pkg.init_weights(64, 128, pkg.generate_bases(64), seed=0, dtype=np.float32))
eng = reg.engine()
r = np.random.default_rng(0)
t = np.sort(r.uniform(0, 0.032, n))
X = np.stack([t, r.integers(0, W, n), r.integers(0, H, n)], 1).astype(np.float64)
ev = torch.empty((K * n, 3), dtype=torch.float64).pin_memory().numpy()
out = torch.empty((K * n, 2), dtype=torch.float32).pin_memory().numpy()
for k in range(K):
    ev[k * n:(k + 1) * n] = X
offs = np.arange(K + 1, dtype=np.int64) * n
ts = np.full(K, X[0, 0])
for _ in range(3):
    eng.predict_batch_host(ev, offs, ts, flows=out)
a = time.perf_counter()
eng.predict_batch_host(ev, offs, ts, flows=out)
print("call ms", (time.perf_counter() - a) * 1e3, "flows/s %.3e" % (K * n / (time.perf_counter() - a)), file=sys.stderr)
