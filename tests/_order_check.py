"""Subprocess body of test_gpu_parity.test_pixel_order_is_the_stable_argsort:
K1's pixel-major event order vs np.argsort(kind="stable") (encoder.py:255-259)
and the hottest pixel's flows vs the oracle.  Usage: python _order_check.py hot|hotrow|dense"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2504_19417_b200 as pkg  # noqa: E402
from oracle import veckm_oracle as vo  # noqa: E402  (checker only)


def main(case):
    W, H = 96, 64
    rng = np.random.default_rng(77)
    if case == "hot":
        X = vo.synth_uniform_noise(30000, W, H, seed=77)
        hot = [(5, 5, 40), (50, 30, 700), (70, 10, 5000), (20, 60, 9000), (3, 3, 257), (4, 3, 256)]
        extra = [np.stack([rng.uniform(0.0, 0.032, k), np.full(k, x), np.full(k, y)], 1) for x, y, k in hot]
        X = np.concatenate([X] + extra)
        X = X[np.argsort(X[:, 0], kind="stable")]
        xs, ys = 70, 10
    elif case == "hotrow":   # 64 adjacent runs of 300 events: more long runs than one run-sort block step sorts together
        X = vo.synth_uniform_noise(20000, W, H, seed=79)
        extra = [np.stack([rng.uniform(0.0, 0.032, 300), np.full(300, x), np.full(300, 40)], 1) for x in range(16, 80)]
        X = np.concatenate([X] + extra)
        X = X[np.argsort(X[:, 0], kind="stable")]
        xs, ys = 47, 40
    else:   # 35 events per pixel (the config-5 density), > 1M events
        W, H = 192, 160
        X = vo.synth_uniform_noise(35 * W * H, W, H, seed=78)
        xs, ys = 40, 30
    X[17] = [X[17, 0], W + 3, 2]        # an event outside the sensor: no slot
    b = pkg.generate_bases(64)
    w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
    eng = pkg.FlowEngine(W, H, 6, 6, 0.016, b, w)
    ev = torch.from_numpy(X).cuda()
    start, order = eng.pixel_order_device(ev, float(X[0, 0]))
    torch.cuda.synchronize()
    inside = X[:, 1] < W
    key = (X[:, 2] * W + X[:, 1]).astype(np.int64)
    key[~inside] = W * H
    want = np.argsort(key, kind="stable")
    counts = np.bincount(key, minlength=W * H + 1)
    want_start = np.concatenate([[0], np.cumsum(counts[:W * H])])
    np.testing.assert_array_equal(start.cpu().numpy(), want_start)
    got = order.cpu().numpy()
    m = int(inside.sum())
    np.testing.assert_array_equal(got[:m], want[:m])
    assert (got[m:] == -1).all()
    f1, c1 = eng.predict_host(X, float(X[0, 0]), return_counts=True)
    q = np.flatnonzero((X[:, 1] == xs) & (X[:, 2] == ys))[::7]
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    t0 = float(X[0, 0])
    ok = inside
    g = vo.accumulate(X[ok, 0] - t0, X[ok, 1].astype(np.int64), X[ok, 2].astype(np.int64), W, H, 6, 6, fr, 0.016)
    emb, c = vo.pool(g, vo.spatial_table(fr, 6, 6), X[q, 0] - t0, X[q, 1].astype(np.int64), X[q, 2].astype(np.int64),
                     fr, 0.016)
    np.testing.assert_array_equal(c, c1[q])
    np.testing.assert_allclose(f1[q], vo.mlp(w.w1, w.b1, w.w2, w.b2, vo.to_features(emb)), rtol=0, atol=1e-4)
    print("order ok", case, os.environ.get("VKM_SORT", "auto"), len(X))


if __name__ == "__main__":
    main(sys.argv[1])
