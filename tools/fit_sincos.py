"""Fit the minimax polynomials of the f32 sin/cos used by the kernels
(reduction by pi: r in [-pi/2, pi/2]; sin(r) = r + r^3 P(r^2), cos(r) = 1 + r^2 Q(r^2)),
then measure the f32 evaluation error (FMA emulated in f64) against the
correctly rounded f32 result over the phase range used by the encoder."""
import numpy as np

def fit(fun, basis, npts=4000, iters=60):
    # iteratively reweighted least squares toward minimax absolute error on [0, pi/2]
    x = np.cos(np.linspace(0, np.pi, npts)) * 0.5 * np.pi / 2 + np.pi / 4   # Chebyshev nodes in [0, pi/2]
    A = np.stack([b(x) for b in basis], 1)
    t = fun(x)
    w = np.ones_like(x)
    for _ in range(iters):
        c, *_ = np.linalg.lstsq(A * w[:, None], t * w, rcond=None)
        e = np.abs(A @ c - t)
        w = w * (e / e.max() + 1e-3) ** 0.5
        w /= w.max()
    return c, np.abs(A @ c - t).max()

def f32(v):
    return np.float32(v)

def fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)

if __name__ == "__main__":
    # sin(r) - r = r^3 * P(u), u = r^2: fit P on relative-to-r^3 residual
    NS, NC = 4, 5   # degree 9 sin / 10 cos: the f32 error of 5, 6 (evaluation rounding dominates)
    cs, es = fit(lambda x: np.sin(x) - x, [lambda x, k=k: x ** (2 * k + 3) for k in range(NS)])
    cc, ec = fit(lambda x: np.cos(x) - 1.0, [lambda x, k=k: x ** (2 * k + 2) for k in range(NC)])
    cs32 = [np.float32(v) for v in cs]
    cc32 = [np.float32(v) for v in cc]
    print("sin coeffs", [f"{v:.9e}" for v in cs32], "fit err", es)
    print("cos coeffs", [f"{v:.9e}" for v in cc32], "fit err", ec)
    PI1 = np.float32(3.14159203); PI2 = np.float32(6.27832946e-07); PI3 = np.float32(1.07806051e-14)
    rng = np.random.default_rng(0)
    x = (rng.uniform(-60, 60, 4_000_000)).astype(np.float32)
    x = np.concatenate([x, (rng.uniform(-2, 2, 1_000_000)).astype(np.float32)])
    magic = np.float32(12582912.0)
    qb = (x * np.float32(1 / np.pi)).astype(np.float32) + magic
    qb = qb.astype(np.float32)
    q = (qb - magic).astype(np.float32)
    r = fma32(q, -PI1 * np.ones_like(q), x)
    r = fma32(q, -PI2 * np.ones_like(q), r)
    # 2-part reduction (the kernels drop q·PI3 < 1e-12 for |x| < 1e3)
    u = (r * r).astype(np.float32)
    ps = np.full_like(u, cs32[-1])
    for k in range(NS - 2, -1, -1):
        ps = fma32(ps, u, np.full_like(u, cs32[k]))
    ps = (ps * u).astype(np.float32)
    sr = fma32(ps, r, r)
    pc = np.full_like(u, cc32[-1])
    for k in range(NC - 2, -1, -1):
        pc = fma32(pc, u, np.full_like(u, cc32[k]))
    cr = fma32(pc, u, np.ones_like(u))
    k = qb.view(np.int32) & 1
    sgn = np.where(k == 1, -1.0, 1.0).astype(np.float32)
    s = sr * sgn; c = cr * sgn
    xs = x.astype(np.float64)
    st, ct = np.sin(xs), np.cos(xs)
    ulp = lambda v: np.spacing(np.abs(v).astype(np.float32)).astype(np.float64)
    es_abs = np.abs(s - st).max(); ec_abs = np.abs(c - ct).max()
    print("max abs err sin %.3e cos %.3e" % (es_abs, ec_abs))
    print("max ulp err (|v|>=0.25) sin %.2f cos %.2f" % ((np.abs(s - st) / ulp(st))[np.abs(st) > .25].max(),
                                                       (np.abs(c - ct) / ulp(ct))[np.abs(ct) > .25].max()))
    ns, nc = np.sin(x), np.cos(x)
    print("bit-identical to numpy f32: sin %.4f cos %.4f" % ((s == ns).mean(), (c == nc).mean()))
