"""Max-abs flow error of every MLP mode against the reference's golden flows
(tests/golden/*.npz) on the GPU path; one line per case."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2504_19417_b200 as pkg  # noqa: E402
from conftest import GOLDEN_CASES, load_golden  # noqa: E402

for case in GOLDEN_CASES:
    g = load_golden(case)
    b = pkg.Bases(g["freqT"], g["freqX"], g["freqY"], float(g["sigma2"]))
    w = pkg.MlpWeights(g["w1"], g["b1"], g["w2"], g["b2"], b)
    errs = {}
    for mode in ("fp32", "f16x3", "bf16"):
        reg = pkg.NormalFlowRegressor(delta_t=float(g["delta_t"]), delta_x=int(g["dx"]), delta_y=int(g["dy"]),
                                      embed_dim=int(g["D"]), width=int(g["width"]), height=int(g["height"]),
                                      weights=w, mlp_mode=mode)
        f = reg.predict(g["X"])
        ok = np.isfinite(g["flows"]).all(axis=1)
        assert np.array_equal(ok, np.isfinite(f).all(axis=1)), case
        errs[mode] = float(np.max(np.abs(f[ok] - g["flows"][ok]))) if ok.any() else 0.0
    print(f"{case:20s} n={len(g['X']):6d} " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()))
