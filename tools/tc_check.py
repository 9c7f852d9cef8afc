"""Dev check: run each MLP mode on one golden case and print max-abs vs the reference."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import load_golden
import paper_2504_19417_b200 as pkg

case = sys.argv[1] if len(sys.argv) > 1 else "cfg1_20k"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fp32", "f16x3", "bf16"]
g = load_golden(case)
b = pkg.Bases(g["freqT"], g["freqX"], g["freqY"], 25.0)
w = pkg.MlpWeights(g["w1"], g["b1"], g["w2"], g["b2"], b)
for mode in modes:
    reg = pkg.NormalFlowRegressor(delta_t=float(g["delta_t"]), delta_x=int(g["dx"]), delta_y=int(g["dy"]),
                                  embed_dim=int(g["D"]), width=int(g["width"]), height=int(g["height"]),
                                  weights=w, mlp_mode=mode)
    t = time.time()
    f = reg.predict(g["X"])
    print(f"{case} {mode}: max|d|={np.nanmax(np.abs(f - g['flows'])):.3e} nan={np.isnan(f).sum()} "
          f"t={time.time()-t:.3f}s", flush=True)
