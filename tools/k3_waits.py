"""Cycles K3's warps spend in each barrier wait (build with -DVKM_K3_WAITPROF;
VKM_LIB points at it).  Prints per-launch averages summed over warps."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_19417_b200 as pkg  # noqa: E402
from paper_2504_19417_b200 import _lib  # noqa: E402
import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
W, H, n, d, _, _ = bench.WORKLOADS[wl]
X = bench._synth(n, W, H, 0)
b = pkg.generate_bases(64)
w = pkg.init_weights(64, 128, b, seed=0, dtype=np.float32)
eng = pkg.FlowEngine(W, H, d, d, 0.016, b, w)
ev = torch.from_numpy(X).cuda()
lib = _lib.load()
buf = (C.c_ulonglong * 8)()
for _ in range(3):
    eng.predict_device(ev, float(X[0, 0]))
torch.cuda.synchronize()
lib.vkm_debug_k3_waits(buf)
reps = 10
for _ in range(reps):
    eng.predict_device(ev, float(X[0, 0]))
torch.cuda.synchronize()
lib.vkm_debug_k3_waits(buf)
names = ["producer gfull (TMA rows)", "producer empty (A stage)", "loader gempty", "epilogue tfull",
         "mma tempty", "mma full"]
warps = {0: 16, 1: 16, 2: 1, 3: 4, 4: 1, 5: 1}
for i, nm in enumerate(names):
    per_warp_us = buf[i] / reps / (148 * warps[i]) / 1965.0
    print(f"{wl} {nm:28s} {per_warp_us:8.1f} us per warp per launch")
