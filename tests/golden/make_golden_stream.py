"""Freeze the reference's stream slicing and EVN1 encoding as fixtures
(run in the build container, where /root/reference is importable):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_stream.py
"""
import os
import numpy as np
from evflow.events import CameraGeometry, EventStream, slice_stream, write_events_binary

HERE = os.path.dirname(os.path.abspath(__file__))


def case(name, t, x, y, p, delta_t, stride, t0):
    g = CameraGeometry(64, 48)
    st = EventStream(t=t, x=x, y=y, geometry=g, polarity=p)
    sl = slice_stream(st, delta_t, stride, t0)
    return {f"{name}_t": t, f"{name}_x": x, f"{name}_y": y,
            f"{name}_params": np.array([delta_t, stride, t0]),
            f"{name}_starts": np.array([s.t_start for s in sl]),
            f"{name}_lens": np.array([len(s) for s in sl]),
            f"{name}_first": np.array([s.t[0] if len(s) else -1.0 for s in sl]),
            f"{name}_xsum": np.array([int(s.x.sum()) for s in sl])}


rng = np.random.default_rng(7)
out = {}
n = 3000
t = np.sort(rng.uniform(0.0, 0.25, n)); x = rng.integers(0, 64, n); y = rng.integers(0, 48, n)
out.update(case("overlap", t, x, y, None, 0.016, 0.01, 0.0))
out.update(case("disjoint", t, x, y, None, 0.016, 0.032, 0.003))
tg = np.concatenate([np.sort(rng.uniform(0.0, 0.05, 500)), np.sort(rng.uniform(0.2, 0.3, 500))])   # interior gap
out.update(case("gap", tg, rng.integers(0, 64, 1000), rng.integers(0, 48, 1000), None, 0.016, 0.02, 0.0))
te = np.array([0.0, 0.032, 0.032, 0.064, 0.0640000001, 0.1])   # events exactly on window edges
out.update(case("edges", te, np.arange(6) % 64, np.arange(6) % 48, None, 0.016, 0.032, 0.0))
tu = rng.uniform(0.0, 0.1, 800)   # unsorted stream
out.update(case("unsorted", tu, rng.integers(0, 64, 800), rng.integers(0, 48, 800), None, 0.016, 0.016, 0.0))
np.savez_compressed(os.path.join(HERE, "stream_slices.npz"), **out)

# EVN1 round trip: a small file written by the reference
g = CameraGeometry(346, 260)
m = 40
st = EventStream(t=np.sort(rng.uniform(0, 0.03, m)), x=rng.integers(0, 346, m), y=rng.integers(0, 260, m),
                 geometry=g, polarity=rng.choice([0, 1], m).astype(np.int8))
write_events_binary(st, os.path.join(HERE, "events_small.evn1"))
np.savez_compressed(os.path.join(HERE, "events_small.npz"), t=st.t, x=st.x, y=st.y, p=st.polarity)
print("wrote stream_slices.npz, events_small.evn1/.npz")
