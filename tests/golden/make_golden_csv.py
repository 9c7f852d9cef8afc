"""Freeze the reference's CSV event parser outcomes (events.py:177-236) as a
fixture: for a set of valid and malformed files, either the parsed columns or
the exception type and message (with the path replaced by "<path>").  Run in
the build container, where /root/reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_csv.py
"""
import json
import os
import tempfile

import numpy as np
from evflow.events import CameraGeometry, load_events

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = np.random.default_rng(3)
    n = 400
    t = np.sort(rng.uniform(0, 0.05, n))
    x = rng.integers(0, 16, n)
    y = rng.integers(0, 12, n)
    p = rng.choice([0, 1, -1], n)
    good = [f"{a!r},{b},{c}" for a, b, c in zip(t.tolist(), x.tolist(), y.tolist())]
    goodp = [f"{a!r},{b},{c},{d}" for a, b, c, d in zip(t.tolist(), x.tolist(), y.tolist(), p.tolist())]
    yield "plain", "\n".join(good) + "\n"
    yield "polarity", "\n".join(goodp) + "\n"
    yield "header_blank", "t,x,y,p\n\n" + "\n".join(goodp[:50]) + "\n\n  \n" + "\n".join(goodp[50:]) + "\n"
    yield "header_not_first", "\n" + "t,x,y\n" + "\n".join(good[:5]) + "\n"
    yield "mixed_3_4", "\n".join(good[:10] + goodp[10:20] + good[20:30]) + "\n"
    yield "spaces_underscores", " 0.001 , 3 ,+4\n1_0e-3,5,6\n0.002,  7,8 ,1\n"
    lines = list(good[:60])
    variants = {
        "fields2": "0.01,3", "fields5": "0.01,3,4,1,9", "bad_t": "abc,3,4", "bad_x": "0.01,3.0,4", "bad_y": "0.01,3,y",
        "nan_t": "nan,3,4", "inf_t": "inf,3,4", "neg_t": "-0.5,3,4", "x_hi": "0.01,16,4", "x_neg": "0.01,-1,4",
        "y_hi": "0.01,3,12", "bad_p": "0.01,3,4,q", "p_two": "0.01,3,4,2", "p_float": "0.01,3,4,1.0",
        "empty_field": "0.01,,4",
    }
    for name, bad in variants.items():
        yield name, "\n".join(lines[:30] + [bad] + lines[30:]) + "\n"
    # two errors: the earlier line wins whatever its kind
    yield "two_errors_range_first", "\n".join(lines[:10] + ["0.01,99,4"] + lines[10:20] + ["zz,1,1"]) + "\n"
    yield "two_errors_parse_first", "\n".join(lines[:10] + ["zz,1,1"] + lines[10:20] + ["0.01,99,4"]) + "\n"
    yield "two_errors_count_last", "\n".join(lines[:10] + ["0.01,3,4,7"] + lines[10:20] + ["1,2"]) + "\n"
    yield "same_line_x_and_p", "\n".join(lines[:5] + ["0.01,99,4,5"]) + "\n"
    yield "header_only", "t,x,y\n"
    yield "empty", ""


def main():
    g = CameraGeometry(16, 12)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name, text in cases():
            path = os.path.join(td, name + ".csv")
            with open(path, "w", encoding="utf-8") as fh:
                fh.write(text)
            try:
                st = load_events(path, "csv", g)
                out[name] = {"text": text, "ok": True, "t": [repr(v) for v in st.t.tolist()], "x": st.x.tolist(),
                             "y": st.y.tolist(), "p": None if st.polarity is None else st.polarity.tolist()}
            except Exception as exc:   # noqa: BLE001 - the fixture records whatever the reference raises
                out[name] = {"text": text, "ok": False, "type": type(exc).__name__,
                             "message": str(exc).replace(path, "<path>")}
    with open(os.path.join(HERE, "csv_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    main()
