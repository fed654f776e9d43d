"""Config-1 calibration on the file tier (B=1 fp64, d=32): t_a, t_b, t_t and
the resulting interval, per-step and fused, plus the in-pass store / fetch
durations from the measured timeline."""
import json
import os
import statistics
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

ops = lstm.operator_pair(lstm.random_cell(32, 1000, 0))
s0 = lstm.random_state(32, 1)
with pkg.FileBackend(tempfile.mkdtemp(prefix="ackpt_cal_")) as fb:
    for fuse in (False, True):
        for _ in range(2):
            t_a, t_b, t_t = pkg.calibrate(ops, fb, 5, s0, fuse=fuse)
            I = pkg.interval_length(t_t, t_a)
            _, st = pkg.execute(pkg.Multistage(10, I), ops, s0, fb, fuse=fuse, timeline=True)
            xs = {}
            for e in st.timeline:
                xs.setdefault(e.kind, []).append(e.end - e.start)
            med = {k: round(statistics.median(v) * 1e6, 1) for k, v in xs.items() if k in ("store", "fetch", "stall")}
            print(json.dumps({"fuse": fuse, "t_a_us": t_a * 1e6, "t_b_us": t_b * 1e6, "t_t_us": t_t * 1e6, "I": I,
                              "wall_ms": st.wall_seconds * 1e3, "stall_ms": st.stall_seconds * 1e3,
                              "median_us": med}))
