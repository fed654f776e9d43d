"""Where does the file tier's in-pass stall come from?  Runs the C2 state
(64 MiB) over the file tier with the measured timeline on and reports the
store / fetch durations inside the pass against the calibrated t_t."""
import json
import os
import shutil
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

d, B, n = 8, 1 << 20, 8000
scratch = sys.argv[1] if len(sys.argv) > 1 else "/tmp/ackpt_ftl"
shutil.rmtree(scratch, ignore_errors=True)
ops = lstm.operator_pair(lstm.random_cell(d, n, 0), B, "f32")
s0 = lstm.random_states(d, 1, B, "f32")
with pkg.FileBackend(scratch) as be:
    t_a, t_b, t_t = pkg.calibrate(ops, be, 5, s0, fuse=True)
    interval = pkg.interval_length(t_t, t_a)
    strat = pkg.Multistage(799, interval)
    pkg.execute(strat, ops, s0, be, fuse=True)
    _, st = pkg.execute(strat, ops, s0, be, fuse=True, timeline=True)
ev = st.timeline
stores = [e.end - e.start for e in ev if e.kind == "store"]
fetches = [e.end - e.start for e in ev if e.kind == "fetch"]
stalls = [(e.from_step, e.end - e.start) for e in ev if e.kind == "stall" and e.end - e.start > 1e-4]
print(json.dumps({"t_t_ms": t_t * 1e3, "t_a_us": t_a * 1e6, "interval": interval, "interval_ms": interval * t_a * 1e3,
                  "store_ms": [round(x * 1e3, 2) for x in stores], "fetch_ms": [round(x * 1e3, 2) for x in fetches],
                  "store_median_ms": statistics.median(stores) * 1e3, "stalls_ms": [(s, round(x * 1e3, 2)) for s, x in stalls],
                  "stall_total_ms": st.stall_seconds * 1e3, "wall_ms": st.wall_seconds * 1e3}))
shutil.rmtree(scratch, ignore_errors=True)
