"""Config 1 (n=1000, d=32, s=10, B=1 float64, file tier) Multistage pass with
the measured timeline: where the time goes (compute kinds, stalls, store /
fetch durations on the copy lanes).  `python tools/c1_timeline.py [fuse]`."""
import json
import os
import statistics
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

fuse = len(sys.argv) > 1 and sys.argv[1] == "fuse"
scratch = tempfile.mkdtemp(prefix="ackpt_c1tl_")
path = os.path.join(scratch, "tl.json")
rep = lstm.bench(pkg.Multistage(10), n=1000, d=32, s=10, backend_config={"kind": "file", "dir": scratch}, runs=3,
                 fuse=fuse, timeline_path=path)
obj = json.load(open(path))
events = obj["events"] if isinstance(obj, dict) else obj
by = {}
for e in events:
    k = (e["lane"], e["kind"])
    by.setdefault(k, []).append(e["end"] - e["start"])
out = {"fuse": fuse, "wall_ms": rep.wall_seconds * 1e3, "stall_ms": rep.stall_seconds * 1e3,
       "forward_evals": rep.forward_evals}
for (lane, kind), v in sorted(by.items()):
    out[f"{lane}/{kind}"] = {"count": len(v), "sum_ms": sum(v) * 1e3, "median_us": statistics.median(v) * 1e6,
                             "max_us": max(v) * 1e6}
print(json.dumps(out, indent=1))
