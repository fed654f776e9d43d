"""Why does the in-line CPU baseline read lower than the standalone
reference arm?  Runs bench.py's inline_cpu_baseline (a clean subprocess of
`bench.py --impl reference`) in successive process states."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

args = bench.parse_args(["--steps", "5"])
out = {}
out["no_cuda"] = bench.inline_cpu_baseline(args, 75)["value"]
import torch  # noqa: E402

torch.cuda.init()
x = torch.empty(1 << 20, device="cuda")
out["cuda_context"] = bench.inline_cpu_baseline(args, 75)["value"]
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

ops = lstm.operator_pair(lstm.random_cell(8, 10000, 0), 1 << 20, "f32")
s0 = lstm.random_states(8, 1, 1 << 20, "f32")
b = pkg.PinnedHostBackend(slot_bytes=ops.state_size)
pkg.execute(pkg.Multistage(999, 72), ops, s0, b, fuse=True)
torch.cuda.synchronize()
out["after_pass_pinned_9GiB"] = bench.inline_cpu_baseline(args, 75)["value"]
b.close()
pkg.release(ops)
out["after_close"] = bench.inline_cpu_baseline(args, 75)["value"]
time.sleep(5)
out["after_sleep"] = bench.inline_cpu_baseline(args, 75)["value"]
print(json.dumps(out))
