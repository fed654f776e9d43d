"""Per-step time of the fused d=8 launches against the steps per launch
(count = 8 .. 64) at the C2 shape: separates a fixed per-launch cost from a
per-step one (CUDA events around back-to-back launches)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
dc = lstm.device_cell(lstm.random_cell(8, 256, 0), B, "f32")
x = lstm.random_states(8, 1, B, "f32")
states = dc.forward_many(0, 64, x)
seed = dc.seed(states[-1])


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3)
    return best


for count in (8, 16, 32, 64):
    reps = 64 // count
    row = {"batch": B, "count": count}
    row["adv_us_per_step"] = timed(lambda: [dc.advance(0, count, x) for _ in range(reps)]) / 64
    row["tape_us_per_step"] = timed(lambda: [dc.forward_many(0, count, x) for _ in range(reps)]) / 64
    row["rev_us_per_step"] = timed(lambda: [dc.backward_many(0, [x] + states[:count - 1], seed)
                                            for _ in range(reps)]) / 64
    print(json.dumps(row), flush=True)
