"""Per-step times of the fused launches (advance / tape / reverse, 64 steps)
at the C2 shape for the active kernel family (ACKPT_TC=1 tensor cores,
ACKPT_TC=0 packed FFMA2; unset = tcgen05)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

cell = lstm.random_cell(8, 128, 0)
dc = lstm.device_cell(cell, 1 << 20, "f32")
x = lstm.random_states(8, 1, 1 << 20, "f32")
fk = bench.fused_kernel_times(dc, x, steps=64)
print(json.dumps({"ACKPT_TC": os.environ.get("ACKPT_TC", "1"), **{k: (v * 1e6 if not k.endswith("bytes") else v) for k, v in fk.items()}}))
