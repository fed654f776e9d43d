"""Per-step times of the fused launches (advance / tape / reverse, 64 steps)
at the C2 shape for the active kernel family (ACKPT_TC=1 tensor cores,
ACKPT_TC=0 packed FFMA2; unset = tcgen05).  Optional batch sizes (argv) show
the wave quantization: e.g. 909312 = 3552 CTAs of 256 sequences = exactly 4
rounds of the 888 resident reverse CTAs (6/SM) and 3 rounds of the 1184
resident tape / advance CTAs (8/SM); per-step times are scaled to 2^20
sequences (us per 64 MiB)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

batches = [int(x) for x in sys.argv[1:]] or [1 << 20]
cell = lstm.random_cell(8, 128, 0)
for B in batches:
    dc = lstm.device_cell(cell, B, "f32")
    x = lstm.random_states(8, 1, B, "f32")
    fk = bench.fused_kernel_times(dc, x, steps=64)
    scale = (1 << 20) / B
    print(json.dumps({"ACKPT_TC": os.environ.get("ACKPT_TC", "1"), "batch": B, "ctas": -(-B // 256),
                      **{k: (v * 1e6 * scale if not k.endswith("bytes") else v) for k, v in fk.items()}}), flush=True)
    del dc, x
