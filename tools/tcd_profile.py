"""Per-step launches of the d=32 tensor-core kernels at a 32 MiB state (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200.lstm as lstm  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 32
B = (1 << 22) // d
dc = lstm.device_cell(lstm.random_cell(d, 16, 0), B, "f32")
x = lstm.random_states(d, 1, B, "f32")
a = lstm.random_states(d, 2, B, "f32")
for k in range(4):
    y = dc.forward(k, x)
    g = dc.backward(k, x, a)
torch.cuda.synchronize()
