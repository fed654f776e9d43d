"""One short fused Multistage pass over the pinned tier (d=8, B=2^18,
n=400) -- a target for NVTX-filtered ncu runs, e.g.

  ncu --nvtx --nvtx-include "ackpt@pass/backward/" \
      --metrics gpu__time_duration.sum python tools/nvtx_probe.py

profiles only the kernels the backward phase launches (ranges: csrc/nvtx.h).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

ops = lstm.operator_pair(lstm.long_memory_cell(8, 400, 0), 1 << 18, "f32")
s0 = lstm.random_states(8, 1, 1 << 18, "f32")
with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
    adj, st = pkg.execute(pkg.Multistage(60, 50), ops, s0, b, fuse=True)
torch.cuda.synchronize()
print("nvtx_probe ok", st.forward_evals, float(adj.double().norm()))
