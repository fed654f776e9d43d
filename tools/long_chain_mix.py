"""Which kernel carries the long-chain adjoint error?  Forward trajectories
from the tcgen05 tape kernel (A) or the FFMA2 per-step K1 (B), reversed by
rev_tc (X) or the per-step K2 (Y), on the long-memory cell at n = 10^4,
each against the float64 oracle on sampled sequences."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200.lstm as lstm  # noqa: E402
from oracle import lstm_oracle as L  # noqa: E402
from oracle import runtime_oracle as RO  # noqa: E402

d, n, batch = 8, int(sys.argv[1]), 8192
fb = float(sys.argv[2])
cell = lstm.long_memory_cell(d, n, 0, fb)
dc = lstm.device_cell(cell, batch, "f32")
s0 = lstm.random_states(d, 1, batch, "f32")
rows = np.arange(0, batch, batch // 64)
ref, _ = RO.execute("full", L.long_memory_cell(d, n, 0, fb), s0[:, :, rows].double().cpu().numpy())


def traj(kind):
    lstm.set_kernel_family("tcgen05")
    states = [s0]
    if kind == "A":
        while len(states) < n + 1:
            cnt = min(64, n + 1 - len(states))
            states += dc.forward_many(len(states) - 1, cnt, states[-1])
    else:
        for k in range(n):
            states.append(dc.forward(k, states[-1]))
    return states


def rev(kind, states):
    adj = dc.seed(states[n])
    if kind == "X":
        lstm.set_kernel_family("tcgen05")
        hi = n
        while hi > 0:
            lo = max(0, hi - 64)
            adj = dc.backward_many(lo, states[lo:hi], adj)
            hi = lo
    else:
        for k in range(n - 1, -1, -1):
            adj = dc.backward(k, states[k], adj)
    return adj


for t in ("A", "B"):
    st = traj(t)
    for r in ("X", "Y"):
        a = rev(r, st)[:, :, rows].double().cpu().numpy()
        print(json.dumps({"fb": fb, "traj": t, "rev": r, "rel_l2": L.rel_l2(a, ref)}), flush=True)
    del st
    torch.cuda.empty_cache()
