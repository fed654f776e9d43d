"""Per-step operator cost at the C2 shape: K1 / K2 (FFMA2, HBM-bound) vs the
tcgen05 fused kernels launched with count = 1."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        best = t if best is None else min(best, t)
    return best


cell = lstm.random_cell(8, 64, 0)
dc = lstm.device_cell(cell, 1 << 20, "f32")
x = lstm.random_states(8, 1, 1 << 20, "f32")
a = lstm.random_states(8, 2, 1 << 20, "f32")
bufs = [torch.empty_like(x) for _ in range(8)]
L = 32


def k1():
    cur = x
    for k in range(L):
        cur = dc.forward(k, cur)


def k2():
    adj = a
    for k in range(L):
        adj = dc.backward(k, bufs[k % 8], adj)


def tc_fwd():
    cur = x
    for k in range(L):
        cur = dc.advance(k, k + 1, cur)


def tc_bwd():
    adj = a
    for k in range(L):
        adj = dc.backward_many(k, [bufs[k % 8]], adj)


print(json.dumps({name: timed(fn) / L * 1e6 for name, fn in
                  (("K1_us", k1), ("K2_us", k2), ("tc_fwd_count1_us", tc_fwd), ("tc_rev_count1_us", tc_bwd))}))
