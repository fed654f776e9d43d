"""Chained K1/K2 launches at the BASELINE config-2 shape (d=8, B=2^20 fp32,
64 MiB state) for ncu captures and CUDA-event timing of each kernel alone.

  python tools/profile_kernels.py [--steps 40] [--d 8] [--batch 1048576] [--fused 0]
Prints one JSON line with per-kernel mean durations and GB/s (algorithmic
bytes: forward 2S, backward 3S).
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--d", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--fused", type=int, default=0)
    ap.add_argument("--fused-only", type=int, default=0, help="only the fused adv/tape/rev launches (for ncu)")
    args = ap.parse_args()
    cell = lstm.random_cell(args.d, max(args.steps, 2), 0)
    dc = lstm.device_cell(cell, args.batch, "f32")
    S = dc.state_bytes
    x = lstm.random_states(args.d, 1, args.batch, "f32")
    # pool of distinct buffers like the executor's (inputs larger than L2)
    bufs = [torch.empty_like(x) for _ in range(8)]
    adj = [torch.empty_like(x) for _ in range(2)]
    bufs[0].copy_(x)
    out = {}
    if args.fused_only:
        L = min(64, args.steps)
        states = dc.forward_many(0, L, x)
        a0 = dc.seed(states[-1])
        for _ in range(3):
            dc.advance(0, L, x)
            dc.forward_many(0, L, x)
            dc.backward_many(0, [x] + states[:-1], a0)
        torch.cuda.synchronize()
        print(json.dumps({"fused_only": True, "steps": L}))
        return
    for name in ("fwd", "bwd"):
        for _ in range(3):  # warm-up
            dc.forward(0, bufs[0])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(args.steps):
            if name == "fwd":
                bufs[(k + 1) % 8] = dc.forward(k, bufs[k % 8])
            else:
                adj[(k + 1) % 2] = dc.backward(k, bufs[k % 8], adj[k % 2])
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / args.steps
        nbytes = (2 if name == "fwd" else 3) * S
        out[name] = {"us": t * 1e6, "gbs": nbytes / t / 1e9}
    if args.fused:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = dc.advance(0, args.steps, bufs[0])
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / args.steps
        out["fused_advance_per_step"] = {"us": t * 1e6}
    out["state_bytes"] = S
    print(json.dumps(out))


if __name__ == "__main__":
    main()
