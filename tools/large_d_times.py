"""Per-step and fused times of the LSTM kernels for hidden sizes beyond the
d=8 fast path, at a 64 MiB fp32 state (B = 2^22 / d): CUDA events around
back-to-back launches.  Prints one JSON line per d."""
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


def main():
    ds = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32,64").split(",")]
    for d in ds:
        B = (1 << 22) // d
        S = 2 * d * B * 4
        cell = lstm.random_cell(d, 64, 0)
        dc = lstm.device_cell(cell, B, "f32")
        x = lstm.random_states(d, 1, B, "f32")
        bufs = [torch.empty_like(x) for _ in range(4)]
        L = 16

        def fwd_chain():
            cur = x
            for k in range(L):
                cur = dc.forward(k, cur)

        def bwd_chain():
            a = x
            for k in range(L):
                a = dc.backward(k, x, a)

        t_f = timed(fwd_chain) / L
        t_b = timed(bwd_chain) / L
        row = {"d": d, "batch": B, "state_mib": S / 2**20, "fwd_us": t_f * 1e6, "bwd_us": t_b * 1e6,
               "fwd_gbs": 2 * S / t_f / 1e9, "bwd_gbs": 3 * S / t_b / 1e9,
               "fwd_tflops": B * 8 * d * d / t_f / 1e12, "bwd_tflops": B * 16 * d * d / t_b / 1e12}
        try:
            t_adv = timed(lambda: dc.advance(0, 64, x)) / 64
            states = dc.forward_many(0, 64, x)
            seed = dc.seed(states[-1])
            t_tape = timed(lambda: dc.forward_many(0, 64, x)) / 64
            t_rev = timed(lambda: dc.backward_many(0, [x] + states[:-1], seed)) / 64
            row.update({"adv_us": t_adv * 1e6, "tape_us": t_tape * 1e6, "rev_us": t_rev * 1e6})
        except Exception as exc:  # fused launches exist for the fast path only
            row["fused"] = f"n/a: {type(exc).__name__}"
        print(json.dumps(row), flush=True)
        del dc, x, bufs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
