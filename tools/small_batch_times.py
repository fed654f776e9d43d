"""Per-step GPU time of the LSTM step kernels at small batches (the
reference's own workload is B=1 float64, d=32): a fused Advance over n
steps, TapeForward / Reverse runs of ACKPT_MAX_FUSED steps, and single-step
launches -- each captured in a CUDA graph and replayed, so host overhead is
excluded.  `python tools/small_batch_times.py d dtype batch [batch ...]`;
one JSON line per batch (microseconds per step).  ACKPT_SB_FIRST / ACKPT_TCD
select the kernel family."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def graph_time(fn, steps, reps=5):
    try:
        return _graph_time(fn, steps, reps)
    except Exception:  # e.g. no fused reverse for this family
        return None


def _graph_time(fn, steps, reps):
    torch.cuda.synchronize()
    fn()  # warm-up (first-use attribute setting, allocations)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3)
    return best / steps


def one(d, dtype, batch, n=1000):
    cell = lstm.random_cell(d, n, 0)
    dc = lstm.device_cell(cell, batch, dtype)
    s0 = dc._tensor(lstm.random_state(d, 1) if batch == 1 and dtype == "f64" else lstm.random_states(d, 1, batch, dtype))
    states = [dc.forward(k, s0) for k in range(64)]
    return {
        "d": d, "dtype": dtype, "batch": batch,
        "advance_us_per_step": graph_time(lambda: dc.advance(0, n, s0), n),
        "tape_us_per_step": graph_time(lambda: dc.forward_many(0, 64, s0), 64),
        "reverse_us_per_step": graph_time(lambda: dc.backward_many(0, states, s0), 64),
        "forward_launch_us": graph_time(lambda: [dc.forward(k, s0) for k in range(100)], 100),
        "backward_launch_us": graph_time(lambda: [dc.backward(k, s0, s0) for k in range(100)], 100),
    }


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    dtype = sys.argv[2] if len(sys.argv) > 2 else "f64"
    for batch in [int(x) for x in sys.argv[3:]] or [1]:
        print(json.dumps(one(d, dtype, batch)), flush=True)


if __name__ == "__main__":
    main()
