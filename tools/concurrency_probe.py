"""Can a TapeForward launch overlap a Reverse run usefully?  Times (C2
shape, 64-step launches) tape alone, reverse alone, both back to back on one
stream, and both concurrently on two streams."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    fam = sys.argv[1] if len(sys.argv) > 1 else "tcgen05"
    lstm.set_kernel_family(fam)
    cell = lstm.random_cell(8, 200, 0)
    dc = lstm.device_cell(cell, 1 << 20, "f32")
    x = lstm.random_states(8, 1, 1 << 20, "f32")
    states = dc.forward_many(0, 64, x)
    seed = dc.seed(states[-1])
    tape_in = states[-1].clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def tape():
        dc.forward_many(64, 64, tape_in)

    def rev():
        dc.backward_many(0, [x] + states[:-1], seed)

    def timeit(fn, reps=5):
        ts = []
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return sorted(ts[1:])[len(ts[1:]) // 2]

    def both_seq():
        tape()
        rev()

    def both_conc():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            tape()
        with torch.cuda.stream(s2):
            rev()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    out = {"family": fam, "tape_ms": timeit(tape), "rev_ms": timeit(rev), "seq_ms": timeit(both_seq),
           "concurrent_ms": timeit(both_conc)}
    out["speedup_vs_seq"] = out["seq_ms"] / out["concurrent_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
