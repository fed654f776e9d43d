"""Would running segment j-1's TapeForward concurrently with segment j's
Reverse (two streams) beat running them back to back?  C2 shape (d=8,
B=2^20 fp32), 64-step tape and reverse launches on separate buffers,
CUDA-event timed: sequential vs concurrent, best of 5."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

d, B, L = 8, 1 << 20, 64
dc = lstm.device_cell(lstm.random_cell(d, 256, 0), B, "f32")
x = lstm.random_states(d, 1, B, "f32")
states = dc.forward_many(0, L, x)
seed = dc.seed(states[-1])
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def tape():
    return dc.forward_many(L, L, x)


def rev():
    return dc.backward_many(0, [x] + states[:-1], seed)


def timed(fn, reps=5):
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def concurrent():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        tape()
    with torch.cuda.stream(s2):
        rev()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


tape(); rev(); concurrent()
t_tape, t_rev = timed(tape), timed(rev)
t_seq = timed(lambda: (tape(), rev()))
t_con = timed(concurrent)
print(json.dumps({"tape_ms": t_tape, "rev_ms": t_rev, "sequential_ms": t_seq, "concurrent_ms": t_con,
                  "gain": t_seq / t_con}))

# a backward-like chain: K intervals of (tape, reverse), sequential on one
# stream vs the next interval's tape on a second stream under this
# interval's reverse (the tape depends only on the prefetched boundary)
K = 4


def chain_seq():
    for _ in range(K):
        tape()
        rev()


def chain_pipe():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        tape()
    for k in range(K):
        done = torch.cuda.Event()
        done.record(s1)
        s2.wait_event(done)  # reverse k needs tape k
        with torch.cuda.stream(s2):
            rev()
        if k + 1 < K:
            with torch.cuda.stream(s1):
                tape()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


chain_seq(); chain_pipe()
t_cs, t_cp = timed(chain_seq), timed(chain_pipe)
print(json.dumps({"intervals": K, "chain_sequential_ms": t_cs, "chain_pipelined_ms": t_cp, "gain": t_cs / t_cp}))
