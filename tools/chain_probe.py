"""Launch-chain parity probe (lstm_f32_tc.cu chain_for, ACKPT_TC_CHAIN).

Runs back-to-back fused d=8 tcgen05 launches of one cell on one stream --
Advance, two TapeForward chunks, two Reverse runs, on a ragged batch (the
last tile partial) -- and a fused Multistage pass through the executor, then
prints a digest of every output.  With ACKPT_TC_CHAIN=force every launch
after the first is chained to its predecessor (programmatic dependent launch
+ per-tile completion flags); with =0 none is; by default only the
executor's fused launches chain.  The digests must agree bit for bit
(tests/test_gpu_chain.py).
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    d, n, batch = 8, 300, (1 << 17) + 37
    lstm.set_kernel_family("tcgen05")
    ops = lstm.operator_pair(lstm.long_memory_cell(d, n, 0), batch, "f32")
    dc = ops.native
    s0 = lstm.random_states(d, 1, batch, "f32")
    digest = hashlib.sha256()

    def note(t):
        assert torch.isfinite(t).all()
        digest.update(t.detach().cpu().numpy().tobytes())

    for rep in range(3):  # the flag epochs advance across repetitions
        x = dc.advance(0, 40, s0)
        t1 = dc.forward_many(40, 64, x)
        t2 = dc.forward_many(104, 64, t1[-1])
        a = dc.seed(t2[-1])
        a = dc.backward_many(104, [t1[-1]] + t2[:-1], a)
        a = dc.backward_many(40, [x] + t1[:-1], a)
        torch.cuda.synchronize()
        for t in (x, t1[-1], t2[-1], a):
            note(t)
    with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
        adj, _ = pkg.execute(pkg.Multistage(20, 25), ops, s0, b, fuse=True)
        note(adj)
    print("chain_probe ok digest", digest.hexdigest())


if __name__ == "__main__":
    main()
