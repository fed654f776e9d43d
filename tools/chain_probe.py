"""Launch-chain parity probe (csrc/chain.cuh, ACKPT_TC_CHAIN).

Runs back-to-back tensor-core launches of one cell on one stream -- fused
Advance, two TapeForward chunks, two Reverse runs, per-step forward and
backward chains -- for d = 8 (tcgen05 fused kernels) and d = 16 / 32 / 64
(tcd kernels) on ragged batches (the last tile partial), and fused and
per-step Multistage passes through the executor, then prints a digest of
every output.  With ACKPT_TC_CHAIN=force every launch after the first is
chained to its predecessor (programmatic dependent launch + per-tile
completion flags); with =0 none is; by default only the launches the
executor marks chain.  The digests must agree bit for bit
(tests/test_gpu_chain.py).
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def chain_run(d, batch, digest):
    """Back-to-back launches of one cell: Advance, two TapeForward chunks, two
    Reverse runs, then per-step forward / backward chains."""
    ops = lstm.operator_pair(lstm.long_memory_cell(d, 200, 0), batch, "f32")
    dc = ops.native
    s0 = lstm.random_states(d, 1, batch, "f32")

    def note(t):
        assert torch.isfinite(t).all()
        digest.update(t.detach().cpu().numpy().tobytes())

    for rep in range(2):  # the flag epochs advance across repetitions
        x = dc.advance(0, 8, s0)
        t1 = dc.forward_many(8, 48, x)
        t2 = dc.forward_many(56, 64, t1[-1])
        a = dc.seed(t2[-1])
        a = dc.backward_many(56, [t1[-1]] + t2[:-1], a)
        a = dc.backward_many(8, [x] + t1[:-1], a)
        y = s0
        for k in range(6):
            y = dc.forward(120 + k, y)
        b = a
        for k in range(6):
            b = dc.backward(126 - k, t2[k], b)
        torch.cuda.synchronize()
        for t in (x, t1[-1], t2[-1], a, y, b):
            note(t)
    with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as be:
        for fuse in (True, False):
            adj, _ = pkg.execute(pkg.Multistage(12, 17), ops, s0, be, fuse=fuse)
            note(adj)


def main():
    lstm.set_kernel_family("tcgen05")
    digest = hashlib.sha256()
    # ragged batches (last tile partial); d = 8 both reverse variants
    # (B % 4 == 0: bulk-copy prefetch of the taped state; else plain loads)
    for d, batch in ((8, (1 << 17) + 100), (8, (1 << 17) + 37), (16, (1 << 16) + 37), (32, (1 << 15) + 37),
                     (64, (1 << 14) + 37)):
        chain_run(d, batch, digest)
    print("chain_probe ok digest", digest.hexdigest())


if __name__ == "__main__":
    main()
