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
(tests/test_gpu_chain.py); executor passes are left out under =force, which
would also chain across the executor's transfer waits.  Forced chaining assumes what the executor's
HBM pool guarantees: no memory a launch reads is freed and reallocated
before the next launch completes -- so the probe keeps every tensor alive
until it synchronizes.
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def chain_run(d, batch, digest, engine_digest):
    """Back-to-back launches of one cell: Advance, two TapeForward chunks, two
    Reverse runs, then per-step forward / backward chains."""
    ops = lstm.operator_pair(lstm.long_memory_cell(d, 200, 0), batch, "f32")
    dc = ops.native
    s0 = lstm.random_states(d, 1, batch, "f32")

    def note(t):
        assert torch.isfinite(t).all()
        digest.update(t.detach().cpu().numpy().tobytes())

    for rep in range(2):  # the flag epochs advance across repetitions
        # every tensor stays referenced until the synchronize: a chained
        # launch may still run while its successor starts, so memory it reads
        # must not be handed back to the caching allocator in between (the
        # executor's HBM pool never moves a buffer)
        keep = []
        x = dc.advance(0, 8, s0)
        t1 = dc.forward_many(8, 48, x)
        t2 = dc.forward_many(56, 64, t1[-1])
        a = dc.seed(t2[-1])
        keep.append(a)
        a = dc.backward_many(56, [t1[-1]] + t2[:-1], a)
        keep.append(a)
        a = dc.backward_many(8, [x] + t1[:-1], a)
        y = s0
        for k in range(6):
            y = dc.forward(120 + k, y)
            keep.append(y)
        b = a
        for k in range(6):
            b = dc.backward(126 - k, t2[k], b)
            keep.append(b)
        torch.cuda.synchronize()
        for t in (x, t1[-1], t2[-1], a, y, b):
            note(t)
        del keep
    if engine_digest is None:  # =force: the executor's own marks are bypassed (transfer waits would chain)
        return
    with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as be:
        for fuse in (True, False):
            adj, _ = pkg.execute(pkg.Multistage(12, 17), ops, s0, be, fuse=fuse)
            assert torch.isfinite(adj).all()
            engine_digest.update(adj.detach().cpu().numpy().tobytes())


def two_cells(d, batch, digest):
    """Two cells alternating on one stream, each reading the other's output:
    no launch may chain across another cell's launch (chain_touch)."""
    A = lstm.device_cell(lstm.long_memory_cell(d, 64, 0), batch, "f32")
    Bc = lstm.device_cell(lstm.long_memory_cell(d, 64, 1), batch, "f32")
    x = lstm.random_states(d, 2, batch, "f32")
    outs, keep = [], []  # (every tensor held until the synchronize, as in chain_run)
    for _ in range(3):
        a = A.forward_many(0, 16, x)
        b = Bc.advance(0, 24, a[-1])
        x = A.advance(16, 40, b)
        outs += [a[-1], b, x]
        keep += a
    torch.cuda.synchronize()
    for t in outs:
        assert torch.isfinite(t).all()
        digest.update(t.detach().cpu().numpy().tobytes())


def two_streams(d, batch, digest):
    """One cell alternating between two streams: no launch may chain across
    streams (per-stream flag arrays, chain.cuh)."""
    A = lstm.device_cell(lstm.long_memory_cell(d, 64, 0), batch, "f32")
    y = lstm.random_states(d, 2, batch, "f32")
    outs = []
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for k in range(4):
        st = s1 if k % 2 == 0 else s2
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            y = A.advance(0, 16, y)
        torch.cuda.current_stream().wait_stream(st)
        outs.append(y)
    torch.cuda.synchronize()
    for t in outs:
        assert torch.isfinite(t).all()
        digest.update(t.detach().cpu().numpy().tobytes())


def main():
    lstm.set_kernel_family("tcgen05")
    digest = hashlib.sha256()
    def section(name, fn, *args):
        h = hashlib.sha256()
        fn(*args, h)
        digest.update(h.digest())
        print("section", name, h.hexdigest()[:16], flush=True)

    for d, batch in ((8, (1 << 17) + 100), (32, (1 << 15) + 37)):
        section(f"two-cells-d{d}", two_cells, d, batch)
        section(f"two-streams-d{d}", two_streams, d, batch)
    # ragged batches (last tile partial); d = 8 both reverse variants
    # (B % 4 == 0: bulk-copy prefetch of the taped state; else plain loads)
    forced = os.environ.get("ACKPT_TC_CHAIN") == "force"
    engine = None if forced else hashlib.sha256()
    for d, batch in ((8, (1 << 17) + 100), (8, (1 << 17) + 37), (16, (1 << 16) + 37), (32, (1 << 15) + 37),
                     (64, (1 << 14) + 37)):
        section(f"run-d{d}-B{batch}", lambda h: chain_run(d, batch, h, engine))
    print("chain_probe ok direct", digest.hexdigest(), "engine", engine.hexdigest() if engine else "skipped")


if __name__ == "__main__":
    main()
