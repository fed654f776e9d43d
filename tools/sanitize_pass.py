"""Small multistage passes for compute-sanitizer (memcheck / racecheck /
synccheck): every tier (pinned, CKPT file stage with its I/O threads and
stream memory operations, three-stage cascade) in both execution modes, plus
the per-step K1 / K2 kernels and the fused tcgen05 / FFMA2 launches at a
batch above the CTA-per-sequence crossover.  Exits non-zero on any mismatch.
Prints a digest of every adjoint it produced, so a run with ACKPT_POISON=1
(released / never-written HBM pool buffers NaN-filled: a copy or kernel that
reads a buffer outside the stream-ordering protocol sees NaN) can be compared
bit for bit with a plain run (tests/test_gpu_poison.py).

  compute-sanitizer --tool racecheck python tools/sanitize_pass.py
  ACKPT_POISON=1 python tools/sanitize_pass.py
"""
import hashlib
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    d, n, batch = 8, 48, 4096
    ops = lstm.operator_pair(lstm.long_memory_cell(d, n, 0), batch, "f32")
    s0 = lstm.random_states(d, 1, batch, "f32")
    ref = None
    digest = hashlib.sha256()

    def note(t):
        assert torch.isfinite(t).all()
        digest.update(t.detach().cpu().numpy().tobytes())

    with tempfile.TemporaryDirectory() as tmp:
        for fam in ("tcgen05", "ffma2"):
            lstm.set_kernel_family(fam)
            for fuse in (True, False):
                tiers = [pkg.PinnedHostBackend(slot_bytes=ops.state_size),
                         pkg.FileBackend(os.path.join(tmp, f"f{fam}{fuse}"), slot_bytes=ops.state_size),
                         pkg.CascadeBackend(os.path.join(tmp, f"c{fam}{fuse}"), slot_bytes=ops.state_size,
                                            dram_slots=4)]
                outs = []
                for b in tiers:
                    with b:
                        adj, _ = pkg.execute(pkg.Multistage(5, 6), ops, s0, b, fuse=fuse)
                        outs.append(adj)
                assert all(torch.equal(o, outs[0]) for o in outs), (fam, fuse)
                note(outs[0])
                # graph capture / replay over the pinned tier (third call replays)
                with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
                    for _ in range(3):
                        g, _ = pkg.execute(pkg.Multistage(5, 6), ops, s0, b, fuse=fuse, graph=True)
                        assert torch.equal(g, outs[0]), (fam, fuse, "graph")
                if fam == "ffma2" and not fuse:
                    ref = outs[0]
        # per-step K1 / K2 and a fused d=32 (tcgen05 tcd) pass
        dc = ops.native
        x = dc.forward(3, s0)
        a = dc.backward(3, x, s0)
        note(a)
        ops32 = lstm.operator_pair(lstm.random_cell(32, 12, 1), 4096, "f32")
        s32 = lstm.random_states(32, 2, 4096, "f32")
        with pkg.PinnedHostBackend(slot_bytes=ops32.state_size) as b:
            g, _ = pkg.execute(pkg.Multistage(3, 4), ops32, s32, b, fuse=True)
        note(g)
    torch.cuda.synchronize()
    print("sanitize_pass ok", float(ref.double().norm()), "digest", digest.hexdigest())


if __name__ == "__main__":
    main()
