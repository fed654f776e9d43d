"""Rank program of tests/test_gpu_multirank.py (launched by torchrun with the
gloo backend; every rank on cuda:0 -- this run has one GPU).

Each rank owns a contiguous batch shard (distributed.shard_of), builds its
own operator pair, HBM pool and pinned tier, agrees the interval with the
other ranks (all_reduce MAX, distributed.agree_interval) and runs the real
multistage engine on its shard -- no collective inside the pass (SURVEY
§8(e)).  Rank 0 also runs the unsharded batch; the shards' adjoints are
gathered and compared with it sequence by sequence.  Prints one JSON line
(rank 0)."""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.distributed as D  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    d, n, global_b, slots = 8, 300, 8192, 29
    fuse = os.environ.get("MR_FUSE", "1") == "1"
    cell = lstm.long_memory_cell(d, n, 0)
    full = lstm.random_states(d, 1, global_b, "f32")  # the global batch (same draws on every rank)
    sh = D.shard_of(global_b, rank, world)
    s0 = full[:, :, sh.start:sh.stop].contiguous()
    ops = lstm.operator_pair(cell, sh.size, "f32")
    with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
        t_a, _, t_t = pkg.calibrate(ops, b, 5, s0, fuse=fuse)
        mine = pkg.interval_length(t_t, t_a)
        interval = D.agree_interval(max(2, min(mine, 25)))
        adj, st = pkg.execute(pkg.Multistage(slots, interval), ops, s0, b, fuse=fuse)
    torch.cuda.synchronize()
    shards = [None] * world
    dist.all_gather_object(shards, (sh.start, sh.stop, adj.cpu().numpy(), st.forward_evals, interval))
    digests = D.gather_digests(D.adjoint_digest(adj))
    if rank == 0:
        ops_all = lstm.operator_pair(cell, global_b, "f32")
        with pkg.PinnedHostBackend(slot_bytes=ops_all.state_size) as b:
            ref, st_ref = pkg.execute(pkg.Multistage(slots, interval), ops_all, full, b, fuse=fuse)
        ref = ref.cpu().numpy()
        same = all(np.array_equal(a, ref[:, :, lo:hi]) for lo, hi, a, _, _ in shards)
        covered = sorted((lo, hi) for lo, hi, *_ in shards)
        print(json.dumps({
            "world": world, "interval": interval, "intervals_agreed": len({s[4] for s in shards}) == 1,
            "bit_identical_to_unsharded": bool(same),
            "covers_batch": covered[0][0] == 0 and covered[-1][1] == global_b and
                            all(covered[i][1] == covered[i + 1][0] for i in range(len(covered) - 1)),
            "forward_evals_equal": all(s[3] == st_ref.forward_evals for s in shards),
            "adjoint_norm": float(np.linalg.norm(ref)), "digests": digests,
        }), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
