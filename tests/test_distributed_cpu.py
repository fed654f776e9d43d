"""World-size-2 gloo tests of the batch-sharded multi-GPU host logic (CPU).

Each rank runs the oracle executor on its shard (the GPU kernels need a
device; the host logic does not): the plan agreement, the sharding, the
max-over-ranks timing and the digest gather must make the sharded run equal
the unsharded run sequence by sequence, with no exchange during the pass."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1806_01117_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from oracle import lstm_oracle as L
    from oracle import runtime_oracle as R

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, n, global_batch = 4, 24, 11
        shard = D.shard_of(global_batch, rank, world)
        cell = L.random_cell(d, n, 5)
        states = L.random_states(d, 9, global_batch)[:, :, shard.start:shard.stop]
        interval = D.agree_interval(6 + rank)  # ranks calibrate differently
        adj, st = R.execute("multistage", cell, np.ascontiguousarray(states), slots=3, interval=interval)
        elapsed = D.max_over_ranks(0.25 * (rank + 1))
        total_fwd = D.sum_over_ranks(st["forward_evals"])
        digests = D.gather_digests(D.adjoint_digest(adj.tobytes()))
        out[rank] = {"shard": (shard.start, shard.stop), "interval": interval, "adj": adj,
                     "elapsed": elapsed, "fwd": st["forward_evals"], "total_fwd": total_fwd,
                     "digests": digests, "stores": st["stores_issued"]}
    finally:
        dist.destroy_process_group()


def test_two_rank_batch_sharding_matches_unsharded_run():
    from oracle import lstm_oracle as L
    from oracle import runtime_oracle as R

    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    assert res[0]["shard"] == (0, 6) and res[1]["shard"] == (6, 11)
    assert res[0]["interval"] == res[1]["interval"] == 7  # identical plan on both ranks
    assert res[0]["elapsed"] == res[1]["elapsed"] == 0.5  # max over ranks
    assert res[0]["fwd"] == res[1]["fwd"] and res[0]["total_fwd"] == 2 * res[0]["fwd"]
    assert res[0]["digests"] == res[1]["digests"] and len(res[0]["digests"]) == 2
    # sharded adjoints == the unsharded run, sequence by sequence
    cell = L.random_cell(4, 24, 5)
    full, st = R.execute("multistage", cell, L.random_states(4, 9, 11), slots=3, interval=7)
    got = np.concatenate([res[0]["adj"], res[1]["adj"]], axis=2)
    np.testing.assert_allclose(got, full, rtol=1e-12, atol=1e-15)
    assert st["forward_evals"] == res[0]["fwd"]


def test_shard_of_covers_batch():
    for gb in (1, 7, 8, 1 << 20):
        for world in (1, 2, 3, 8):
            if world > gb:
                continue
            shards = [D.shard_of(gb, r, world) for r in range(world)]
            assert shards[0].start == 0 and shards[-1].stop == gb
            assert all(a.stop == b.start for a, b in zip(shards, shards[1:]))
            assert max(s.size for s in shards) - min(s.size for s in shards) <= 1
    with pytest.raises(ValueError):
        D.shard_of(8, 2, 2)


def test_helpers_without_process_group():
    assert D.agree_interval(5) == 5
    assert D.max_over_ranks(1.5) == 1.5
    assert D.gather_digests("x") == ["x"]
