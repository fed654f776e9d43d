"""Multi-GPU plumbing for the batch-sharded reverse pass.

The chain's time axis is serial, the batch of independent sequences is not:
every rank owns a contiguous shard of the global batch, runs the IDENTICAL
schedule on it (same interval, same plan) with its own HBM pool and its own
pinned tier on its own host link, and exchanges nothing during the pass.
Collectives only agree on the plan before the pass and reduce results after
it (torch.distributed; NCCL on GPUs, gloo for the CPU tests).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int  # first global sequence of this rank
    size: int   # sequences on this rank

    @property
    def stop(self) -> int:
        return self.start + self.size


def shard_of(global_batch: int, rank: int, world: int) -> Shard:
    """Contiguous near-equal split (the first `global_batch % world` ranks get
    one more sequence)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return Shard(rank, world, start, base + (1 if rank < extra else 0))


def _device_for_backend() -> torch.device:
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def agree_interval(interval: int) -> int:
    """All ranks adopt the largest calibrated interval, so every rank runs
    the identical multistage plan (stores still hide behind compute on the
    slowest link)."""
    if not (dist.is_available() and dist.is_initialized()):
        return int(interval)
    t = torch.tensor([int(interval)], dtype=torch.int64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return int(t.item())


def max_over_ranks(value: float) -> float:
    """Device-timed durations are reported as the max over ranks."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def adjoint_digest(adjoint) -> str:
    """sha256 of one shard's adjoint bytes (host copy)."""
    if isinstance(adjoint, torch.Tensor):
        data = adjoint.detach().contiguous().view(torch.uint8).cpu().numpy().tobytes()
    else:
        data = bytes(adjoint)
    return hashlib.sha256(data).hexdigest()


def gather_digests(digest: str) -> list:
    """Per-rank adjoint digests in rank order (end-of-run sanity check)."""
    if not (dist.is_available() and dist.is_initialized()):
        return [digest]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, digest)
    return out
