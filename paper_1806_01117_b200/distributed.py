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


# ---- host placement (each GPU pipelines its offload over its
# own host link, from a NUMA-local pinned slab) ------------------------------

def _gpu_pci(local_rank: int) -> str:
    p = torch.cuda.get_device_properties(local_rank)
    return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"


def _cpulist(text: str) -> set:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus


def bind_local_numa(local_rank: int) -> dict:
    """Pins this process to the CPUs of its GPU's NUMA node and prefers that
    node for new pages, so the pinned host slab (allocated and first touched
    by this process) and the tier's I/O threads sit next to the GPU's PCIe
    root.  Reads the topology from sysfs; a single-node host (or missing
    sysfs) leaves everything unchanged.  Returns what was done."""
    import ctypes
    import os

    out = {"gpu_pci": None, "numa_node": None, "cpus": None, "mempolicy": False}
    try:
        pci = _gpu_pci(local_rank)
        out["gpu_pci"] = pci
        with open(f"/sys/bus/pci/devices/{pci}/numa_node") as fh:
            node = int(fh.read().strip())
    except (OSError, ValueError, AttributeError, RuntimeError):
        return out
    nodes = [d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")] if os.path.isdir(
        "/sys/devices/system/node") else []
    out["numa_nodes"] = len(nodes)
    if node < 0 or len(nodes) < 2:
        return out  # one node: nothing to place
    with open(f"/sys/devices/system/node/node{node}/cpulist") as fh:
        cpus = _cpulist(fh.read()) & os.sched_getaffinity(0)
    if cpus:
        os.sched_setaffinity(0, cpus)
        out["cpus"] = sorted(cpus)
    out["numa_node"] = node
    try:  # set_mempolicy(MPOL_PREFERRED, {node}): new pages (the pinned slab) on the GPU's node
        libc = ctypes.CDLL(None, use_errno=True)
        mask = ctypes.c_ulong(1 << node)
        MPOL_PREFERRED, SYS_set_mempolicy = 1, 238  # x86-64
        out["mempolicy"] = libc.syscall(SYS_set_mempolicy, MPOL_PREFERRED, ctypes.byref(mask), 64) == 0
    except OSError:
        pass
    return out


def host_memory_available() -> int:
    """MemAvailable from /proc/meminfo, bytes (0 if unknown)."""
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def pinned_key_budget(state_bytes: int, local_ranks: int = 1, fraction: float = 0.8) -> int:
    """How many boundary states this rank may keep in pinned host DRAM: its
    share of `fraction` x MemAvailable (every rank of the node pins its own
    slab)."""
    avail = host_memory_available()
    if avail <= 0:
        return 1 << 30
    return max(0, int(avail * fraction) // max(1, local_ranks) // max(1, state_bytes))


def make_rank_backend(pkg, state_bytes: int, n_keys: int, local_ranks: int = 1, spill_dir=None):
    """The Level-2 backend of one rank for a plan with `n_keys` boundary
    states: the pinned-host tier when ⌈n/I⌉ x S x local_ranks fits the host-RAM
    budget (pinned_key_budget), else the three-stage cascade (pinned DRAM for
    the budget's worth of recent boundaries, older ones spilled to CKPT
    files under `spill_dir`)."""
    budget = pinned_key_budget(state_bytes, local_ranks)
    if n_keys <= budget:
        return pkg.PinnedHostBackend(slot_bytes=state_bytes)
    import tempfile

    directory = spill_dir or tempfile.mkdtemp(prefix="ackpt_spill_")
    return pkg.CascadeBackend(directory, slot_bytes=state_bytes, dram_slots=max(4, budget))
