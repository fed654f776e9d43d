"""Two-level checkpoint storage: the reference's storage API over HBM and
pinned host DRAM.

Reference: pkg/src/asyncckpt/storage.py.  The Level-2 backend's FIFO queue +
worker thread (storage.py:181-278) becomes the native tier (csrc/tier.cpp):
two copy-engine streams (D2H stores, H2D fetches) and one CUDA event per
TransferTicket.  Payload data are torch CUDA tensors (``bytes`` are accepted
and staged to the device).  Errors raised by a transfer surface at wait()
with the reference's exception classes.

The checkpoint file format (storage.py:9-18, 41-127) is kept byte-for-byte
for the optional third stage; its CRC32C runs natively (SSE4.2).
"""

from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Any, Optional

import torch

from . import _native as N
from .errors import (
    ChecksumMismatch,
    MissingKey,
    SizeMismatch,
    SlotOutOfRange,
    SlotUnwritten,
    StorageFull,
)

MAGIC = b"CKPT"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<HQQ")  # version, step, payload length
HEADER_BYTES = len(MAGIC) + _HEADER.size  # 22
TRAILER_BYTES = 4
FILE_OVERHEAD = HEADER_BYTES + TRAILER_BYTES


def crc32c(data, crc: int = 0) -> int:
    """CRC32C (Castagnoli); crc32c(b"123456789") == 0xE3069283."""
    buf = data if isinstance(data, bytes) else bytes(data)
    return int(N.lib.ackpt_crc32c(buf, len(buf), crc & 0xFFFFFFFF))


def nbytes_of(data: Any) -> int:
    if isinstance(data, torch.Tensor):
        return data.numel() * data.element_size()
    return len(data)


def as_host_bytes(data: Any) -> bytes:
    """Byte image of a payload (device tensors are copied back)."""
    if isinstance(data, torch.Tensor):
        return data.detach().contiguous().view(torch.uint8).cpu().numpy().tobytes()
    return bytes(data)


def as_device_bytes(data: Any, device=None) -> torch.Tensor:
    """Contiguous uint8 CUDA view (or staged copy) of a payload."""
    if isinstance(data, torch.Tensor):
        t = data.detach()
        if not t.is_cuda:
            t = t.to(device or "cuda")
        return t.contiguous().view(torch.uint8).reshape(-1)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if len(data) else torch.empty(0, dtype=torch.uint8)
    return host.to(device or "cuda")


@dataclass(frozen=True)
class CheckpointPayload:
    """Image of one program state: a device tensor or bytes (storage.py:71-80)."""

    step: int
    data: Any

    def __post_init__(self) -> None:
        if self.step < 0:
            raise ValueError(f"step must be >= 0, got {self.step}")

    def __eq__(self, other) -> bool:
        if not isinstance(other, CheckpointPayload):
            return NotImplemented
        return self.step == other.step and as_host_bytes(self.data) == as_host_bytes(other.data)

    def __hash__(self) -> int:
        return hash((self.step, nbytes_of(self.data)))


# ---- file format (storage.py:83-127) ----


def encode_checkpoint(payload: CheckpointPayload) -> bytes:
    data = as_host_bytes(payload.data)
    body = MAGIC + _HEADER.pack(FORMAT_VERSION, payload.step, len(data)) + data
    return body + struct.pack("<I", crc32c(body))


def decode_checkpoint(blob: bytes) -> CheckpointPayload:
    if len(blob) < FILE_OVERHEAD:
        raise ChecksumMismatch(f"checkpoint truncated: {len(blob)} bytes")
    if blob[:4] != MAGIC:
        raise ChecksumMismatch("bad magic bytes")
    version, step, length = _HEADER.unpack_from(blob, 4)
    if version != FORMAT_VERSION:
        raise ChecksumMismatch(f"unsupported format version {version}")
    if len(blob) != FILE_OVERHEAD + length:
        raise ChecksumMismatch(f"length field says {length}, file holds {len(blob) - FILE_OVERHEAD}")
    (stored,) = struct.unpack_from("<I", blob, HEADER_BYTES + length)
    actual = crc32c(blob[: HEADER_BYTES + length])
    if actual != stored:
        raise ChecksumMismatch(f"crc mismatch: {actual:#x} != {stored:#x}")
    return CheckpointPayload(step=step, data=blob[HEADER_BYTES : HEADER_BYTES + length])


def write_checkpoint_file(path: Path, payload: CheckpointPayload) -> None:
    """tmp file + os.replace; ENOSPC becomes StorageFull (storage.py:109-118)."""
    path = Path(path)
    tmp = path.with_suffix(path.suffix + ".tmp")
    try:
        with open(tmp, "wb") as fh:
            fh.write(encode_checkpoint(payload))
        os.replace(tmp, path)
    except OSError as exc:
        if exc.errno == 28:
            raise StorageFull(str(exc)) from exc
        raise


def read_checkpoint_file(path: Path, key: Optional[int] = None) -> CheckpointPayload:
    path = Path(path)
    if not path.exists():
        raise MissingKey(str(path))
    payload = decode_checkpoint(path.read_bytes())
    if key is not None and payload.step != key:
        raise ChecksumMismatch(f"file holds step {payload.step}, expected {key}")
    return payload


# ---- Level 1 (storage.py:130-178) ----


class Level1Pool:
    """Fixed set of same-sized checkpoint slots (references to device
    buffers; the executor's own pool lives in csrc/engine.cpp)."""

    def __init__(self, capacity: int, slot_size: int) -> None:
        if capacity < 0:
            raise ValueError(f"capacity must be >= 0, got {capacity}")
        if slot_size <= 0:
            raise ValueError(f"slot_size must be positive, got {slot_size}")
        self.capacity = capacity
        self.slot_size = slot_size
        self._slots: dict = {}
        self._peak = 0

    def _check(self, slot: int) -> None:
        if not 0 <= slot < self.capacity:
            raise SlotOutOfRange(f"slot {slot} outside capacity {self.capacity}")

    def save(self, slot: int, payload: CheckpointPayload) -> None:
        self._check(slot)
        size = nbytes_of(payload.data)
        if size != self.slot_size:
            raise SizeMismatch(f"payload is {size} bytes, slots hold {self.slot_size}")
        self._slots[slot] = payload
        self._peak = max(self._peak, len(self._slots))

    def load(self, slot: int) -> CheckpointPayload:
        self._check(slot)
        try:
            return self._slots[slot]
        except KeyError:
            raise SlotUnwritten(f"slot {slot} read before write") from None

    def free(self, slot: int) -> None:
        self._slots.pop(slot, None)

    def clear(self) -> None:
        self._slots.clear()

    @property
    def occupancy(self) -> int:
        return len(self._slots)

    @property
    def peak_occupancy(self) -> int:
        return self._peak

    @property
    def occupied_bytes(self) -> int:
        return len(self._slots) * self.slot_size


# ---- Level 2 (storage.py:181-278) ----


class TransferTicket:
    """Handle of one in-flight store or fetch (a CUDA event in the tier)."""

    def __init__(self, backend: "Level2Backend", kind: str, key: int, native_id: int, keep=None):
        self.backend = backend
        self.kind = kind
        self.key = key
        self.id = native_id
        self._keep = keep  # device buffer of a fetch / staged source of a store
        self._result: Optional[CheckpointPayload] = None
        self._waited = False

    @property
    def done(self) -> bool:
        return self.backend.poll(self)


class Level2Backend:
    """Asynchronous Level-2 stage in pinned host DRAM.

    Stores copy device bytes to a pinned host slot on the D2H copy engine;
    fetches copy them back on the H2D engine into a fresh device buffer.
    Keys are step indices; per-key FIFO order matches the reference's single
    worker.  ``latency``/``bandwidth`` throttle each transfer to at least
    latency + bytes / bandwidth seconds (SimulatedBackend semantics,
    storage.py:300-301) for stall-injection tests.
    """

    def __init__(
        self,
        slot_bytes: Optional[int] = None,
        capacity: int = 0,
        latency: float = 0.0,
        bandwidth: float = 0.0,
        device=None,
    ) -> None:
        self._slot_bytes = slot_bytes
        self._capacity = capacity
        self._latency = latency
        self._bandwidth = bandwidth
        self._device = torch.device(device or "cuda")
        self._handle: Optional[int] = None
        self._closed = False
        if slot_bytes is not None:
            self._ensure(slot_bytes)

    # -- native tier ----------------------------------------------------------
    def _ensure(self, nbytes: int) -> int:
        if self._closed:
            raise RuntimeError("backend is closed")
        if self._handle is None:
            size = max(int(nbytes), int(self._slot_bytes or 0), 1)
            self._handle = self._create_native(size)
            self._slot_bytes = size
            if self._latency or self._bandwidth:
                N.check(N.lib.ackpt_tier_set_throttle(self._handle, float(self._latency), float(self._bandwidth)))
        # payloads larger than the slab slots get dedicated pinned buffers per key
        return self._handle

    def _create_native(self, slot_bytes: int) -> int:
        h = C.c_void_p()
        N.check(N.lib.ackpt_tier_create(self._capacity, slot_bytes, C.byref(h)))
        return h.value

    @property
    def native(self) -> Optional[int]:
        return self._handle

    @property
    def slot_bytes(self) -> Optional[int]:
        return self._slot_bytes

    def set_throttle(self, latency: float, bandwidth: float = 0.0) -> None:
        self._latency, self._bandwidth = latency, bandwidth
        if self._handle is not None:
            N.check(N.lib.ackpt_tier_set_throttle(self._handle, float(latency), float(bandwidth)))

    # -- public API (storage.py:233-263) --------------------------------------
    def _hold(self, ticket_id: int, buf: torch.Tensor) -> None:
        """Keeps a transfer's device buffer alive until its ticket completed:
        the copy engines read (store) or write (fetch) it asynchronously, so a
        dropped ticket must not let the caching allocator hand the block to
        someone else mid-copy.  Released at wait / a completed poll / close
        (after the tier drained its streams)."""
        if buf.numel():
            if not hasattr(self, "_inflight"):
                self._inflight = {}
            self._inflight[ticket_id] = buf

    def begin_store(self, key: int, payload: CheckpointPayload) -> TransferTicket:
        """Asynchronous store; the payload must not be modified until the
        ticket completed (the reference stores immutable bytes, storage.py:233)."""
        src = as_device_bytes(payload.data, self._device)
        h = self._ensure(src.numel())
        out = C.c_int64(-1)
        stream = torch.cuda.current_stream(self._device).cuda_stream
        N.check(N.lib.ackpt_tier_begin_store(h, key, payload.step, src.data_ptr(), src.numel(), stream, C.byref(out)))
        self._hold(out.value, src)
        return TransferTicket(self, "store", key, out.value, keep=src)

    def begin_fetch(self, key: int) -> TransferTicket:
        h = self._ensure(0)
        size = C.c_int64(0)
        rc = N.lib.ackpt_tier_key_bytes(h, key, C.byref(size))
        dst = torch.empty(size.value if rc == N.OK else 0, dtype=torch.uint8, device=self._device)
        out = C.c_int64(-1)
        stream = torch.cuda.current_stream(self._device).cuda_stream
        N.check(N.lib.ackpt_tier_begin_fetch(h, key, dst.data_ptr(), dst.numel(), stream, C.byref(out)))
        self._hold(out.value, dst)
        return TransferTicket(self, "fetch", key, out.value, keep=dst)

    def wait(self, ticket: TransferTicket) -> Optional[CheckpointPayload]:
        step = C.c_int64(0)
        try:
            N.check(N.lib.ackpt_tier_wait(self._handle, ticket.id, C.byref(step)))
        finally:
            getattr(self, "_inflight", {}).pop(ticket.id, None)
        if ticket.kind == "fetch":
            if ticket._result is None:
                ticket._result = CheckpointPayload(step.value, ticket._keep)
            return ticket._result
        return None

    def poll(self, ticket: TransferTicket) -> bool:
        rc = N.lib.ackpt_tier_poll(self._handle, ticket.id)
        if rc == N.NOT_READY:
            return False
        getattr(self, "_inflight", {}).pop(ticket.id, None)
        return True  # complete (an error surfaces at wait)

    def contains(self, key: int) -> bool:
        if self._handle is None:
            return False
        out = C.c_int32(0)
        N.check(N.lib.ackpt_tier_contains(self._handle, key, C.byref(out)))
        return bool(out.value)

    def host_view(self, key: int) -> memoryview:
        """Pinned host bytes stored under key (valid once its store completed)."""
        ptr = C.c_void_p()
        N.check(N.lib.ackpt_tier_host_ptr(self._handle, key, C.byref(ptr)))
        size = C.c_int64(0)
        N.check(N.lib.ackpt_tier_key_bytes(self._handle, key, C.byref(size)))
        return memoryview((C.c_char * size.value).from_address(ptr.value)).cast("B")

    def close(self) -> None:
        if self._handle is not None and not self._closed:
            N.check(N.lib.ackpt_tier_destroy(self._handle))  # drains the copy streams first
        self._handle = None
        self._closed = True
        getattr(self, "_inflight", {}).clear()

    def __enter__(self) -> "Level2Backend":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass


class PinnedHostBackend(Level2Backend):
    """HBM <-> pinned host DRAM at full copy-engine speed (the product tier)."""


class FileBackend(Level2Backend):
    """Third stage: one CKPT file per key, ``<dir>/ckpt_<key>.bin``, in the
    reference's byte format (storage.py:321-340, tmp + rename, CRC32C).
    HBM -> pinned staging -> file on the D2H engine's stream, and back on the
    H2D stream; the file I/O and checksum run natively off the compute path.
    Corruption / truncation raise ChecksumMismatch, ENOSPC StorageFull, at
    wait (or at the end of an execute() that used the backend).  Existing
    files in the directory can be fetched (resume)."""

    def __init__(self, directory, slot_bytes=None, device=None):
        self.directory = Path(directory)
        self.directory.mkdir(parents=True, exist_ok=True)
        super().__init__(slot_bytes=slot_bytes, device=device)

    def _create_native(self, slot_bytes: int) -> int:
        h = C.c_void_p()
        N.check(N.lib.ackpt_tier_create_file(str(self.directory).encode(), slot_bytes, C.byref(h)))
        return h.value

    def path_for(self, key: int) -> Path:
        return self.directory / f"ckpt_{key}.bin"

    def contains(self, key: int) -> bool:
        self._ensure(1)  # files on disk count even before the first transfer
        return super().contains(key)

    def host_view(self, key: int):
        raise ValueError("file-stage keys live on disk; read path_for(key)")


class CascadeBackend(Level2Backend):
    """Three stages, HBM -> pinned host DRAM -> CKPT files (SURVEY §8(f)
    row 1, BASELINE config 5): ``dram_slots`` recent boundaries stay in pinned
    DRAM; older ones are spilled by a native I/O thread to
    ``<dir>/ckpt_<key>.bin`` in the reference's byte format (storage.py:9-18,
    CRC32C, O_DIRECT, atomic publish) and read back ahead of their fetch
    (two boundaries ahead, in the descending order of the multistage backward,
    runtime.py:297-322).  Errors surface at wait like FileBackend's; existing
    files can be fetched (resume).  Not capturable into a CUDA graph."""

    def __init__(self, directory, slot_bytes=None, dram_slots: int = 8, device=None):
        self.directory = Path(directory)
        self.directory.mkdir(parents=True, exist_ok=True)
        self.dram_slots = int(dram_slots)
        super().__init__(slot_bytes=slot_bytes, device=device)

    def _create_native(self, slot_bytes: int) -> int:
        h = C.c_void_p()
        N.check(N.lib.ackpt_tier_create_cascade(str(self.directory).encode(), slot_bytes, self.dram_slots,
                                                C.byref(h)))
        return h.value

    def path_for(self, key: int) -> Path:
        return self.directory / f"ckpt_{key}.bin"

    def contains(self, key: int) -> bool:
        self._ensure(1)
        return super().contains(key)

    def stats(self) -> dict:
        """Spill / read counters and host I/O seconds of the file stage."""
        out = N.CascadeStats()
        N.check(N.lib.ackpt_tier_cascade_stats(self._ensure(1), C.byref(out)))
        return {name: getattr(out, name) for name, _ in N.CascadeStats._fields_}


class SimulatedBackend(Level2Backend):
    """Pinned-host tier whose transfers take at least latency + size /
    bandwidth (x time_scale) of real time, like the reference's test double
    (storage.py:281-318), for contention and stall tests."""

    def __init__(self, bandwidth: float, latency: float, time_scale: float = 1.0, slot_bytes=None, device=None):
        if bandwidth <= 0:
            raise ValueError("bandwidth must be positive")
        if latency < 0:
            raise ValueError("latency must be >= 0")
        self.bandwidth = bandwidth
        self.latency = latency
        self.time_scale = time_scale
        super().__init__(
            slot_bytes=slot_bytes,
            latency=latency * time_scale,
            bandwidth=bandwidth / time_scale if time_scale > 0 else bandwidth,
            device=device,
        )

    def transfer_seconds(self, nbytes: int) -> float:
        return (self.latency + nbytes / self.bandwidth) * self.time_scale
