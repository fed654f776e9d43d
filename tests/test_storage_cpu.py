"""Storage host logic on CPU: the CKPT byte format (vs the reference's own
golden encodings), corruption / truncation / magic detection, ENOSPC ->
StorageFull, and the Level-1 pool (pkg/tests/test_storage.py:38-169)."""

import os
import struct

import pytest

from paper_1806_01117_b200.errors import (ChecksumMismatch, MissingKey, SizeMismatch, SlotOutOfRange,
                                          SlotUnwritten, StorageFull)
from paper_1806_01117_b200.schedule import LoadCheckpoint, SaveCheckpoint, ScheduleParams, revolve_schedule, slot_read_liveness
from paper_1806_01117_b200.storage import (FILE_OVERHEAD, CheckpointPayload, Level1Pool, decode_checkpoint,
                                           encode_checkpoint, read_checkpoint_file, write_checkpoint_file, crc32c)


def test_encoding_matches_reference_bytes(storage_golden):
    assert encode_checkpoint(CheckpointPayload(5, b"\xab" * 8)).hex() == storage_golden["encoded_step5"]
    blob = encode_checkpoint(CheckpointPayload(123456789, bytes(range(40))))
    assert blob.hex() == storage_golden["encoded_step123456789"]
    assert decode_checkpoint(blob) == CheckpointPayload(123456789, bytes(range(40)))


def test_layout_is_fixed():
    blob = encode_checkpoint(CheckpointPayload(step=5, data=b"\xab" * 8))
    assert blob[:4] == b"CKPT"
    assert struct.unpack("<HQQ", blob[4:22]) == (1, 5, 8)
    assert struct.unpack("<I", blob[30:])[0] == crc32c(blob[:30])
    assert len(blob) == 8 + FILE_OVERHEAD


def test_decode_rejects_corruption_truncation_magic():
    blob = bytearray(encode_checkpoint(CheckpointPayload(1, b"x" * 64)))
    bad = bytearray(blob)
    bad[30] ^= 0xFF
    with pytest.raises(ChecksumMismatch):
        decode_checkpoint(bytes(bad))
    for cut in (40, 10):
        with pytest.raises(ChecksumMismatch):
            decode_checkpoint(bytes(blob[:cut]))
    bad = bytearray(blob)
    bad[0] = ord("X")
    with pytest.raises(ChecksumMismatch):
        decode_checkpoint(bytes(bad))


def test_file_round_trip_and_errors(tmp_path, monkeypatch):
    path = tmp_path / "ckpt_5.bin"
    write_checkpoint_file(path, CheckpointPayload(5, b"\x00" * 64))
    assert read_checkpoint_file(path, key=5) == CheckpointPayload(5, b"\x00" * 64)
    assert path.stat().st_size == 64 + FILE_OVERHEAD
    with pytest.raises(MissingKey):
        read_checkpoint_file(tmp_path / "ckpt_9.bin")
    write_checkpoint_file(path, CheckpointPayload(4, b"y" * 8))
    with pytest.raises(ChecksumMismatch):
        read_checkpoint_file(path, key=5)
    import builtins

    real_open = builtins.open

    def failing_open(*args, **kwargs):
        if args and str(args[0]).endswith(".tmp"):
            raise OSError(28, "No space left on device")
        return real_open(*args, **kwargs)

    monkeypatch.setattr(builtins, "open", failing_open)
    with pytest.raises(StorageFull):
        write_checkpoint_file(tmp_path / "ckpt_0.bin", CheckpointPayload(0, b"z"))


def test_level1_pool():
    pool = Level1Pool(capacity=2, slot_size=4)
    pool.save(1, CheckpointPayload(7, b"abcd"))
    assert pool.load(1) == CheckpointPayload(7, b"abcd")
    with pytest.raises(SlotOutOfRange):
        pool.save(2, CheckpointPayload(0, b"abcd"))
    with pytest.raises(SlotOutOfRange):
        pool.load(-1)
    with pytest.raises(SizeMismatch):
        pool.save(0, CheckpointPayload(0, b"toolong!"))
    with pytest.raises(SlotUnwritten):
        pool.load(0)
    pool = Level1Pool(capacity=4, slot_size=1)
    pool.save(0, CheckpointPayload(0, b"a"))
    pool.save(2, CheckpointPayload(1, b"b"))
    assert (pool.occupancy, pool.occupied_bytes) == (2, 2)
    pool.free(0)
    assert pool.occupancy == 1 and pool.peak_occupancy == 2
    pool.clear()
    assert pool.occupancy == 0


def test_pool_replaying_schedule_stays_within_budget():
    actions = revolve_schedule(ScheduleParams(10, 3))
    last_read = slot_read_liveness(actions)
    write_idx = {}
    pool = Level1Pool(capacity=3, slot_size=1)
    for idx, a in enumerate(actions):
        if isinstance(a, SaveCheckpoint):
            pool.save(a.slot, CheckpointPayload(a.step, b"s"))
            write_idx[a.slot] = idx
        elif isinstance(a, LoadCheckpoint):
            pool.load(a.slot)
            if last_read.get(write_idx[a.slot]) == idx:
                pool.free(a.slot)
    assert pool.peak_occupancy <= 3


def test_payload_validation():
    with pytest.raises(ValueError):
        CheckpointPayload(-1, b"")
    assert CheckpointPayload(3, os.urandom(0)).data == b""


@pytest.mark.parametrize("size", [12287, 12288, 12288 + 13, 100_003, (4 << 20) + 5, (16 << 20) - 1,
                                  (16 << 20) + 7, (33 << 20) + 3])
def test_crc32c_long_buffers_match_chained_short_calls(size):
    # long buffers take the 3-way interleaved and multi-threaded paths; short
    # calls (< 12 KiB each) take the single-chain path the golden vectors pin
    import numpy as np

    data = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8).tobytes()
    want = 0x1234
    for lo in range(0, size, 8000):
        want = crc32c(data[lo:lo + 8000], want)
    assert crc32c(data, 0x1234) == want
    assert crc32c(b"123456789") == 0xE3069283
