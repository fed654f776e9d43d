"""Three-stage tier HBM -> pinned DRAM -> CKPT files (CascadeBackend,
csrc/cascade_impl.h): SURVEY §8(f) row 1, BASELINE config 5.

Checks the reference's Level-2 contract (storage.py:181-278: FIFO per key,
idempotent wait, errors at wait) on a tier whose DRAM holds only a few
boundaries, the byte format of the spilled files (storage.py:9-18, 83-127),
read-ahead, resume, corruption / ENOSPC, and a multistage execute() through
it: same adjoint bits and counters as the pinned tier."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_1806_01117_b200 as p

    assert torch.cuda.is_available()
    return p


def _host(payload):
    from paper_1806_01117_b200.storage import as_host_bytes

    return as_host_bytes(payload.data)


def _blob(i, n):
    return np.random.default_rng(i).integers(0, 256, n, dtype=np.uint8).tobytes()


def test_spill_and_read_back_in_descending_order(pkg, tmp_path):
    from paper_1806_01117_b200.storage import read_checkpoint_file

    n, keys = 1 << 20, list(range(0, 120, 10))
    with pkg.CascadeBackend(tmp_path, slot_bytes=n, dram_slots=4) as b:
        for k in keys:  # one store in flight, like the multistage sweep (runtime.py:281-293)
            b.wait(b.begin_store(k, pkg.CheckpointPayload(k, _blob(k, n))))
        assert all(b.contains(k) for k in keys)
        for k in reversed(keys):  # the backward's order, one fetch ahead
            out = b.wait(b.begin_fetch(k))
            assert out.step == k and _host(out) == _blob(k, n), k
        st = b.stats()
        assert st["spills"] >= len(keys) - 4
        assert st["dram_hits"] >= 2 and st["ring_hits"] >= 1
        # every spilled file is a CKPT file in the reference's format
        spilled = [k for k in keys if (tmp_path / f"ckpt_{k}.bin").exists()]
        assert len(spilled) >= len(keys) - 4
        for k in spilled:
            p = read_checkpoint_file(tmp_path / f"ckpt_{k}.bin", k)
            assert p.step == k and bytes(p.data) == _blob(k, n)
            assert os.path.getsize(tmp_path / f"ckpt_{k}.bin") == 22 + n + 4


def test_random_access_restore_and_idempotent_wait(pkg, tmp_path):
    n = 64 << 10
    with pkg.CascadeBackend(tmp_path, slot_bytes=n, dram_slots=4) as b:
        for k in range(10):
            b.wait(b.begin_store(k, pkg.CheckpointPayload(k, _blob(k, n))))
        b.wait(b.begin_store(2, pkg.CheckpointPayload(2, _blob(200, n))))  # a new version of a spilled key
        for k in (0, 7, 2, 9, 1, 2, 5):
            t = b.begin_fetch(k)
            out = b.wait(t)
            assert b.wait(t) is out and b.poll(t)
            assert _host(out) == (_blob(200, n) if k == 2 else _blob(k, n)), k
        with pytest.raises(pkg.MissingKey):
            b.wait(b.begin_fetch(99))


def test_resume_from_files_and_corruption(pkg, tmp_path):
    n = 256 << 10
    with pkg.CascadeBackend(tmp_path, slot_bytes=n, dram_slots=4) as b:
        for k in range(8):
            b.wait(b.begin_store(k, pkg.CheckpointPayload(k, _blob(k, n))))
        b.wait(b.begin_fetch(0))  # spilled keys are on file once read back
    # a new tier on the same directory fetches the files (resume)
    with pkg.CascadeBackend(tmp_path, slot_bytes=n, dram_slots=4) as b:
        assert b.contains(1)
        assert _host(b.wait(b.begin_fetch(1))) == _blob(1, n)
        path = tmp_path / "ckpt_3.bin"
        raw = bytearray(path.read_bytes())
        raw[100] ^= 0xFF
        path.write_bytes(bytes(raw))
        with pytest.raises(pkg.ChecksumMismatch):
            b.wait(b.begin_fetch(3))
        path.write_bytes(b"CKPT" + b"\x00" * 10)
        with pytest.raises(pkg.ChecksumMismatch):
            b.wait(b.begin_fetch(3))


def test_spill_enospc_surfaces_as_storage_full(pkg, tmp_path):
    if not os.path.exists("/dev/full"):
        pytest.skip("no /dev/full")
    n = 64 << 10
    os.symlink("/dev/full", tmp_path / "ckpt_0.bin.tmp")
    with pkg.CascadeBackend(tmp_path, slot_bytes=n, dram_slots=4) as b:
        for k in range(8):  # key 0 is spilled (fails) and evicted
            b.wait(b.begin_store(k, pkg.CheckpointPayload(k, _blob(k, n))))
        with pytest.raises(pkg.StorageFull):
            b.wait(b.begin_fetch(0))
        assert _host(b.wait(b.begin_fetch(1))) == _blob(1, n)  # the tier keeps working


def test_multistage_execute_matches_pinned_tier(pkg, tmp_path):
    import paper_1806_01117_b200.lstm as lstm

    d, n, batch, s, interval = 8, 240, 4096, 11, 10
    ops = lstm.operator_pair(lstm.long_memory_cell(d, n, 3), batch, "f32")
    s0 = lstm.random_states(d, 4, batch, "f32")
    strategy = pkg.Multistage(s, interval)
    for fuse in (False, True):
        with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
            ref, st_ref = pkg.execute(strategy, ops, s0, b, fuse=fuse)
        with pkg.CascadeBackend(tmp_path / f"f{int(fuse)}", slot_bytes=ops.state_size, dram_slots=5) as b:
            got, st = pkg.execute(strategy, ops, s0, b, fuse=fuse)
            got2, _ = pkg.execute(strategy, ops, s0, b, fuse=fuse)  # second pass re-stores every key
            cs = b.stats()
        assert torch.equal(got, ref) and torch.equal(got2, ref)
        assert got.double().norm().item() > 0
        for key in ("forward_evals", "backward_evals", "stores_issued", "prefetches_issued", "peak_l1_bytes"):
            assert getattr(st, key) == getattr(st_ref, key), key
        assert cs["spills"] >= 2 * (n // interval - 5) and cs["ring_hits"] + cs["ring_misses"] > 0


def test_calibrate_paces_stores_by_the_spill_stage(pkg, tmp_path):
    import paper_1806_01117_b200.lstm as lstm

    d, n, batch = 8, 2000, 1 << 18
    ops = lstm.operator_pair(lstm.random_cell(d, n, 0), batch, "f32")
    s0 = lstm.random_states(d, 1, batch, "f32")
    with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
        _, _, t_pinned = pkg.calibrate(ops, b, 5, s0, fuse=True)
    with pkg.CascadeBackend(tmp_path, slot_bytes=ops.state_size, dram_slots=4) as b:
        _, _, t_cascade = pkg.calibrate(ops, b, 5, s0, fuse=True)
    # the file stage (~2-3 GB/s) is far slower than the pinned copy (~55 GB/s)
    assert t_cascade > 3 * t_pinned


def test_graph_capture_is_rejected(pkg, tmp_path):
    import paper_1806_01117_b200.lstm as lstm

    ops = lstm.operator_pair(lstm.random_cell(8, 40, 0), 4096, "f32")
    s0 = lstm.random_states(8, 1, 4096, "f32")
    with pkg.CascadeBackend(tmp_path, slot_bytes=ops.state_size, dram_slots=4) as b:
        pkg.execute(pkg.Multistage(3, 4), ops, s0, b, graph=True)  # eager run: records the buffers
        with pytest.raises(ValueError):
            pkg.execute(pkg.Multistage(3, 4), ops, s0, b, graph=True)  # capture attempt
