"""Level-2 tiers on the GPU: pinned host and the CKPT file stage
(pkg/tests/test_storage.py:171-291, acceptance gate 10 test_acceptance.py:243-269)."""

import os
import threading
import time

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


def test_pinned_round_trip_missing_idempotent(pkg):
    with pkg.SimulatedBackend(bandwidth=1e12, latency=0.0) as b:
        data = os.urandom(512)
        b.wait(b.begin_store(3, pkg.CheckpointPayload(3, data)))
        assert b.contains(3)
        out = b.wait(b.begin_fetch(3))
        assert _host(out) == data and out.step == 3
        t = b.begin_fetch(3)
        assert b.wait(t) is b.wait(t) and b.poll(t)
        with pytest.raises(pkg.MissingKey):
            b.wait(b.begin_fetch(99))


def test_simulated_latency_and_bandwidth(pkg):
    b = pkg.SimulatedBackend(bandwidth=1e12, latency=0.05)
    try:
        el = []
        for i in range(5):
            t0 = time.perf_counter()
            b.wait(b.begin_store(i, pkg.CheckpointPayload(i, b"q" * 64)))
            el.append(time.perf_counter() - t0)
        assert 0.05 <= sorted(el)[2] <= 0.055 * 1.1
    finally:
        b.close()
    b = pkg.SimulatedBackend(bandwidth=16 * 2**20, latency=0.0)
    try:
        b.wait(b.begin_store(0, pkg.CheckpointPayload(0, b"\x01" * 2**20)))  # first use: pinned allocation
        el = []
        for i in range(3):
            t0 = time.perf_counter()
            b.wait(b.begin_store(i, pkg.CheckpointPayload(i, b"\x01" * 2**20)))
            el.append(time.perf_counter() - t0)
        assert sorted(el)[1] == pytest.approx(0.0625, rel=0.10)
    finally:
        b.close()


def test_concurrent_store_and_fetch_distinct_keys(pkg):
    with pkg.PinnedHostBackend() as b:
        blobs = {k: os.urandom(128) for k in range(40)}
        for k in range(20):
            b.wait(b.begin_store(k, pkg.CheckpointPayload(k, blobs[k])))
        errors = []

        def writer():
            try:
                for k in range(20, 40):
                    b.wait(b.begin_store(k, pkg.CheckpointPayload(k, blobs[k])))
            except Exception as exc:  # pragma: no cover
                errors.append(exc)

        def reader():
            try:
                for k in range(20):
                    assert _host(b.wait(b.begin_fetch(k))) == blobs[k]
            except Exception as exc:  # pragma: no cover
                errors.append(exc)

        threads = [threading.Thread(target=writer), threading.Thread(target=reader)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors
        for k in range(40):
            assert _host(b.wait(b.begin_fetch(k))) == blobs[k]


def test_file_backend_format_and_errors(pkg, tmp_path):
    from paper_1806_01117_b200.storage import FILE_OVERHEAD, decode_checkpoint

    with pkg.FileBackend(tmp_path) as b:
        data = os.urandom(96)
        b.wait(b.begin_store(7, pkg.CheckpointPayload(7, data)))
        path = tmp_path / "ckpt_7.bin"
        assert path.exists() and path.stat().st_size == 96 + FILE_OVERHEAD
        assert decode_checkpoint(path.read_bytes()) == pkg.CheckpointPayload(7, data)  # reference format
        assert _host(b.wait(b.begin_fetch(7))) == data
        with pytest.raises(pkg.MissingKey):
            b.wait(b.begin_fetch(0))
        b.wait(b.begin_store(2, pkg.CheckpointPayload(2, b"m" * 32)))
        raw = bytearray((tmp_path / "ckpt_2.bin").read_bytes())
        raw[25] ^= 0x01
        (tmp_path / "ckpt_2.bin").write_bytes(bytes(raw))
        with pytest.raises(pkg.ChecksumMismatch):
            b.wait(b.begin_fetch(2))
        (tmp_path / "ckpt_7.bin").write_bytes(path.read_bytes()[:40])  # truncation
        with pytest.raises(pkg.ChecksumMismatch):
            b.wait(b.begin_fetch(7))
    # a new backend resumes from files already on disk
    with pkg.FileBackend(tmp_path) as b2:
        b2.wait(b2.begin_store(9, pkg.CheckpointPayload(9, b"resume")))
    with pkg.FileBackend(tmp_path) as b3:
        assert b3.contains(9)
        assert _host(b3.wait(b3.begin_fetch(9))) == b"resume"


def test_file_backend_plan_boundaries(pkg, tmp_path):
    from paper_1806_01117_b200.storage import FILE_OVERHEAD

    plan = pkg.plan_multistage(1000, 10, 100)
    with pkg.FileBackend(tmp_path) as b:
        tickets = [b.begin_store(k, pkg.CheckpointPayload(k, bytes([k % 251]) * 64)) for k in plan.boundaries]
        for t in tickets:
            b.wait(t)
    files = sorted(tmp_path.glob("ckpt_*.bin"))
    assert len(files) == 10 and all(f.stat().st_size == 64 + FILE_OVERHEAD for f in files)


def test_storage_round_trip_torture(pkg, tmp_path):
    # acceptance gate 10: 2000 round trips bit-identical; corruption detected
    rng = np.random.default_rng(71)
    backends = {"sim": pkg.SimulatedBackend(bandwidth=1e12, latency=0.0), "file": pkg.FileBackend(tmp_path / "t")}
    try:
        for name, b in backends.items():
            for i in range(1000):
                key = int(rng.integers(0, 500))
                data = rng.bytes(int(rng.integers(1, 513)))
                b.wait(b.begin_store(key, pkg.CheckpointPayload(key, data)))
                assert _host(b.wait(b.begin_fetch(key))) == data, (name, i)
    finally:
        for b in backends.values():
            b.close()
    with pkg.FileBackend(tmp_path / "corrupt") as b:
        b.wait(b.begin_store(1, pkg.CheckpointPayload(1, b"n" * 128)))
        p = tmp_path / "corrupt" / "ckpt_1.bin"
        raw = bytearray(p.read_bytes())
        raw[40] ^= 0x10
        p.write_bytes(bytes(raw))
        with pytest.raises(pkg.ChecksumMismatch):
            b.wait(b.begin_fetch(1))


def test_execute_multistage_through_file_stage(pkg, tmp_path):
    import paper_1806_01117_b200.lstm as lstm

    cell = lstm.random_cell(8, 40, 3)
    ops = lstm.operator_pair(cell, 4096, "f32")
    s0 = lstm.random_states(8, 4, 4096, "f32")
    with pkg.FileBackend(tmp_path) as b:
        for fuse in (False, True):
            ref, _ = pkg.execute(pkg.FullStorage(), ops, s0, fuse=fuse)
            adj, st = pkg.execute(pkg.Multistage(5, interval=8), ops, s0, b, fuse=fuse)
            assert torch.equal(adj, ref)
            assert st.stores_issued == st.prefetches_issued == 5
    assert sorted(p.name for p in tmp_path.glob("ckpt_*.bin")) == [f"ckpt_{k}.bin" for k in (0, 16, 24, 32, 8)]
    # corrupt a boundary file between the passes' sweeps: the run must fail loudly
    with pkg.FileBackend(tmp_path) as b:
        plan = pkg.plan_multistage(40, 5, 8)
        _, fin = pkg.run_forward_sweep(plan, ops, b, s0)
        raw = bytearray((tmp_path / "ckpt_16.bin").read_bytes())
        raw[100] ^= 0xFF
        (tmp_path / "ckpt_16.bin").write_bytes(bytes(raw))
        with pytest.raises(pkg.ChecksumMismatch):
            pkg.run_backward_sweep(plan, ops, b, lstm.loss_gradient_seed(cell, fin))


def test_bench_file_backend_round_trip(pkg, tmp_path):
    import paper_1806_01117_b200.lstm as lstm

    rep = lstm.bench(pkg.Multistage(3, interval=8), n=24, d=4, s=3,
                     backend_config={"kind": "file", "dir": str(tmp_path)}, seed=4, runs=1)
    for k in (0, 8, 16):
        assert (tmp_path / f"ckpt_{k}.bin").exists()
    base = lstm.bench(pkg.FullStorage(), n=24, d=4, s=3, seed=4, runs=1)
    assert rep.gradient_checksum == base.gradient_checksum


@pytest.mark.timeout(180)
def test_file_stage_write_failure_surfaces_without_hanging(pkg, tmp_path):
    # the CKPT directory disappears before a pass: every store's file write
    # fails on the tier's I/O thread; the copy streams must still drain and
    # the run must raise (not hang), and the backend must close cleanly
    import shutil

    import paper_1806_01117_b200.lstm as lstm

    cell = lstm.random_cell(8, 40, 3)
    ops = lstm.operator_pair(cell, 4096, "f32")
    s0 = lstm.random_states(8, 4, 4096, "f32")
    d = tmp_path / "gone"
    d.mkdir()
    b = pkg.FileBackend(d)
    try:
        shutil.rmtree(d)
        for fuse in (False, True):
            with pytest.raises((pkg.ExecutionError, pkg.MissingKey, pkg.StorageFull, pkg.ChecksumMismatch)):
                pkg.execute(pkg.Multistage(5, interval=8), ops, s0, b, fuse=fuse)
        # the engine and tier stay usable once the directory is back
        d.mkdir()
        ref, _ = pkg.execute(pkg.FullStorage(), ops, s0, fuse=True)
        adj, _ = pkg.execute(pkg.Multistage(5, interval=8), ops, s0, b, fuse=True)
        assert torch.equal(adj, ref)
    finally:
        b.close()


def test_file_stage_enospc_maps_to_storage_full(pkg, tmp_path):
    # storage.py:109-118 + errors: a full device surfaces as StorageFull at
    # wait.  The native file stage writes <key>.tmp first: pointing that name
    # at /dev/full (every write fails with ENOSPC) exercises the real path.
    if not os.path.exists("/dev/full"):
        pytest.skip("no /dev/full")
    with pkg.FileBackend(tmp_path) as b:
        os.symlink("/dev/full", tmp_path / "ckpt_5.bin.tmp")
        with pytest.raises(pkg.StorageFull):
            b.wait(b.begin_store(5, pkg.CheckpointPayload(5, b"x" * 4096)))
        assert not (tmp_path / "ckpt_5.bin").exists()
        # the tier keeps working for other keys
        b.wait(b.begin_store(6, pkg.CheckpointPayload(6, b"y" * 64)))
        assert _host(b.wait(b.begin_fetch(6))) == b"y" * 64
