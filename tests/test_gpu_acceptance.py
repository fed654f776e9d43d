"""The reference's acceptance gates (pkg/tests/test_acceptance.py, one per
SPEC criterion) run against the GPU path.  Gates 1-3 are host-only and live
in tests/test_schedule_api.py and tests/test_native_abi.py."""

import numpy as np
import pytest
import torch

from oracle import lstm_oracle as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1806_01117_b200 as pkg
    import paper_1806_01117_b200.lstm as lstm
    import paper_1806_01117_b200.runtime as rt

    assert torch.cuda.is_available()
    return pkg, lstm, rt


def _loss64(lstm, cell, s0_bytes):
    dc = lstm.device_cell(cell, 1, "f64")
    x = dc._tensor(s0_bytes)
    for k in range(cell.n_steps):
        x = dc.forward(k, x)
    return float(dc.losses(x).item())


@pytest.mark.parametrize("d,n,seed", [(4, 8, 21), (8, 16, 22), (16, 32, 23)])
def test_04_gradient_matches_finite_differences(P, d, n, seed):
    pkg, lstm, _ = P
    cell = lstm.random_cell(d, n, seed)
    s0 = lstm.random_state(d, seed + 1)
    adjoint, _ = pkg.execute(pkg.FullStorage(), lstm.operator_pair(cell), s0)
    analytic = np.frombuffer(adjoint, "<f8")
    base = np.frombuffer(s0, "<f8").copy()
    numeric = np.empty_like(base)
    eps = 1e-6
    for i in range(base.size):
        plus, minus = base.copy(), base.copy()
        plus[i] += eps
        minus[i] -= eps
        numeric[i] = (_loss64(lstm, cell, plus.tobytes()) - _loss64(lstm, cell, minus.tobytes())) / (2 * eps)
    np.testing.assert_allclose(analytic, numeric, rtol=1e-5, atol=1e-8)


def test_05_bit_identical_adjoints_twenty_configs(P, tmp_path):
    pkg, lstm, _ = P
    configs = [(n, d, s, i) for n in (8, 12, 20, 32, 40) for d, s, i in [(4, 2, 4), (6, 3, 8), (8, 5, 6), (5, 4, 16)]]
    assert len(configs) == 20
    for seed, (n, d, s, interval) in enumerate(configs):
        cell = lstm.random_cell(d, n, 100 + seed)
        ops = lstm.operator_pair(cell)
        s0 = lstm.random_state(d, 200 + seed)
        g_full, _ = pkg.execute(pkg.FullStorage(), ops, s0)
        g_rev, _ = pkg.execute(pkg.Revolve(s), ops, s0)
        backend = pkg.FileBackend(tmp_path / f"c{seed}") if seed % 5 == 0 else pkg.SimulatedBackend(1e12, 0.0)
        try:
            g_ms, _ = pkg.execute(pkg.Multistage(s, interval=interval), ops, s0, backend)
        finally:
            backend.close()
        assert g_full == g_rev == g_ms, (n, d, s, interval)


def test_06_07_constant_multistage_vs_growing_revolve(P):
    pkg, lstm, _ = P
    d, s, interval, batch = 8, 4, 16, 4096
    multi, rev, peaks, full_peaks = {}, {}, {}, {}
    with pkg.PinnedHostBackend() as backend:
        for n in (64, 128, 256, 512):
            # long-memory cell: the adjoint stays far from fp32 underflow up
            # to n = 512, so the bit-identity below compares real numbers
            cell = lstm.long_memory_cell(d, n, 31)
            ops = lstm.operator_pair(cell, batch, "f32")
            s0 = lstm.random_states(d, 32, batch, "f32")
            g_ms, st = pkg.execute(pkg.Multistage(s, interval=interval), ops, s0, backend, fuse=True)
            assert g_ms.double().norm().item() > 1e-20
            multi[n], peaks[n] = st.forward_evals, st.peak_l1_bytes
            g_rev, st = pkg.execute(pkg.Revolve(s), ops, s0, fuse=True)
            rev[n] = st.forward_evals
            g_full, st = pkg.execute(pkg.FullStorage(), ops, s0, fuse=True)
            full_peaks[n] = st.peak_l1_bytes
            assert torch.equal(g_ms, g_rev) and torch.equal(g_ms, g_full)
    assert all(multi[a] * b == multi[b] * a for a in multi for b in multi)
    assert multi[64] == 64 + 4 * 33
    assert [rev[n] for n in (64, 128, 256, 512)] == [229, 587, 1475, 3657]
    assert len(set(peaks.values())) == 1
    for n in (64, 128, 256):
        assert full_peaks[2 * n] == 2 * full_peaks[n]


def test_08_asynchrony_stall_budget(P, monkeypatch):
    pkg, lstm, rt = P
    n, d, s, interval, step = 128, 4, 7, 8, 1e-3
    cell = lstm.random_cell(d, n, 51)
    ops = rt.pad_operator(lstm.operator_pair(cell), step, step)
    s0 = lstm.random_state(d, 52)

    def run():
        backend = pkg.SimulatedBackend(bandwidth=1e12, latency=(interval - 1) * step)
        try:
            return pkg.execute(pkg.Multistage(s, interval=interval), ops, s0, backend)
        finally:
            backend.close()

    # stall is wall-clock based (host sleeps on the copy streams): best of two
    # runs per mode, so one scheduling hiccup cannot decide the gate
    monkeypatch.delenv("CKPT_DISABLE_PREFETCH", raising=False)
    g_async, st_async = min((run() for _ in range(2)), key=lambda r: r[1].stall_seconds / r[1].wall_seconds)
    assert st_async.stall_seconds < 0.05 * st_async.wall_seconds
    monkeypatch.setenv("CKPT_DISABLE_PREFETCH", "1")
    g_sync, st_sync = min((run() for _ in range(2)), key=lambda r: r[1].stall_seconds)
    assert g_sync == g_async and st_sync.stall_seconds > st_async.stall_seconds


def test_09_wall_clock_dominance(P):
    # The reference pads nothing here: its Python steps (d=128) take ~100 us
    # against a 10 us transfer.  A GPU step is microseconds, so the steps are
    # stretched on the device to keep that compute/transfer ratio.
    pkg, lstm, rt = P
    grid = [(64, 2, 8), (128, 2, 8), (64, 3, 8), (128, 3, 8), (128, 4, 16), (256, 4, 16)]
    wins = 0
    for n, s, interval in grid:
        assert pkg.recompute_factor(n, s) > pkg.recompute_factor(interval, s)
        cell = lstm.random_cell(8, n, 61)
        ops = rt.pad_operator(lstm.operator_pair(cell), 1e-4, 1e-4)
        s0 = lstm.random_state(8, 62)
        with pkg.SimulatedBackend(bandwidth=1e12, latency=1e-5) as backend:
            multi = min((pkg.execute(pkg.Multistage(s, interval=interval), ops, s0, backend) for _ in range(3)),
                        key=lambda r: r[1].wall_seconds)
        rev = min((pkg.execute(pkg.Revolve(s), ops, s0) for _ in range(3)), key=lambda r: r[1].wall_seconds)
        assert multi[0] == rev[0]
        mw, rw = multi[1].wall_seconds, rev[1].wall_seconds
        assert mw <= 1.10 * rw, (n, s, interval, mw, rw)
        wins += mw < rw
    assert wins >= len(grid) / 2


def test_bench_report_fields_and_checksums(P):
    pkg, lstm, _ = P
    rep = lstm.bench(pkg.Multistage(3, interval=4), n=16, d=4, s=3, backend_config={"kind": "sim", "latency": 0.0},
                     seed=2, runs=2)
    assert (rep.n, rep.strategy, rep.forward_evals) == (16, "multistage", 32)
    assert rep.recompute_factor_measured == rep.forward_evals / 16
    assert len(rep.gradient_checksum) == 64 and rep.wall_seconds > 0
    kw = dict(n=16, d=4, s=3, seed=11, runs=1)
    full = lstm.bench(pkg.FullStorage(), **kw)
    rev = lstm.bench(pkg.Revolve(3), **kw)
    ms = lstm.bench(pkg.Multistage(3, interval=4), backend_config={"kind": "sim", "latency": 0.0}, **kw)
    assert full.gradient_checksum == rev.gradient_checksum == ms.gradient_checksum


def test_zero_cell_analytic(P):
    pkg, lstm, _ = P
    d = 3
    z = np.zeros
    cell = lstm.LstmCell(z((d, 2 * d)), z((d, 2 * d)), z((d, 2 * d)), z((d, 2 * d)), z(d), z(d), z(d), z(d),
                         xs=z((1, d)), target=z(d))
    c0 = np.array([1.0, -2.0, 0.5])
    out = lstm.lstm_forward_step(cell, 0, lstm.pack_state(np.zeros(d), c0))
    h, c = lstm.unpack_state(out, d)
    np.testing.assert_allclose(c, 0.5 * c0, rtol=1e-15)
    np.testing.assert_allclose(h, 0.5 * np.tanh(0.5 * c0), rtol=1e-15)
