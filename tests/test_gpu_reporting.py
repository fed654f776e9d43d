"""Measured timelines of the GPU executor against the reference's simulator
semantics, and the CLI's bench on the device."""

import contextlib
import io
import json

import pytest
import torch

import paper_1806_01117_b200 as pkg
import paper_1806_01117_b200.lstm as lstm
from paper_1806_01117_b200 import cli
from paper_1806_01117_b200.simulator import BACKWARD, FETCH, FORWARD, STALL, STORE

pytestmark = pytest.mark.gpu


def _steps(events, kind):
    return sorted(k for e in events if e.kind == kind for k in range(e.from_step, e.to_step))


@pytest.mark.parametrize("fuse", [False, True])
def test_measured_multistage_timeline_matches_simulator(fuse):
    # t_a = 1 ms, t_b = 2 ms (device-side padding), t_t = 7 ms (throttled
    # tier), interval forced to 4 < t_t / t_a: the simulator's stall case
    n, s, interval, ta, tb, tt = 24, 2, 4, 1e-3, 2e-3, 7e-3
    d, batch = 8, 256
    ops = pkg.runtime.pad_operator(lstm.operator_pair(lstm.random_cell(d, n, 0), batch, "f32"), ta, tb)
    s0 = lstm.random_states(d, 1, batch, "f32")
    strat = pkg.Multistage(s, interval)
    with pkg.SimulatedBackend(bandwidth=1e15, latency=tt) as backend:
        adj_plain, _ = pkg.execute(strat, ops, s0, backend, fuse=fuse)
        adj, st = pkg.execute(strat, ops, s0, backend, fuse=fuse, timeline=True)
    assert torch.equal(adj, adj_plain)  # the timeline mode does not change results
    sim, sim_total = pkg.simulate(strat, pkg.PerfParams(n=n, s=s, t_a=ta, t_b=tb, t_t=tt))
    got = st.timeline
    # transfer lane: the same stores and fetches, same keys, same order
    lane = lambda evs: [(e.kind, e.from_step) for e in evs if e.lane == "transfer"]
    assert lane(got) == lane(sim)
    assert len([e for e in got if e.kind == STORE]) == st.stores_issued
    assert len([e for e in got if e.kind == FETCH]) == st.prefetches_issued
    # reverse coverage equal; the executor re-runs each interval's first
    # traversal (runtime.py:23-27), so its forward coverage is the
    # simulator's plus one pass over every step
    assert _steps(got, BACKWARD) == _steps(sim, BACKWARD)
    assert _steps(got, FORWARD) == sorted(_steps(sim, FORWARD) + list(range(n)))
    assert len(_steps(got, FORWARD)) == st.forward_evals
    # stalls: wherever the simulator stalls the store wait is exposed too
    sim_stalls = {e.from_step for e in sim if e.kind == STALL}
    got_stalls = {e.from_step for e in got if e.kind == STALL and e.end - e.start > 0.2 * ta}
    assert sim_stalls and sim_stalls <= got_stalls
    # compute-lane busy time: the simulator's plus the re-run first traversals,
    # within launch overheads (stall lengths depend on host-sleep jitter of
    # the throttled tier, so the total is only bounded below)
    busy = lambda evs: sum(float(e.end - e.start) for e in evs if e.kind in (FORWARD, BACKWARD))
    assert busy(got) == pytest.approx(busy(sim) + n * ta, rel=0.25)
    gpu = st.device["gpu_seconds"]
    assert gpu >= busy(got)
    # events are ordered and inside the run
    starts = [e.start for e in got]
    assert starts == sorted(starts) and all(0 <= e.start <= e.end <= gpu * 1.01 + 1e-4 for e in got)


def test_cli_bench_on_device(tmp_path):
    path = tmp_path / "timeline.json"
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        rc = cli.main(["bench", "--strategy", "multistage", "--n", "40", "--d", "8", "--s", "8", "--interval", "8",
                       "--runs", "2", "--batch", "4096", "--dtype", "f32", "--fuse", "--backend", "pinned",
                       "--timeline", str(path)])
    assert rc == 0
    rep = json.loads(out.getvalue())
    assert rep["strategy"] == "multistage" and rep["forward_evals"] == 80
    assert rep["recompute_factor_measured"] == 2.0
    tl = json.loads(path.read_text())
    assert tl["strategy"] == "multistage" and tl["total"] > 0
    kinds = {e["kind"] for e in tl["events"]}
    assert {"forward_compute", "backward_compute", "store", "fetch"} <= kinds
    # the reference's default workload (batch 1, float64 byte image)
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        assert cli.main(["bench", "--strategy", "revolve", "--n", "30", "--d", "8", "--s", "4", "--runs", "1"]) == 0
    assert json.loads(out.getvalue())["forward_evals"] == pkg.forward_cost(30, 4)


def test_cli_bench_graph_same_checksum():
    # --graph replays the pass as a CUDA graph: same counters and gradient checksum
    reps = []
    for extra in ([], ["--graph"]):
        out = io.StringIO()
        with contextlib.redirect_stdout(out):
            assert cli.main(["bench", "--strategy", "revolve", "--n", "40", "--d", "32", "--s", "5", "--runs", "3"]
                            + extra) == 0
        reps.append(json.loads(out.getvalue()))
    assert reps[0]["gradient_checksum"] == reps[1]["gradient_checksum"]
    assert reps[0]["forward_evals"] == reps[1]["forward_evals"] == pkg.forward_cost(40, 5)
