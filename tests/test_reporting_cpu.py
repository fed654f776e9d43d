"""Reporting parity on CPU: the simulator's timelines,
the model curves and the CLI's schedule / model / simulate outputs equal the
unmodified reference's, byte for byte (tests/golden/reporting_golden.json,
made by tests/golden/make_golden.py)."""

import contextlib
import io
import json
import os

import pytest

import paper_1806_01117_b200 as pkg
from paper_1806_01117_b200 import cli
from paper_1806_01117_b200.simulator import BACKWARD, FORWARD, coarsen

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "reporting_golden.json")) as fh:
        return json.load(fh)


def _strategy(kind, s, interval):
    return {"full": pkg.FullStorage(), "revolve": pkg.Revolve(s), "multistage": pkg.Multistage(s, interval)}[kind]


def test_simulator_timelines_match_reference(golden):
    for case in golden["simulate"]:
        kind, n, s, ta, tb, tt, interval = case["case"]
        strat = _strategy(kind, s, interval)
        events, total = pkg.simulate(strat, pkg.PerfParams(n=n, s=s, t_a=ta, t_b=tb, t_t=tt))
        assert pkg.timeline_to_json(strat, events, total) == case["json"], case["case"]


def test_simulated_totals_equal_model_when_interval_calibrated(golden):
    for case in golden["simulate"]:
        kind, n, s, ta, tb, tt, interval = case["case"]
        if interval is not None:
            continue
        strat = _strategy(kind, s, interval)
        p = pkg.PerfParams(n=n, s=s, t_a=ta, t_b=tb, t_t=tt)
        _, total = pkg.simulate(strat, p)
        model = {"full": pkg.t_infinity, "revolve": pkg.t_revolve, "multistage": pkg.t_async}[kind](p)
        assert model == case["t_model"]
        # the closed form n R(I, s) t_a + n t_b assumes whole intervals (or the fallback)
        if kind != "multistage" or n % pkg.interval_length(tt, ta) == 0 or pkg.interval_length(tt, ta) >= n:
            assert total == model, case["case"]


def test_forced_short_interval_stalls():
    p = pkg.PerfParams(n=24, s=2, t_a=1.0, t_b=2.0, t_t=7.0)
    events, total = pkg.simulate(pkg.Multistage(2, 4), p)
    stalls = [e for e in events if e.kind == "stall"]
    assert stalls and all(e.lane == "compute" and e.end > e.start for e in stalls)
    _, unloaded = pkg.simulate(pkg.Multistage(2, 4), pkg.PerfParams(n=24, s=2, t_a=1.0, t_b=2.0, t_t=1.0))
    assert total == unloaded + float(sum(e.end - e.start for e in stalls))


def test_model_curves_match_reference(golden):
    for case in golden["curves"]:
        s, intervals, n_max = case["case"]
        assert pkg.curves_to_csv(pkg.emit_curves(s, intervals, n_max)) == case["csv"]
    with pytest.raises(ValueError):
        pkg.emit_curves(2, [4], 0)


def test_cli_outputs_match_reference(golden):
    for case in golden["cli"]:
        out, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            rc = cli.main(case["argv"])
        assert rc == case["rc"], case["argv"]
        assert out.getvalue() == case["stdout"], case["argv"]
        if rc:
            assert err.getvalue().startswith("error: ")


def test_cli_bad_flags_exit_2():
    with pytest.raises(SystemExit) as exc, contextlib.redirect_stderr(io.StringIO()):
        cli.main(["simulate", "--strategy", "bogus", "--n", "3"])
    assert exc.value.code == 2


def test_coarsen_merges_fused_granularity():
    events, _ = pkg.simulate(pkg.Revolve(3), pkg.PerfParams(n=10, s=3, t_a=1.0, t_b=2.0, t_t=1.0))
    merged = coarsen(events)
    assert len(merged) < len(events)
    # same compute time and same per-kind step coverage
    def cover(evs, kind):
        return sorted(k for e in evs if e.kind == kind for k in range(e.from_step, e.to_step))
    for kind in (FORWARD, BACKWARD):
        assert cover(merged, kind) == cover(events, kind)
    assert sum(e.end - e.start for e in merged) == sum(e.end - e.start for e in events)
