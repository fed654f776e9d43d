"""Property tests (hypothesis) of the native scheduler against the oracle's
restatement of schedule.py on random (n, s, I): costs, the Revolve action
sequence (JSON, byte for byte), multistage plans and their segments, and the
exact rational interval_length.  CPU only (host-side C code)."""

import math
from fractions import Fraction

from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import schedule_oracle as S
from paper_1806_01117_b200 import schedule as MS
from paper_1806_01117_b200.perfmodel import interval_length

SETTINGS = settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])


@SETTINGS
@given(n=st.integers(1, 90), s=st.integers(1, 12))
def test_revolve_schedule_and_cost_match_oracle(n, s):
    acts = MS.revolve_schedule(MS.ScheduleParams(n, s))
    ref = S.revolve(n, s)
    assert MS.actions_to_json(acts) == S.to_json(ref)
    assert MS.forward_cost(n, s) == S.forward_executions(ref)
    MS.validate_schedule(acts, MS.ScheduleParams(n, s))


@SETTINGS
@given(n=st.integers(2, 120), s=st.integers(1, 10), interval=st.integers(1, 130))
def test_multistage_plan_matches_oracle(n, s, interval):
    plan = MS.plan_multistage(n, s, interval)
    bounds, segs, fallback = S.plan_multistage(n, s, interval)
    assert plan.fallback == fallback
    assert tuple(plan.boundaries) == tuple(bounds)
    assert len(plan.segments) == len(segs)
    for got, (start, end, acts) in zip(plan.segments, segs):
        assert (got.start, got.end) == (start, end)
        assert MS.actions_to_json(got.actions) == S.to_json(acts)
    # the plan's count covers the segments (the executor adds the sweep's n)
    assert plan.forward_executions == sum(S.forward_executions(a) for _, _, a in segs)


@SETTINGS
@given(num=st.integers(1, 10**6), den=st.integers(1, 10**6), scale=st.sampled_from([1e-9, 1e-6, 1e-3, 1.0]))
def test_interval_length_is_exact_rational_ceiling(num, den, scale):
    t_t, t_a = num * scale, den * scale
    want = max(1, math.ceil(Fraction(t_t) / Fraction(t_a)))
    assert interval_length(t_t, t_a) == want == S.interval_length(t_t, t_a)
