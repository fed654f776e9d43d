"""The C-ABI library: loads on a CPU-only host, exports every symbol the
header declares, and its host-side functions (scheduler, exact interval,
CRC32C) are bit-exact with the reference's golden vectors.  No GPU calls."""

import ctypes as C
import hashlib
import os
import re

import pytest

from paper_1806_01117_b200 import _native as N
from paper_1806_01117_b200 import errors as E
from paper_1806_01117_b200 import schedule as MS
from paper_1806_01117_b200.perfmodel import interval_length
from paper_1806_01117_b200.storage import crc32c

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ackpt.h")).read()
    return sorted(set(re.findall(r"ACKPT_API\s+[\w\s\*]+?\b(ackpt_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 40
    for name in syms:
        assert hasattr(N.lib, name), name
    assert set(syms) == set(N.EXPORTED), set(syms) ^ set(N.EXPORTED)


def test_library_is_in_tree_and_versioned():
    assert os.path.dirname(N.LIB_PATH) == os.path.join(ROOT, "paper_1806_01117_b200")
    assert b"sm_100a" in N.lib.ackpt_version()


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(E.InfeasibleSchedule):
        N.check(N.INFEASIBLE_SCHEDULE)
    with pytest.raises(E.MissingKey):
        N.check(N.MISSING_KEY)
    with pytest.raises(ValueError):
        N.check(N.VALUE_ERROR)
    out = C.c_int64()
    assert N.lib.ackpt_forward_cost(10, 0, C.byref(out)) == N.INFEASIBLE_SCHEDULE
    assert "zero checkpoint slots" in N.last_error()
    assert N.lib.ackpt_forward_cost(0, 3, C.byref(out)) == N.VALUE_ERROR


def test_native_costs_match_reference(sched_golden):
    for key, cost in sched_golden["costs"].items():
        n, s = map(int, key.split(","))
        assert MS.forward_cost(n, s) == cost, key


def test_native_schedules_bit_exact(sched_golden):
    for key, text in sched_golden["json_small"].items():
        n, s = map(int, key.split(","))
        assert MS.actions_to_json(MS.revolve_schedule(MS.ScheduleParams(n, s))) == text
    for key, digest in sched_golden["sha256"].items():
        n, s = map(int, key.split(","))
        acts = MS.revolve_schedule(MS.ScheduleParams(n, s))
        assert len(acts) == sched_golden["lengths"][key], key
        assert hashlib.sha256(MS.actions_to_json(acts).encode()).hexdigest() == digest, key


def test_native_plans_match_reference(sched_golden):
    for key, want in sched_golden["plans"].items():
        n, s, i = map(int, key.split(","))
        plan = MS.plan_multistage(n, s, i)
        assert list(plan.boundaries) == want["boundaries"], key
        assert plan.fallback == want["fallback"]
        assert plan.forward_executions == want["forward_executions"], key
        segs = plan.segments
        picked = list(segs[:3]) + ([segs[-1]] if len(segs) > 3 else [])
        for seg, (start, end, digest) in zip(picked, want["segments"]):
            assert (seg.start, seg.end) == (start, end)
            assert hashlib.sha256(MS.actions_to_json(seg.actions).encode()).hexdigest() == digest


def test_survey_scale_costs():
    # SURVEY §8(c) survey-computed values (cross-checked against the reference
    # goldens above): ratio-0.1 Revolve at n=10^4 and the s=62 sweep.
    assert MS.forward_cost(10**4, 999) == 19010
    assert MS.forward_cost(10**4, 10) == 60960
    assert [MS.forward_cost(n, 62) for n in (1000, 2000, 5000, 10**4)] == [1955, 3994, 13037, 28139]


def test_native_interval_length_exact(sched_golden):
    for tt, ta, want in sched_golden["interval_length"]:
        assert interval_length(tt, ta) == want, (tt, ta)
    assert interval_length(0.035, 0.001) == 36  # float ceil would say 35
    assert interval_length(1e-300, 1e300) == 1
    with pytest.raises(ValueError):
        interval_length(0.0, 1.0)


def test_native_crc32c(storage_golden):
    for hexdata, want in storage_golden["crc32c"]:
        assert crc32c(bytes.fromhex(hexdata)) == want
    assert crc32c(b"world", crc32c(b"hello ")) == storage_golden["chained_hello_world"]


def test_best_split_is_smallest_argmin():
    # ties exist: the native split must be the FIRST argmin
    from oracle import schedule_oracle as S

    table = S.cost_table(200, 12)
    for length in range(14, 200, 7):
        for slots in (2, 3, 5, 12):
            if length > slots + 1:
                assert MS.best_split(length, slots) == S.best_split(length, slots, table)


def test_chain_bookkeeping_selftest():
    """Launch-chain bookkeeping (csrc/lstm_cell.h chain_step), host only: which
    launch may chain to which -- same cell and stream, adjacent, equal tile
    counts, marked; per-stream flag slots with eviction; stream handle 0."""
    rc = N.lib.ackpt_chain_selftest()
    assert rc == 0, N.last_error()
