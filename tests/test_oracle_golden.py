"""Pins the CPU oracle (oracle/) to golden vectors produced by the
unmodified reference (tests/golden/make_golden.py) and to the reference
tests' own known answers.  CPU only."""

import hashlib

import numpy as np

from oracle import lstm_oracle as L
from oracle import runtime_oracle as R
from oracle import schedule_oracle as S


def test_oracle_costs(sched_golden):
    table = S.cost_table(64, 16)
    for key, cost in sched_golden["costs"].items():
        n, s = map(int, key.split(","))
        if n <= 64 and s <= 16:
            assert table[s][n] == cost, key
    # the reference tests' frozen values
    assert table[3][10] == 19 and table[2][5] == 8 and table[2][4] == 6
    assert table[3][8] == 14 and table[2][8] == 18 and table[4][16] == 33 and table[4][64] == 229


def test_oracle_schedules(sched_golden):
    for key, text in sched_golden["json_small"].items():
        n, s = map(int, key.split(","))
        assert S.to_json(S.revolve(n, s)) == text, key
    for key, digest in sched_golden["sha256"].items():
        n, s = map(int, key.split(","))
        if n <= 300:
            acts = S.revolve(n, s)
            assert hashlib.sha256(S.to_json(acts).encode()).hexdigest() == digest, key
            assert len(acts) == sched_golden["lengths"][key]


def test_oracle_plans(sched_golden):
    for key, plan in sched_golden["plans"].items():
        n, s, i = map(int, key.split(","))
        if n > 200:
            continue
        bounds, segs, fallback = S.plan_multistage(n, s, i)
        assert list(bounds) == plan["boundaries"]
        assert fallback == plan["fallback"]
        assert sum(S.forward_executions(a) for _, _, a in segs) == plan["forward_executions"]


def test_oracle_interval(sched_golden):
    for tt, ta, want in sched_golden["interval_length"]:
        assert S.interval_length(tt, ta) == want


def test_oracle_steps_match_reference(step_golden):
    for d, n, seed in [(4, 6, 5), (8, 10, 6), (6, 5, 7), (16, 4, 8), (5, 3, 9)]:
        cell = L.random_cell(d, n, seed)
        np.testing.assert_array_equal(cell.w[0], step_golden[f"d{d}_s{seed}_cell_w_f"])
        np.testing.assert_array_equal(cell.xs, step_golden[f"d{d}_s{seed}_cell_xs"])
        for k in range(n):
            x = step_golden[f"d{d}_s{seed}_k{k}_in"].reshape(2, d, 1)
            a = step_golden[f"d{d}_s{seed}_k{k}_adjin"].reshape(2, d, 1)
            fwd = L.forward_step(cell, k, x)
            bwd = L.backward_step(cell, k, x, a)
            assert L.rel_l2(fwd, step_golden[f"d{d}_s{seed}_k{k}_fwd"]) < 1e-14
            assert L.rel_l2(bwd, step_golden[f"d{d}_s{seed}_k{k}_bwd"]) < 1e-13


def test_oracle_random_state_matches_reference_draws(step_golden):
    # random_states(d, seed, 1) is the reference's random_state(d, seed)
    s = L.random_states(8, 7, 1)
    np.testing.assert_array_equal(s.ravel(), step_golden["d8_s6_k0_in"])


def test_oracle_executor_matches_reference(runtime_golden):
    cfgs, arrays = runtime_golden
    for cfg in cfgs:
        cell = L.random_cell(cfg["d"], cfg["n"], cfg["seed"])
        s0 = L.random_states(cfg["d"], cfg["state_seed"], 1)
        adj, st = R.execute(cfg["strategy"], cell, s0, slots=cfg["slots"], interval=cfg["interval"])
        for k, v in cfg["stats"].items():
            assert st[k] == v, (cfg["key"], k, st[k], v)
        assert L.rel_l2(adj, arrays[cfg["key"] + "_adjoint"]) < 1e-12, cfg["key"]
