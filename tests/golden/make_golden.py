"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The reference is imported read-only from /root/reference/pkg/src (no copy of
its sources lands in this repo); outputs are small JSON / npz fixtures that
travel with the repo, so the GPU box never needs /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("ACKPT_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from asyncckpt import lstm as RL  # noqa: E402
from asyncckpt import perfmodel as RP  # noqa: E402
from asyncckpt import runtime as RR  # noqa: E402
from asyncckpt import schedule as RS  # noqa: E402
from asyncckpt import storage as RST  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def schedule_golden() -> dict:
    costs = {}
    for n in range(1, 65):
        for s in range(0 if n == 1 else 1, 17):
            costs[f"{n},{s}"] = RS.forward_cost(n, s)
    for n, s in [(1000, 10), (1024, 100), (500, 2), (2000, 5), (300, 1), (4000, 100), (10000, 10)]:
        costs[f"{n},{s}"] = RS.forward_cost(n, s)
    shas = {}
    lengths = {}
    for n, s in [(10, 3), (16, 4), (64, 4), (128, 4), (1000, 10), (1000, 62), (500, 7), (257, 13), (300, 1), (64, 63)]:
        acts = RS.revolve_schedule(RS.ScheduleParams(n, s))
        shas[f"{n},{s}"] = sha(RS.actions_to_json(acts))
        lengths[f"{n},{s}"] = len(acts)
    json_small = {
        f"{n},{s}": RS.actions_to_json(RS.revolve_schedule(RS.ScheduleParams(n, s)))
        for n, s in [(10, 3), (9, 2), (1, 0), (4, 3), (17, 3)]
    }
    plans = {}
    for n, s, i in [(10, 2, 4), (12, 100, 4), (5, 2, 8), (64, 3, 8), (128, 4, 16), (48, 2, 4), (1000, 10, 60), (10000, 999, 60), (24, 2, 8)]:
        p = RS.plan_multistage(n, s, i)
        plans[f"{n},{s},{i}"] = {
            "boundaries": list(p.boundaries),
            "forward_executions": p.forward_executions,
            "fallback": p.fallback,
            "segments": [[seg.start, seg.end, sha(RS.actions_to_json(seg.actions))] for seg in p.segments[:3]]
            + ([[p.segments[-1].start, p.segments[-1].end, sha(RS.actions_to_json(p.segments[-1].actions))]] if len(p.segments) > 3 else []),
        }
    rng = np.random.default_rng(2024)
    intervals = [[0.035, 0.001, RP.interval_length(0.035, 0.001)]]
    for _ in range(300):
        ta = float(10 ** rng.uniform(-7, -2))
        tt = float(ta * rng.uniform(0.1, 200.0))
        intervals.append([tt, ta, RP.interval_length(tt, ta)])
    for k in range(1, 60):  # exact multiples stress the rounding
        ta = 1e-5 * (1 + rng.integers(0, 100))
        tt = ta * k
        intervals.append([tt, ta, RP.interval_length(tt, ta)])
    return {"costs": costs, "sha256": shas, "lengths": lengths, "json_small": json_small, "plans": plans, "interval_length": intervals}


def runtime_golden() -> tuple:
    """Counters + peaks + adjoints of the reference executor (fp64, B=1)."""
    configs = []
    arrays = {}
    cases = [
        # n, d, seed, strategy, slots, interval
        (8, 6, 3, "full", 0, None),
        (8, 6, 3, "revolve", 3, None),
        (8, 6, 3, "multistage", 3, 4),
        (24, 5, 9, "multistage", 2, 8),
        (5, 4, 3, "multistage", 2, 8),
        (12, 4, 1, "multistage", 3, 5),
        (32, 4, 3, "multistage", 7, 8),
        (64, 8, 31, "multistage", 4, 16),
        (64, 8, 31, "revolve", 4, None),
        (40, 8, 104, "revolve", 5, None),
        (40, 5, 119, "multistage", 4, 16),
        (100, 8, 0, "full", 0, None),
        (100, 32, 0, "full", 0, None),
        (50, 16, 4, "revolve", 3, None),
        (16, 4, 2, "multistage", 3, 4),
        (1, 4, 5, "full", 0, None),
        (2, 4, 5, "revolve", 1, None),
    ]
    backend = RST.SimulatedBackend(bandwidth=1e12, latency=0.0)
    try:
        for idx, (n, d, seed, kind, slots, interval) in enumerate(cases):
            cell = RL.random_cell(d=d, n=n, seed=seed)
            ops = RL.operator_pair(cell)
            s0 = RL.random_state(d, seed + 100)
            strat = {"full": RR.FullStorage(), "revolve": RR.Revolve(slots), "multistage": RR.Multistage(slots, interval)}[kind]
            adj, st = RR.execute(strat, ops, s0, backend)
            state = s0
            for k in range(n):
                state = RL.lstm_forward_step(cell, k, state)
            key = f"case{idx}"
            arrays[key + "_adjoint"] = np.frombuffer(adj, dtype="<f8")
            arrays[key + "_final"] = np.frombuffer(state, dtype="<f8")
            configs.append({
                "key": key, "n": n, "d": d, "seed": seed, "state_seed": seed + 100, "strategy": kind,
                "slots": slots, "interval": interval,
                "stats": {k: v for k, v in st.to_dict().items() if k not in ("wall_seconds", "stall_seconds")},
                "adjoint_sha256": hashlib.sha256(adj).hexdigest(),
                "loss": RL.loss(cell, state),
            })
    finally:
        backend.close()
    return configs, arrays


def step_golden() -> dict:
    """Single forward/backward steps of the reference cell."""
    arrays = {}
    for d, n, seed in [(4, 6, 5), (8, 10, 6), (6, 5, 7), (16, 4, 8), (5, 3, 9)]:
        cell = RL.random_cell(d=d, n=n, seed=seed)
        s = RL.random_state(d, seed + 1)
        adj = RL.loss_gradient_seed(cell, s)
        for k in range(n):
            s2 = RL.lstm_forward_step(cell, k, s)
            a2 = RL.lstm_backward_step(cell, k, s, adj)
            arrays[f"d{d}_s{seed}_k{k}_in"] = np.frombuffer(s, "<f8")
            arrays[f"d{d}_s{seed}_k{k}_fwd"] = np.frombuffer(s2, "<f8")
            arrays[f"d{d}_s{seed}_k{k}_adjin"] = np.frombuffer(adj, "<f8")
            arrays[f"d{d}_s{seed}_k{k}_bwd"] = np.frombuffer(a2, "<f8")
            s, adj = s2, RL.loss_gradient_seed(cell, s2)
        arrays[f"d{d}_s{seed}_cell_w_f"] = cell.w_f
        arrays[f"d{d}_s{seed}_cell_xs"] = cell.xs
    return arrays


def storage_golden() -> dict:
    rng = np.random.default_rng(7)
    crcs = [["", 0], ["313233343536373839", RST.crc32c(b"123456789")], ["00" * 32, RST.crc32c(b"\x00" * 32)]]
    for size in (1, 3, 7, 8, 9, 15, 16, 17, 63, 64, 65, 255, 1000, 4096):
        data = rng.bytes(size)
        crcs.append([data.hex(), RST.crc32c(data)])
    chained = RST.crc32c(b"world", RST.crc32c(b"hello "))
    blob = RST.encode_checkpoint(RST.CheckpointPayload(step=5, data=b"\xab" * 8))
    blob2 = RST.encode_checkpoint(RST.CheckpointPayload(step=123456789, data=bytes(range(40))))
    return {"crc32c": crcs, "chained_hello_world": chained, "encoded_step5": blob.hex(), "encoded_step123456789": blob2.hex()}


SIM_CASES = [
    # strategy, n, s, t_a, t_b, t_t, interval
    ("full", 6, 2, 1.0, 2.0, 3.5, None),
    ("revolve", 10, 3, 1.0, 2.0, 3.5, None),
    ("revolve", 33, 4, 0.001, 0.0025, 0.035, None),
    ("multistage", 24, 2, 1.0, 2.0, 7.0, None),      # calibrated I = 7, no stalls
    ("multistage", 24, 2, 1.0, 2.0, 7.0, 4),         # forced I < t_t / t_a: stalls
    ("multistage", 40, 6, 0.001, 0.0025, 0.035, None),
    ("multistage", 64, 3, 1.0, 1.5, 2.5, 8),
    ("multistage", 10, 3, 1.0, 2.0, 50.0, None),     # I >= n: fallback
]

CURVE_CASES = [(4, [8, 64], 1024), (10, [60], 10000), (1, [2, 3], 64)]


def reporting_golden() -> dict:
    """simulator timelines, model curves and CLI outputs of the reference
    (simulator.py, perfmodel.emit_curves / curves_to_csv, cli.py)."""
    from asyncckpt import cli as RC  # noqa: E402
    from asyncckpt import simulator as RSIM  # noqa: E402
    import contextlib
    import io

    sims = []
    for kind, n, s, ta, tb, tt, interval in SIM_CASES:
        strat = {"full": RR.FullStorage(), "revolve": RR.Revolve(s), "multistage": RR.Multistage(s, interval)}[kind]
        events, total = RSIM.simulate(strat, RP.PerfParams(n=n, s=s, t_a=ta, t_b=tb, t_t=tt))
        sims.append({"case": [kind, n, s, ta, tb, tt, interval],
                     "json": RSIM.timeline_to_json(strat, events, total),
                     "t_model": {"full": RP.t_infinity, "revolve": RP.t_revolve,
                                 "multistage": RP.t_async}[kind](RP.PerfParams(n=n, s=s, t_a=ta, t_b=tb, t_t=tt))})
    curves = []
    for s, intervals, n_max in CURVE_CASES:
        curves.append({"case": [s, intervals, n_max], "csv": RP.curves_to_csv(RP.emit_curves(s, intervals, n_max))})
    cli = []
    for argv in (["schedule", "--n", "10", "--s", "3"], ["schedule", "--n", "24", "--s", "2", "--interval", "8"],
                 ["schedule", "--n", "10", "--s", "2", "--interval", "40"],
                 ["model", "--s", "4", "--intervals", "8,64", "--n-max", "256"],
                 ["model", "--s", "3", "--n-max", "64", "--ta", "0.001", "--tt", "0.035"],
                 ["simulate", "--strategy", "multistage", "--n", "24", "--s", "2", "--ta", "1", "--tb", "2",
                  "--tt", "7"],
                 ["simulate", "--strategy", "revolve", "--n", "12", "--s", "3", "--ta", "1", "--tb", "2", "--tt", "1"],
                 ["schedule", "--n", "5", "--s", "0"]):
        out, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            rc = RC.main(argv)
        cli.append({"argv": argv, "rc": rc, "stdout": out.getvalue(), "stderr_prefix": err.getvalue()[:60]})
    return {"simulate": sims, "curves": curves, "cli": cli}


def main() -> None:
    sched = schedule_golden()
    with open(os.path.join(HERE, "schedule_golden.json"), "w") as fh:
        json.dump(sched, fh, indent=0, sort_keys=True)
    configs, arrays = runtime_golden()
    with open(os.path.join(HERE, "runtime_golden.json"), "w") as fh:
        json.dump(configs, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "runtime_golden.npz"), **arrays)
    np.savez_compressed(os.path.join(HERE, "step_golden.npz"), **step_golden())
    with open(os.path.join(HERE, "storage_golden.json"), "w") as fh:
        json.dump(storage_golden(), fh, indent=1)
    with open(os.path.join(HERE, "reporting_golden.json"), "w") as fh:
        json.dump(reporting_golden(), fh, indent=1)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
