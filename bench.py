#!/usr/bin/env python
"""Headline benchmark: reverse-pass overhead vs store-all and steps/s at
memory ratio 0.1, n = 10^4 (BASELINE.json), on BASELINE config 2:

  one 64 MiB fp32 state per GPU = LSTM cell d=8 over B = 2^20 independent
  sequences (layout (2, d, B)), n = 10^4 steps, Multistage(slots=999, I) with
  I = interval_length(t_t, t_a) from calibration, HBM slot pool + async
  pinned-host tier.

A "step" of this benchmark is one full forward/backward pass (execute) over
the n-step chain.  ``value`` = state-steps per second over all GPUs
(n x N_gpus / pass time, weak scaling: every rank owns its own 64 MiB shard
of the batch and runs the identical schedule; there is no collective in the
timed region).  Launch: ``python bench.py`` (1 GPU) or
``torchrun --nproc-per-node N bench.py --gpus N``.

``--impl reference`` times the CPU restatement of the reference algorithm
(oracle/, numpy, all host cores) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "reverse-pass steps/s at memory ratio 0.1, n=10^4 (overhead vs store-all reported beside)"
# interval of the reference arm's bounded sample when --interval is not given
# (the calibrated I of the ours arm at C2 is 79-85 since the 64-step fused
# calibration; the CPU cost per chain step does not depend on it)
REF_SAMPLE_INTERVAL = 80


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", "--n-steps", dest="n", type=int, default=10_000,
                   help="pass length (--n-steps under torchrun, whose parser claims --n)")
    p.add_argument("--config", choices=["c2", "c4"], default="c2",
                   help="BASELINE config: c2 = 64 MiB fp32 state per GPU (B=2^20), memory ratio 0.1; "
                        "c4 = 8 GiB over 8 GPUs, i.e. 1 GiB per GPU (B=2^24), memory ratio 0.05")
    p.add_argument("--d", type=int, default=8)
    p.add_argument("--batch", type=int, default=None, help="sequences per GPU (default: from --config)")
    p.add_argument("--memory-ratio", type=float, default=None, help="default: from --config")
    p.add_argument("--interval", type=int, default=0, help="0: calibrate")
    p.add_argument("--no-parity", action="store_true", help="skip the long-memory-cell parity leg")
    p.add_argument("--per-step", dest="fuse", action="store_false",
                   help="headline = the reference's per-step operator contract (default: temporally fused "
                        "launches; same schedule, counters and bits)")
    p.add_argument("--no-revolve", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--full-n", type=int, default=1000, help="n of the measured FullStorage run")
    p.add_argument("--no-other-mode", action="store_true")
    p.add_argument("--no-c1", action="store_true", help="skip the BASELINE config-1 block (reference workload)")
    p.add_argument("--family", choices=["ffma2", "tcgen05"], default="tcgen05",
                   help="kernel family of the fused d=8 launches (lstm.set_kernel_family)")
    args = p.parse_args(argv)
    if args.batch is None:
        args.batch = (1 << 24) if args.config == "c4" else (1 << 20)
    if args.memory_ratio is None:
        args.memory_ratio = 0.05 if args.config == "c4" else 0.1
    if args.config == "c4":
        # 1 GiB states: the per-step mode's shorter interval needs more pinned
        # boundary slots than the host RAM holds next to the headline tier
        args.no_other_mode = True
    return args


# ---------------------------------------------------------------------------
# clocks (B200_PROFILING.md "clocks DURING the timed region")

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "power_w_max": max(power) if power else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


# ---------------------------------------------------------------------------
# CPU port (oracle/) -- the reference algorithm restated in numpy

def _cpu_worker(args):
    d, n, seed, state_seed, b, lo, slots, interval = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    from oracle import lstm_oracle as L
    from oracle import runtime_oracle as R

    cell = L.random_cell(d, n, seed)
    s0 = L.random_states(d, state_seed, lo + b)[:, :, lo:]
    t0 = time.perf_counter()
    R.execute("multistage", cell, np.ascontiguousarray(s0), slots=slots, interval=interval, dtype=np.float32)
    return time.perf_counter() - t0


def cpu_port_steps(d, interval, slots, reps, cores, per_core=4096, pool=None, batch=1 << 20, shards=1):
    """Times the oracle executor (Multistage over n = 2 I steps, fp32) on
    cores x per_core sequences in parallel; returns (steps/s scaled to
    `shards` states of `batch` sequences, description, walls).  The CPU cost
    per chain step does not depend on I while I <= s + 1 (every interval is
    taped: 2 forwards + 1 backward per step, runtime.py:23-27)."""
    import multiprocessing as mp

    n = 2 * interval
    own = pool is None
    if own:
        pool = mp.get_context("spawn").Pool(cores, initializer=_pin_blas)
    try:
        walls = []
        for _ in range(reps):
            jobs = [(d, n, 0, 1, per_core, c * per_core, slots, interval) for c in range(cores)]
            t0 = time.perf_counter()
            pool.map(_cpu_worker, jobs)
            walls.append(time.perf_counter() - t0)
    finally:
        if own:
            pool.close()
            pool.join()
    seqs = cores * per_core
    best = min(walls)
    value = n / best * seqs / float(batch * shards)
    sample = (f"oracle/runtime_oracle.execute Multistage(slots={slots}, I={interval}) over n={n} steps, "
              f"{seqs} sequences (d={d}, fp32) split over {cores} processes; steps/s scaled to "
              f"{shards} x {batch}-sequence ({2 * d * batch * 4 >> 20} MiB) states; best of {reps}")
    return value, sample, walls


def _pin_blas():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["MKL_NUM_THREADS"] = "1"


def run_reference(args) -> None:
    """--impl reference: the CPU restatement on this host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    interval = args.interval or REF_SAMPLE_INTERVAL
    slots = max(1, int(args.memory_ratio * args.n) - 1)
    pool = mp.get_context("spawn").Pool(cores, initializer=_pin_blas)
    kw = dict(pool=pool, batch=args.batch, shards=max(1, args.gpus))
    try:
        cpu_port_steps(args.d, interval, slots, max(1, args.warmup), cores, **kw)
        value, sample, walls = cpu_port_steps(args.d, interval, slots, args.steps, cores, **kw)
    finally:
        pool.close()
        pool.join()
    n_sample = 2 * interval
    ms = statistics.mean(walls) * 1e3
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "steps/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": workload_config(args, slots),
        "interval": interval,
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": f"each step is one bounded sample ({n_sample} chain steps; value = best step); the "
                "reference package is pure Python/numpy (no native code), restated in oracle/ and run on "
                "all host cores; its cost per chain step is independent of the interval while I <= s+1",
    }
    print(json.dumps(line), flush=True)


def kernel_chain_times(dc, state0, chain=64):
    """Mean K1 / K2 launch durations at the bench shape: CUDA events around
    `chain` back-to-back launches through distinct buffers (like the pass)."""
    import torch

    bufs = [torch.empty_like(state0) for _ in range(6)]
    bufs[0].copy_(state0)
    adj = [torch.empty_like(state0) for _ in range(2)]
    out = []
    for kind in ("fwd", "bwd"):
        for rep in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(chain):
                if kind == "fwd":
                    bufs[(k + 1) % 6] = dc.forward(k % dc.n_steps, bufs[k % 6])
                else:
                    adj[(k + 1) % 2] = dc.backward(k % dc.n_steps, bufs[k % 6], adj[k % 2])
            e1.record()
            torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e-3 / chain)
    return out[0], out[1]


def fused_kernel_times(dc, state0, steps=64, reps=5):
    """Per-step durations of the fused launches (64 steps each): advance
    (state in registers), tape (every output stored), reverse (adjoint in
    registers, taped states read), plus their algorithmic bytes per launch."""
    import torch

    S = state0.numel() * state0.element_size()
    states = dc.forward_many(0, steps, state0)
    adj = dc.seed(states[-1])
    out = {}
    for kind in ("adv", "tape", "rev"):
        times = []
        for rep in range(reps + 1):  # first launch is a warm-up
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "adv":
                dc.advance(0, steps, state0)
            elif kind == "tape":
                dc.forward_many(0, steps, state0)
            else:
                dc.backward_many(0, [state0] + states[:-1], adj)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1) * 1e-3 / steps)
        out[kind] = sorted(times)[len(times) // 2]  # median
    out["adv_bytes"] = 2 * S
    out["tape_bytes"] = (steps + 1) * S
    out["rev_bytes"] = (steps + 2) * S
    return out


# reference CPU numbers for config 1 (unmodified
# reference, min of 5 runs, this build container's Xeon): d=32 row
C1_REFERENCE_MS = {"full": 116.2, "revolve": 244.2, "multistage": 282.4}


def run_c1(pkg, lstm) -> dict:
    """BASELINE config 1 exactly as the reference runs it (`asyncckpt bench
    --strategy X --n 1000 --d 32 --s 10 --backend file --runs 5`): B=1
    float64 byte-image states, CKPT file tier, min of 5 runs, through the
    same lstm.bench API (per-step contract).  A GPU launch per step: this
    workload is launch-latency bound, not bandwidth bound."""
    import shutil
    import tempfile

    out = {"workload": "n=1000, d=32, s=10, B=1 float64, file tier, min of 5 (asyncckpt bench)",
           "reference_cpu_ms": C1_REFERENCE_MS, "reference_cpu_source": "BASELINE.md section 2 (build container)"}
    scratch = tempfile.mkdtemp(prefix="ackpt_c1_")
    try:
        for name, strat in (("full", pkg.FullStorage()), ("revolve", pkg.Revolve(10)),
                            ("multistage", pkg.Multistage(10))):
            rep = lstm.bench(strat, n=1000, d=32, s=10, backend_config={"kind": "file", "dir": scratch}, seed=0,
                             runs=5)
            fused = lstm.bench(strat, n=1000, d=32, s=10, backend_config={"kind": "file", "dir": scratch}, seed=0,
                               runs=5, fuse=True)
            assert fused.gradient_checksum == rep.gradient_checksum  # same kernels, same bits
            graphed = lstm.bench(strat, n=1000, d=32, s=10, backend_config={"kind": "file", "dir": scratch}, seed=0,
                                 runs=5, graph=True)
            assert graphed.gradient_checksum == rep.gradient_checksum
            out[name] = {"wall_ms": rep.wall_seconds * 1e3, "forward_evals": rep.forward_evals,
                         "recompute_factor": rep.recompute_factor_measured, "stall_ms": rep.stall_seconds * 1e3,
                         "speedup_vs_reference_cpu": C1_REFERENCE_MS[name] / (rep.wall_seconds * 1e3),
                         "fused_wall_ms": fused.wall_seconds * 1e3,
                         "fused_speedup_vs_reference_cpu": C1_REFERENCE_MS[name] / (fused.wall_seconds * 1e3),
                         "graph_wall_ms": graphed.wall_seconds * 1e3,
                         "graph_speedup_vs_reference_cpu": C1_REFERENCE_MS[name] / (graphed.wall_seconds * 1e3)}
    finally:
        shutil.rmtree(scratch, ignore_errors=True)
    out["cpu_port_same_box"] = c1_cpu_port()
    return out


def c1_cpu_port() -> dict:
    """Config 1 on THIS box's host: the oracle's numpy restatement of the
    reference executor (oracle/runtime_oracle.py, one thread, fp64, B=1,
    d=32, n=1000), min of 3 -- the same-box counterpart of the reference's
    own `bench` numbers (measured in the build container: the reference
    cannot travel to the GPU box).  Multistage keeps its boundary states in
    memory (no CKPT files) with I = 11 (the reference's zero-latency
    `--interval 11` case)."""
    import numpy as np

    from oracle import lstm_oracle as L
    from oracle import runtime_oracle as R

    cell = L.random_cell(32, 1000, 0)
    s0 = L.random_states(32, 1, 1)
    res = {"cores": 1, "kind": "port", "sample": "oracle/runtime_oracle.execute, n=1000, d=32, B=1 float64, min of 3"}
    for name, kw in (("full", {}), ("revolve", {"slots": 10}),
                     ("multistage", {"slots": 10, "interval": 11})):
        best = min(R.execute(name, cell, np.ascontiguousarray(s0), **kw)[1]["wall_seconds"] for _ in range(3))
        res[name + "_ms"] = best * 1e3  # executor wall, plan excluded (runtime.py:359-363)
    return res


def workload_config(args, slots) -> dict:
    S = 2 * args.d * args.batch * 4
    if args.config == "c4":
        work = (f"BASELINE config 4: 8 GB state sharded by batch over 8 GPUs -> {S >> 20} MiB fp32 per GPU "
                f"(LSTM d={args.d} over {args.batch} sequences), n=10^4, memory ratio {args.memory_ratio}, "
                f"HBM snapshots + async pinned-host tier")
    else:
        work = (f"BASELINE config 2: 1 GPU, {S >> 20} MiB fp32 state, n=10^4, memory ratio {args.memory_ratio}, "
                f"HBM snapshots + async pinned-host tier (LSTM d={args.d} over {args.batch} sequences)")
    return {
        "workload": work,
        "n": args.n,
        "d": args.d,
        "batch_per_gpu": args.batch,
        "state_bytes_per_gpu": S,
        "strategy": f"Multistage(slots={slots}, interval=calibrated: interval_length(t_t, t_a))",
        "memory_ratio": args.memory_ratio,
        "execution": "temporally fused launches (Advance / TapeForward / Reverse runs)" if args.fuse
                     else "per-step operator launches (reference contract)",
        "kernel_family": args.family if args.fuse else "ffma2 (per-step kernels)",
        "l2": f"inputs larger than L2: every pass cycles >= I+2 distinct {S >> 20} MiB buffers (126 MB L2)",
        "parallelism": f"batch-sharded x{args.gpus}, identical schedule per rank, no collective in the timed region",
    }


# ---------------------------------------------------------------------------


def link_peak_gbs(S: int, reps: int = 5) -> dict:
    """Pinned host <-> HBM copy bandwidth on this box (best of `reps` plain
    copies of one state, CUDA events): the host-link denominator of the pass
    roofline (MEASURED_PEAKS.json has no link figure)."""
    import torch

    dev = torch.empty(S, dtype=torch.uint8, device="cuda")
    host = torch.empty(S, dtype=torch.uint8).pin_memory()
    out = {}
    for name, (dst, src) in (("d2h", (host, dev)), ("h2d", (dev, host))):
        best = float("inf")
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        out[name] = S / best / 1e9
    del dev, host
    return out


def fused_pass_bytes(n: int, boundaries: list, S: int, fuse: bool, stats) -> dict:
    """Algorithmic bytes of one Multistage pass, per phase.

    Fused launches (engine.cpp: one Advance launch per interval of the sweep;
    TapeForward in launches of <= 64 steps from the bottom, Reverse runs in
    launches of <= 64 steps from the top): advance 2S, tape of L steps
    (L+1)S, reverse run of L steps (L+2)S.  Per-step contract: forward 2S,
    backward 3S.  A store reads S from HBM and a fetch writes S; both move S
    over the host link."""
    ends = list(boundaries[1:]) + [n]
    lens = [e - b for b, e in zip(boundaries, ends)]

    def chunks(L):
        return [64] * (L // 64) + ([L % 64] if L % 64 else [])

    stores = len(boundaries)
    if fuse:
        sweep_hbm = sum(2 * S for _ in lens)
        tape = sum((c + 1) * S for L in lens for c in chunks(L))
        rev = sum((c + 2) * S for L in lens for c in chunks(L))
        bwd_hbm = tape + rev
    else:
        sweep_hbm = n * 2 * S
        bwd_hbm = (stats.forward_evals - n) * 2 * S + stats.backward_evals * 3 * S
    return {"sweep_hbm": sweep_hbm + stores * S, "sweep_link": stores * S,
            "backward_hbm": bwd_hbm + stats.prefetches_issued * S, "backward_link": stats.prefetches_issued * S}


def phase_times(pkg, strategy, ops, state0, backend, fuse) -> dict:
    """Sweep / backward split of one pass from the measured event timeline
    (two events per launch; the backward starts where the first fetch does,
    runtime.py:297-322)."""
    _, st = pkg.execute(strategy, ops, state0, backend, fuse=fuse, timeline=True)
    ev = st.timeline
    total = st.device["gpu_seconds"]
    fetch_starts = [e.start for e in ev if e.kind == "fetch"]
    split = min(fetch_starts) if fetch_starts else total
    return {"sweep_s": split, "backward_s": total - split, "total_s": total}


def parity_leg(pkg, lstm, args, strategy, backend, dev) -> dict:
    """The headline execution path (same strategy, interval, tier, kernel
    family and execution mode) on long_memory_cell -- the reference cell with
    forget-gate bias 5, whose fp32 adjoint does not underflow at n = 10^4
    (random_cell's is exactly 0 past n ~ 190) -- on the same initial states,
    against the float64 oracle executor on 64 sampled sequences.  Part of the
    CPU leg: the oracle is the checker here (SURVEY §8(c) protocol 2 at the
    headline n)."""
    import numpy as np
    import torch

    from oracle import lstm_oracle as L
    from oracle import runtime_oracle as R

    ops = lstm.operator_pair(lstm.long_memory_cell(args.d, args.n, 0), args.batch, "f32")
    s0 = lstm.random_states(args.d, 1, args.batch, "f32", device=dev)
    adj, st = pkg.execute(strategy, ops, s0, backend, fuse=args.fuse)
    torch.cuda.synchronize()
    rows = np.unique(np.linspace(0, args.batch - 1, 64).astype(np.int64))
    got = adj[:, :, rows].double().cpu().numpy()
    full_norm = adj.double().norm().item()
    t0 = time.perf_counter()
    ref, _ = R.execute("full", L.long_memory_cell(args.d, args.n, 0), s0[:, :, rows].double().cpu().numpy())
    oracle_s = time.perf_counter() - t0
    err = L.rel_l2(got, ref)
    per = [L.rel_l2(got[:, :, i], ref[:, :, i]) for i in range(len(rows))]
    del ops, adj
    torch.cuda.empty_cache()
    return {"cell": f"long_memory_cell(d={args.d}, n={args.n}, seed=0, forget_bias=5)",
            "path": "identical to the headline: same strategy / interval / tier / execution mode / kernel family",
            "checker": "oracle/runtime_oracle.execute, float64, 64 sampled sequences",
            "rows": int(len(rows)), "rel_l2": err, "tol": 2e-4, "ok": bool(err <= 2e-4 and full_norm > 0),
            "median_rel_l2_per_sequence": float(np.median(per)), "max_rel_l2_per_sequence": float(np.max(per)),
            "adjoint_norm_sampled": float(np.linalg.norm(ref)), "adjoint_norm_full_batch": full_norm,
            "forward_evals": st.forward_evals, "oracle_seconds": oracle_s}


def inline_cpu_baseline(args, interval: int) -> dict:
    """The reference arm's own measurement (`bench.py --impl reference`, same
    config, warm-up + best of 5) in a clean subprocess, so the in-line
    cpu_baseline and the driver's reference arm are one method."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "5", "--warmup", "1",
           "--config", args.config, "--d", str(args.d), "--batch", str(args.batch), "--n-steps", str(args.n),
           "--memory-ratio", str(args.memory_ratio), "--interval", str(interval), "--gpus", "1"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    cb = dict(line["cpu_baseline"])
    cb["how"] = "bench.py --impl reference --steps 5 --warmup 1 in a subprocess (the reference arm's method)"
    return cb


def main(argv=None) -> None:
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # ACKPT_BENCH_DIST=1: run the process-group plumbing (NCCL interval
    # agreement, barriers, max-over-ranks timing) even with a single rank
    dist_on = world > 1 or os.environ.get("ACKPT_BENCH_DIST") == "1"
    if dist_on:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1806_01117_b200 as pkg
    import paper_1806_01117_b200.distributed as D
    import paper_1806_01117_b200.lstm as lstm

    numa = D.bind_local_numa(local)  # pinned slabs and I/O threads next to this GPU (no-op on one node)
    lstm.set_kernel_family(args.family)
    dev = torch.device("cuda", local)
    cell = lstm.random_cell(args.d, args.n, 0)
    ops = lstm.operator_pair(cell, args.batch, "f32")
    S = ops.state_size
    # each rank owns batch shard `rank` of the global batch (seeded per shard)
    state0 = lstm.random_states(args.d, 1 + rank, args.batch, "f32", device=dev)
    slots = max(1, int(args.memory_ratio * args.n) - 1)
    link = link_peak_gbs(S)
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", world))

    # --- calibration (outside the timed window, runtime.py:359-361) ---
    with pkg.PinnedHostBackend(slot_bytes=S) as cal_backend:
        t_a, t_b, t_t = pkg.calibrate(ops, cal_backend, 5, state0, fuse=args.fuse)
    # identical schedule on every rank: the largest calibrated interval
    interval = D.agree_interval(args.interval or pkg.interval_length(t_t, t_a))
    n_keys = -(-args.n // interval)
    # pinned slab for every boundary if the host RAM allows, else the cascade
    backend = D.make_rank_backend(pkg, S, n_keys, local_ranks=local_ranks)
    if not isinstance(backend, pkg.PinnedHostBackend):  # stores are paced by the spill stage: re-calibrate
        t_a, t_b, t_t = pkg.calibrate(ops, backend, 5, state0, fuse=args.fuse)
        interval = D.agree_interval(args.interval or pkg.interval_length(t_t, t_a))
    strategy = pkg.Multistage(slots, interval)
    tier_desc = {"kind": type(backend).__name__, "boundary_keys": -(-args.n // interval),
                 "pinned_key_budget": D.pinned_key_budget(S, local_ranks), "local_ranks": local_ranks,
                 "numa": numa}

    def run_once():
        return pkg.execute(strategy, ops, state0, backend, fuse=args.fuse)

    for _ in range(args.warmup):
        adj, st = run_once()
    torch.cuda.synchronize()

    # --- timed region: K passes, inputs resident in HBM, nothing else on the GPU ---
    clocks = ClockSampler(local)
    clocks.start()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    stats = []
    for _ in range(args.steps):
        adj, st = run_once()
        stats.append(st)
    e1.record(stream)
    torch.cuda.synchronize()
    host_elapsed = time.perf_counter() - h0
    elapsed = D.max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    clock = clocks.stop()
    ms_per_step = elapsed / args.steps * 1e3
    value = world * args.n * args.steps / elapsed
    last = stats[-1]
    launches = sum(s.device["kernel_launches"] for s in stats)

    # --- per-kernel durations: CUDA-event-timed chains of the same launches
    # (event pairs inside the pass would perturb it: each completion flushes
    # the dirty L2 lines the next step reuses) ---
    t_fwd, t_bwd = kernel_chain_times(ops.native, state0, chain=64)
    # 64-step launches as in the pass; fewer at config 4 (1 GiB states) so
    # the two taped chains fit next to the engine's HBM pool
    fk_steps = int(min(64, max(8, 20e9 // S)))
    fk = fused_kernel_times(ops.native, state0, steps=fk_steps)
    phases = phase_times(pkg, strategy, ops, state0, backend, args.fuse)

    # --- store-all (FullStorage) measured at the largest n kept affordable in
    # HBM next to the other pools; T_inf = n x its per-step time, in both the
    # per-step and the fused execution mode ---
    n_full = min(args.n, args.full_n, max(8, int(40e9 // S)))
    full_ops = lstm.operator_pair(lstm.random_cell(args.d, n_full, 0), args.batch, "f32")
    t_store_all = {}
    for mode in (False, True):
        pkg.execute(pkg.FullStorage(), full_ops, state0, fuse=mode)
        _, fst = pkg.execute(pkg.FullStorage(), full_ops, state0, fuse=mode)
        t_store_all["fused" if mode else "per_step"] = fst.wall_seconds / n_full
    t_inf = args.n * t_store_all["fused" if args.fuse else "per_step"]
    t_inf_per_step = args.n * t_store_all["per_step"]
    t_inf_kernels = args.n * (t_fwd + t_bwd)
    overhead = (ms_per_step * 1e-3) / t_inf
    del full_ops
    torch.cuda.empty_cache()

    # --- roofline: dominant kernel of the headline pass + whole pass ---
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    if args.fuse:
        # per step of the pass: n sweep steps (fused advance), n taped steps, n reverse steps
        shares = {"lstm_rev_fused (K2f)": (args.n * fk["rev"], fk["rev_bytes"], fk["rev"] * fk_steps),
                  "lstm_tape_fused (K1t)": (args.n * fk["tape"], fk["tape_bytes"], fk["tape"] * fk_steps),
                  "lstm_adv_fused (K1f)": (args.n * fk["adv"], fk["adv_bytes"], fk["adv"] * fk_steps)}
    else:
        shares = {"lstm_fwd (K1)": (last.forward_evals * t_fwd, 2 * S, t_fwd),
                  "lstm_bwd (K2)": (last.backward_evals * t_bwd, 3 * S, t_bwd)}
    dominant = max(shares, key=lambda k: shares[k][0])
    _, bytes_dom, t_dom = shares[dominant]
    achieved = bytes_dom / t_dom / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    pipes = None
    base = dominant.split()[0]
    kfam = "tcgen05" if (args.fuse and args.family == "tcgen05") else "ffma2"
    if os.path.exists(tfile):
        with open(tfile) as fh:
            tj = json.load(fh)
        traffic = tj.get(f"{base}@{kfam}", tj.get(base))
        if S != 64 << 20 or (args.fuse and fk_steps != 64):
            traffic = None  # the ncu captures are of the config-2 launch shape
        pipes = tj.get("pipes", {}).get(f"{base}@{kfam}", tj.get("pipes", {}).get(base))
    # issue-bound roofline of the dominant fused launch: its ncu instruction
    # count (scaled to this batch and launch length) at one warp instruction
    # per SMSP per cycle at the maximum SM clock, against the measured time
    issue = None
    if args.fuse and pipes and pipes.get("inst_per_launch"):
        inst = pipes["inst_per_launch"] * (args.batch / pipes["inst_batch"]) * (fk_steps / pipes["inst_steps"])
        smsps = 4 * torch.cuda.get_device_properties(0).multi_processor_count
        clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        floor = inst / (smsps * clk)
        issue = {"instructions_per_launch": inst, "floor_us": floor * 1e6, "measured_us": t_dom * 1e6,
                 "frac": floor / t_dom,
                 "how": "ncu smsp__inst_executed.sum of the launch (profiles/ncu_traffic.json pipes) / "
                        "(4 x SMs x sm_max_mhz): the time at 100 % issue; frac = floor / measured"}
    link_gbs = S / t_t / 1e9
    # phase-wise pass roofline: sum over phases of max(HBM, link)
    pb = fused_pass_bytes(args.n, pkg.plan_multistage(args.n, slots, interval).boundaries, S, args.fuse, last)
    link_d2h, link_h2d = link["d2h"] * 1e9, link["h2d"] * 1e9
    sweep_rf = max(pb["sweep_hbm"] / (hbm_peak * 1e9), pb["sweep_link"] / link_d2h)
    bwd_rf = max(pb["backward_hbm"] / (hbm_peak * 1e9), pb["backward_link"] / link_h2d)
    pass_roofline = sweep_rf + bwd_rf

    # --- the other execution mode (same schedule, same counters) ---
    other = None
    if not args.no_other_mode:
        mode = not args.fuse
        ot_a, _, ot_t = pkg.calibrate(ops, backend, 5, state0, fuse=mode)
        o_interval = D.agree_interval(args.interval or pkg.interval_length(ot_t, ot_a))
        o_strategy = pkg.Multistage(slots, o_interval)
        for _ in range(2):
            o_adj, _ = pkg.execute(o_strategy, ops, state0, backend, fuse=mode)
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            o_adj, ost = pkg.execute(o_strategy, ops, state0, backend, fuse=mode)
        g1.record()
        torch.cuda.synchronize()
        o_el = g0.elapsed_time(g1) * 1e-3 / args.steps
        o_inf = args.n * t_store_all["fused" if mode else "per_step"]
        other = {"mode": "fused" if mode else "per_step", "interval": o_interval,
                 "ms_per_step": o_el * 1e3, "steps_per_s": world * args.n / o_el,
                 "overhead_vs_store_all": o_el / o_inf, "overhead_vs_per_step_store_all": o_el / t_inf_per_step,
                 "calibrated_t_a_us": ot_a * 1e6, "forward_evals": ost.forward_evals,
                 "stall_seconds": ost.stall_seconds, "kernel_launches": ost.device["kernel_launches"],
                 "note": "the reference cell's fp32 adjoint is exactly 0 at n=10^4 (both modes); parity of "
                         "the headline path is checked on the long-memory cell (key parity)"}

    # --- BASELINE config 1: the reference's own workload, same API, on the GPU ---
    c1 = None
    if not args.no_c1 and rank == 0 and world == 1:
        c1 = run_c1(pkg, lstm)

    # --- Revolve(s) at the same memory ratio, for comparison (when s+1 states fit in HBM) ---
    revolve = None
    if not args.no_revolve:
        free_hbm = torch.cuda.mem_get_info()[0]
        if (slots + 2) * S > 0.9 * free_hbm:
            revolve = {"skipped": f"Revolve({slots}) needs {(slots + 2) * S / 2**30:.0f} GiB of HBM "
                                  f"(free {free_hbm / 2**30:.0f} GiB)"}
        else:
            try:
                pkg.execute(pkg.Revolve(slots), ops, state0, fuse=args.fuse)
                _, rst = pkg.execute(pkg.Revolve(slots), ops, state0, fuse=args.fuse)
                revolve = {
                    "slots": slots,
                    "wall_seconds": rst.wall_seconds,
                    "steps_per_s": args.n / rst.wall_seconds,
                    "overhead_vs_store_all": rst.wall_seconds / t_inf,
                    "forward_evals": rst.forward_evals,
                    "recompute_factor": rst.forward_evals / args.n,
                    "peak_l1_bytes": rst.peak_l1_bytes,
                }
            except pkg.CheckpointError as exc:  # e.g. HBM too small for s+1 states
                revolve = {"error": str(exc)}
            pkg.release(ops)  # the Revolve pool (s+1 states) back before the other legs
            torch.cuda.empty_cache()

    # --- end to end through the public API with host buffers ---
    e2e = None
    if not args.no_e2e:
        host_in = state0.cpu().pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            adj_dev, _ = pkg.execute(strategy, ops, host_in, backend, fuse=args.fuse)
            host_out.copy_(adj_dev)
        g1.record()
        torch.cuda.synchronize()
        e2e_elapsed = D.max_over_ranks(g0.elapsed_time(g1) * 1e-3)
        e2e = {"value": world * args.n * args.steps / e2e_elapsed, "unit": "steps/s",
               "h2d_bytes_per_step": S, "d2h_bytes_per_step": S,
               "ms_per_step": e2e_elapsed / args.steps * 1e3}

    # --- CPU leg (rank 0, N=1 only): the reference arm's measurement in a
    # clean subprocess, and the parity check of the headline path ---
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = inline_cpu_baseline(args, interval)
    if rank == 0 and not args.no_parity:
        pkg.release(ops)
        torch.cuda.empty_cache()
        parity = parity_leg(pkg, lstm, args, strategy, backend, dev)

    if dist_on:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "steps/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(args, slots),
            "interval": interval,
            "impl": "ours",
            "overhead_vs_store_all": overhead,
            "t_inf_seconds": t_inf,
            "t_inf_source": f"measured FullStorage pass at n={n_full} (same execution mode) x n/{n_full}",
            "t_inf_from_kernel_chains_seconds": t_inf_kernels,
            "t_a_us": t_fwd * 1e6,
            "t_b_us": t_bwd * 1e6,
            "calibrated": {"t_a_us": t_a * 1e6, "t_b_us": t_b * 1e6, "t_t_ms": t_t * 1e3, "interval": interval},
            "link_gbs": link_gbs,
            "link_peak_gbs": link,
            "tier": tier_desc,
            "recompute_factor_measured": last.forward_evals / args.n,
            "forward_evals": last.forward_evals,
            "backward_evals": last.backward_evals,
            "stores_issued": last.stores_issued,
            "prefetches_issued": last.prefetches_issued,
            "stall_seconds": last.stall_seconds,
            "peak_l1_bytes": last.peak_l1_bytes,
            "host_wall_seconds_per_pass": host_elapsed / args.steps,
            "pass_roofline": {
                "seconds": pass_roofline, "frac": pass_roofline / (ms_per_step * 1e-3),
                "formula": "sum over phases of max(HBM bytes / hbm_gbs, link bytes / measured link GB/s)",
                "sweep": {"hbm_bytes": pb["sweep_hbm"], "link_bytes": pb["sweep_link"], "roofline_s": sweep_rf,
                          "measured_s": phases["sweep_s"],
                          "bound": "link" if pb["sweep_link"] / link_d2h > pb["sweep_hbm"] / (hbm_peak * 1e9)
                          else "hbm"},
                "backward": {"hbm_bytes": pb["backward_hbm"], "link_bytes": pb["backward_link"],
                             "roofline_s": bwd_rf, "measured_s": phases["backward_s"],
                             "bound": "link" if pb["backward_link"] / link_h2d > pb["backward_hbm"] / (hbm_peak * 1e9)
                             else "hbm"},
                "phase_split_source": "one extra pass with the measured event timeline (2 events per launch)",
            },
            "roofline": {"kernel": f"{dominant} [{kfam}]", "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": bytes_dom, "avg_launch_us": t_dom * 1e6,
                         "timing": "CUDA events around back-to-back launches of the same kernel",
                         "peak_source": peak_src,
                         "binding_pipes": pipes,
                         "issue_bound": issue,
                         "note": ("the fused launches are compute bound (FMA / MUFU issue, see binding_pipes "
                                  "from ncu); frac is their HBM fraction, not a pipe fraction")
                         if args.fuse else "per-step kernels: HBM bound"},
            "parity": parity,
            "other_mode": other,
            "c1_reference_workload": c1,
            "fused_kernels_us_per_step": {k: fk[k] * 1e6 for k in ("adv", "tape", "rev")},
            "store_all_us_per_step": {k: v * 1e6 for k, v in t_store_all.items()},
            "overhead_vs_per_step_store_all": (ms_per_step * 1e-3) / t_inf_per_step,
            "revolve": revolve,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clock,
        }
        print(json.dumps(line), flush=True)
    backend.close()
    if dist_on:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
