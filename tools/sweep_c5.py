"""BASELINE config 5: compute/transfer ratio sweep on one GPU.

Two axes:
  * state size S = 16 MiB .. 4 GiB (B = S / (2 d 4), d = 8, fp32) over the
    pinned-host tier, the file (CKPT, page cache) tier and the three-stage
    cascade (pinned DRAM for --dram-slots boundaries, the rest spilled to CKPT
    files with O_DIRECT and read back ahead of the backward);
  * at S = 64 MiB, the host link throttled to 56 / 16 / 4 / 1 GB/s
    (SimulatedBackend), which sweeps t_t / t_a at a fixed step cost.
For each point: calibrated t_a, t_b, t_t, the interval I = ceil(t_t / t_a),
Multistage(slots, I) wall time over n = max(n0, 8 I) steps (steady state:
the start-up store and drain fetch amortised over >= 8 intervals), stall,
measured recompute factor against the paper's model (1 + R(I, s) per step, runtime.py:23-27 / perfmodel.t_async),
overhead vs the measured store-all per-step time, and the link bytes / s the
run achieved.  Level-1 budget: slots = min(0.1 n - 1, 96 GiB / S - 2).
One JSON line per point, then a summary line.

  python tools/sweep_c5.py [--sizes-mib 16,64,256,1024,4096] [--tiers pinned,file]
                           [--sim-gbs 16,4,1] [--n 2000] [--file-dir /tmp/ackpt_c5] [--dram-slots 8]
"""

import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

GiB = 1 << 30
MiB = 1 << 20


def store_all_per_step(d, B, S, fuse):
    """Measured FullStorage per-step time at the largest n <= 200 that keeps
    the stored states under 40 GiB of HBM."""
    n_full = max(4, min(200, int(40 * GiB // S) - 2))
    ops = lstm.operator_pair(lstm.random_cell(d, n_full, 0), B, "f32")
    s0 = lstm.random_states(d, 1, B, "f32")
    pkg.execute(pkg.FullStorage(), ops, s0, fuse=fuse)
    _, st = pkg.execute(pkg.FullStorage(), ops, s0, fuse=fuse)
    del ops, s0
    torch.cuda.empty_cache()
    return st.wall_seconds / n_full, n_full


def point(d, B, S, n, tier, backend, t_step, fuse, extra, n_max):
    s0 = lstm.random_states(d, 1, B, "f32")
    ops = lstm.operator_pair(lstm.random_cell(d, n, 0), B, "f32")
    t_a, t_b, t_t = pkg.calibrate(ops, backend, 5, s0, fuse=fuse)
    interval = pkg.interval_length(t_t, t_a)
    # steady state: at least 8 intervals per pass (start-up store / drain fetch amortised)
    n_run = max(n, min(n_max, -(-8 * interval // 1000) * 1000))
    if n_run != n:
        del ops
        n = n_run
        ops = lstm.operator_pair(lstm.random_cell(d, n, 0), B, "f32")
    slots = max(1, min(int(0.1 * n) - 1, int(96 * GiB // S) - 2))
    strat = pkg.Multistage(slots, interval=interval)
    pkg.execute(strat, ops, s0, backend, fuse=fuse)  # warm-up (allocations, table)
    t0 = time.perf_counter()
    adj, st = pkg.execute(strat, ops, s0, backend, fuse=fuse)
    host_wall = time.perf_counter() - t0
    fallback = interval >= n
    inner = 0 if fallback else None
    if not fallback:
        full, rem = divmod(n, interval)
        inner = full * pkg.forward_cost(interval, slots) + (pkg.forward_cost(rem, slots) if rem else 0)
    model_r = (st.forward_evals / n) if fallback else (n + inner) / n
    model = pkg.perfmodel.overhead_model(n, slots, interval, t_a, t_b)
    moved = (st.stores_issued + st.prefetches_issued) * S
    row = {
        "state_mib": S / MiB,
        "batch": B,
        "tier": tier,
        **extra,
        "n": n,
        "slots": slots,
        "t_a_us": t_a * 1e6,
        "t_b_us": t_b * 1e6,
        "t_t_ms": t_t * 1e3,
        "ratio_t_t_over_t_a": t_t / t_a,
        "interval": interval,
        "fallback_revolve": fallback,
        "wall_s": st.wall_seconds,
        "host_wall_s": host_wall,
        "steps_per_s": n / st.wall_seconds,
        "stall_s": st.stall_seconds,
        "stall_frac": st.stall_seconds / st.wall_seconds,
        "stores": st.stores_issued,
        "prefetches": st.prefetches_issued,
        "link_gbs_over_pass": moved / st.wall_seconds / 1e9,
        "recompute_factor": st.forward_evals / n,
        "model_recompute_factor": model_r,
        "store_all_us_per_step": t_step * 1e6,
        "overhead_vs_store_all": st.wall_seconds / (n * t_step),
        "model_overhead_calibrated": (model["multistage_overhead"] if not fallback else model["revolve_overhead"]),
        "peak_l1_states": st.peak_l1_bytes / S,
        "adjoint_finite": bool(torch.isfinite(adj).all()),
    }
    if hasattr(backend, "stats"):  # three-stage tier: what the file stage did in the timed pass and its warm-up
        cs = backend.stats()
        row["cascade"] = {**cs,
                          "spill_gbs": cs["spill_bytes"] / cs["spill_seconds"] / 1e9 if cs["spill_seconds"] else None,
                          "read_gbs": cs["read_bytes"] / cs["read_seconds"] / 1e9 if cs["read_seconds"] else None,
                          "note": "O_DIRECT file I/O (no page cache); counters cover the warm-up pass too"}
    del ops, s0, adj
    torch.cuda.empty_cache()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mib", default="16,64,256,1024,4096")
    ap.add_argument("--tiers", default="pinned,file")
    ap.add_argument("--file-sizes-mib", default="16,64,256,1024", help="sizes run over the file tier")
    ap.add_argument("--sim-gbs", default="16,4,1", help="throttled link GB/s at 64 MiB")
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--n-large", type=int, default=1000, help="n for states >= 1 GiB")
    ap.add_argument("--n-max", type=int, default=20000, help="cap of n when scaling n to 8 intervals")
    ap.add_argument("--file-dir", default="/tmp/ackpt_c5")
    ap.add_argument("--dram-slots", type=int, default=8, help="DRAM boundaries of the cascade tier")
    ap.add_argument("--per-step", dest="fuse", action="store_false")
    ap.add_argument("--d", type=int, default=8)
    args = ap.parse_args()
    d = args.d
    rows = []
    sizes = [int(x) for x in args.sizes_mib.split(",") if x]
    file_sizes = {int(x) for x in args.file_sizes_mib.split(",") if x}
    tiers = [x for x in args.tiers.split(",") if x]
    for mib in sizes:
        S = mib * MiB
        B = S // (2 * d * 4)
        n = args.n if S < GiB else args.n_large
        t_step, n_full = store_all_per_step(d, B, S, args.fuse)
        for tier in tiers:
            if tier in ("file", "cascade") and mib not in file_sizes:
                continue
            if tier == "pinned":
                backend = pkg.PinnedHostBackend(slot_bytes=S)
            elif tier == "cascade":
                shutil.rmtree(args.file_dir, ignore_errors=True)
                backend = pkg.CascadeBackend(args.file_dir, slot_bytes=S, dram_slots=args.dram_slots)
            else:
                shutil.rmtree(args.file_dir, ignore_errors=True)
                backend = pkg.FileBackend(args.file_dir, slot_bytes=S)
            try:
                row = point(d, B, S, n, tier, backend, t_step, args.fuse, {"store_all_n": n_full}, args.n_max)
            finally:
                backend.close()
                if tier in ("file", "cascade"):
                    shutil.rmtree(args.file_dir, ignore_errors=True)
            rows.append(row)
            print(json.dumps(row), flush=True)
        if mib == 64 and args.sim_gbs:
            for gbs in [float(x) for x in args.sim_gbs.split(",") if x]:
                backend = pkg.SimulatedBackend(gbs * 1e9, 0.0, slot_bytes=S)
                try:
                    row = point(d, B, S, args.n, f"sim{gbs:g}GBs", backend, t_step, args.fuse,
                                {"store_all_n": n_full, "link_gbs_throttle": gbs}, args.n_max)
                finally:
                    backend.close()
                rows.append(row)
                print(json.dumps(row), flush=True)
    print(json.dumps({
        "summary": "C5",
        "fused": args.fuse,
        "family": lstm.kernel_family(),
        "points": [[r["state_mib"], r["tier"], round(r["ratio_t_t_over_t_a"], 1), r["interval"],
                    round(r["overhead_vs_store_all"], 3), round(r["recompute_factor"], 3),
                    round(r["model_recompute_factor"], 3), round(r["stall_frac"], 4)] for r in rows],
        "columns": ["state_mib", "tier", "t_t/t_a", "I", "overhead", "R_meas", "R_model", "stall_frac"],
    }), flush=True)


if __name__ == "__main__":
    main()
