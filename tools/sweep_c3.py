"""BASELINE config 3: n = 10^3 -> 10^5 at fixed snaps on one GPU.

Multistage(I) (calibrated I, slots >= I so intervals are taped) against
Revolve(I) with the same Level-1 budget, fused execution,
C2 state (d=8, B=2^20 fp32, 64 MiB).  Overhead is against the measured
fused store-all per-step time.  One JSON line per n, then a summary line.
The chain is lstm.long_memory_cell (forget bias +5, same cost per step as
random_cell), whose fp32 adjoint stays far from underflow up to n = 10^5, so
the Multistage-vs-Revolve bit-identity column compares non-zero adjoints
(the reference cell's adjoint is exactly 0 past n ~ 190); the adjoint norm
is reported beside it.

  python tools/sweep_c3.py [--ns 1000,2000,...] [--per-step]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="1000,2000,5000,10000,20000,50000,100000")
    ap.add_argument("--per-step", dest="fuse", action="store_false")
    ap.add_argument("--batch", type=int, default=1 << 20)
    args = ap.parse_args()
    ns = [int(x) for x in args.ns.split(",")]
    d, B = 8, args.batch
    state0 = lstm.random_states(d, 1, B, "f32")
    backend = pkg.PinnedHostBackend(slot_bytes=2 * d * B * 4)

    # store-all per-step time at n=1000 (same execution mode)
    full_ops = lstm.operator_pair(lstm.random_cell(d, 1000, 0), B, "f32")
    pkg.execute(pkg.FullStorage(), full_ops, state0, fuse=args.fuse)
    _, fst = pkg.execute(pkg.FullStorage(), full_ops, state0, fuse=args.fuse)
    t_step = fst.wall_seconds / 1000
    t_a, t_b, t_t = pkg.calibrate(full_ops, backend, 5, state0, fuse=args.fuse)
    interval = pkg.interval_length(t_t, t_a)
    del full_ops
    torch.cuda.empty_cache()

    rows = []
    for n in ns:
        ops = lstm.operator_pair(lstm.long_memory_cell(d, n, 0), B, "f32")
        row = {"n": n, "interval": interval, "store_all_us_per_step": t_step * 1e6}
        for name, strat in (("multistage", pkg.Multistage(interval, interval)), ("revolve", pkg.Revolve(interval))):
            adj, st = pkg.execute(strat, ops, state0, backend, fuse=args.fuse)  # warm-up (+ table build)
            adj, st = pkg.execute(strat, ops, state0, backend, fuse=args.fuse)
            row[name] = {
                "wall_s": st.wall_seconds,
                "steps_per_s": n / st.wall_seconds,
                "overhead_vs_store_all": st.wall_seconds / (n * t_step),
                "recompute_factor": st.forward_evals / n,
                "model_recompute_factor": (1 + float(pkg.recompute_factor(min(interval, n), interval)))
                if name == "multistage" and interval < n else float(pkg.recompute_factor(n, interval)),
                "peak_l1_states": st.peak_l1_bytes / (2 * d * B * 4),
                "stall_s": st.stall_seconds,
            }
            if name == "multistage":
                ms_adj = adj
            else:
                norm = float(ms_adj.double().norm())
                row["adjoint_norm"] = norm
                row["adjoint_nonzero_frac"] = float((ms_adj != 0).double().mean())
                row["bit_identical"] = bool(torch.equal(adj, ms_adj)) and norm > 0
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ops
        torch.cuda.empty_cache()
    print(json.dumps({"summary": "C3", "fused": args.fuse, "interval": interval,
                      "multistage_overhead": [r["multistage"]["overhead_vs_store_all"] for r in rows],
                      "revolve_overhead": [r["revolve"]["overhead_vs_store_all"] for r in rows],
                      "ns": ns}), flush=True)
    backend.close()


if __name__ == "__main__":
    main()
