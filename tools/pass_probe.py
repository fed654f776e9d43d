"""Diagnostics for the C2 pass: where does the time go?

Runs the d=8, B=2^20 fp32 workload at n=2000 under several conditions and
prints one JSON line each: multistage at different intervals, revolve,
fused, with/without kernel sampling, and a K1 chain with/without a
concurrent D2H+H2D copy loop (copy-engine interference)."""

import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402

n = int(os.environ.get("PROBE_N", "2000"))
cell = lstm.random_cell(8, n, 0)
ops = lstm.operator_pair(cell, 1 << 20, "f32")
s0 = lstm.random_states(8, 1, 1 << 20, "f32")
backend = pkg.PinnedHostBackend(slot_bytes=ops.state_size)


def report(tag, st):
    dv = st.device
    out = {
        "tag": tag,
        "wall_ms": st.wall_seconds * 1e3,
        "gpu_ms": dv["gpu_seconds"] * 1e3,
        "enqueue_ms": dv["host_enqueue_seconds"] * 1e3,
        "us_per_launch": dv["gpu_seconds"] / max(1, dv["kernel_launches"]) * 1e6,
        "fwd_us": dv["fwd_sample_seconds"] / max(1, dv["fwd_samples"]) * 1e6,
        "bwd_us": dv["bwd_sample_seconds"] / max(1, dv["bwd_samples"]) * 1e6,
        "stall_ms": st.stall_seconds * 1e3,
        "stores": st.stores_issued,
        "fwd": st.forward_evals,
    }
    print(json.dumps(out), flush=True)


for tag, strat, kw in [
    ("revolve99", pkg.Revolve(99), {}),
    ("ms_I40", pkg.Multistage(199, 40), {}),
    ("ms_I40_nosample", pkg.Multistage(199, 40), {"sample": 0}),
    ("ms_I200", pkg.Multistage(199, 200), {}),
    ("ms_I1000", pkg.Multistage(999, 1000), {}),
    ("ms_I40_fused", pkg.Multistage(199, 40), {"fuse": True}),
    ("full", pkg.FullStorage(), {}),
]:
    for rep in range(2):
        _, st = pkg.execute(strat, ops, s0, backend, fuse=kw.get("fuse", False), sample_kernels=kw.get("sample", 8))
    report(tag, st)

# K1 chain with and without concurrent copies
dc = ops.native
bufs = [torch.empty_like(s0) for _ in range(4)]
bufs[0].copy_(s0)


def chain(k=200):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(k):
        bufs[(i + 1) % 4] = dc.forward(i % n, bufs[i % 4])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


alone = chain()
host = torch.empty(ops.state_size, dtype=torch.uint8).pin_memory()
host2 = torch.empty(ops.state_size, dtype=torch.uint8).pin_memory()
dev = torch.empty(ops.state_size, dtype=torch.uint8, device="cuda")
dev2 = torch.empty(ops.state_size, dtype=torch.uint8, device="cuda")
stop = threading.Event()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def copier():
    while not stop.is_set():
        with torch.cuda.stream(s1):
            host.copy_(dev, non_blocking=True)
        with torch.cuda.stream(s2):
            dev2.copy_(host2, non_blocking=True)
        s1.synchronize()
        s2.synchronize()


th = threading.Thread(target=copier)
th.start()
with_copies = chain()
stop.set()
th.join()
print(json.dumps({"tag": "k1_chain", "alone_us": alone, "with_d2h_h2d_us": with_copies}), flush=True)
backend.close()
