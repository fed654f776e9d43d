"""Adjoint error of each execution mode / kernel family at the headline
shape (C2: d=8, B=2^20, n=10^4, Multistage(999, I=75)) on the long-memory
cell, against the float64 oracle on sampled sequences.  Prints JSON lines."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402
from oracle import lstm_oracle as L  # noqa: E402
from oracle import runtime_oracle as RO  # noqa: E402

d = 8
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
fb = float(sys.argv[3]) if len(sys.argv) > 3 else 5.0
cell = lstm.long_memory_cell(d, n, 0, fb)
ops = lstm.operator_pair(cell, batch, "f32")
s0 = lstm.random_states(d, 1, batch, "f32")
rows = np.unique(np.linspace(0, batch - 1, 64).astype(np.int64))
s0r = s0[:, :, rows].double().cpu().numpy()
ref, _ = RO.execute("full", L.long_memory_cell(d, n, 0, fb), s0r)
ref32, _ = RO.execute("full", L.long_memory_cell(d, n, 0, fb), s0r, dtype=np.float32)
print(json.dumps({"forget_bias": fb, "mode": "numpy-fp32", "rel_l2": L.rel_l2(ref32, ref),
                  "norm": float(np.linalg.norm(ref))}))
for fam in ("tcgen05", "ffma2"):
    lstm.set_kernel_family(fam)
    for fuse in (True, False):
        if not fuse and fam == "ffma2":
            continue
        with pkg.PinnedHostBackend(slot_bytes=ops.state_size) as b:
            adj, st = pkg.execute(pkg.Multistage(999, 75), ops, s0, b, fuse=fuse)
        got = adj[:, :, rows].double().cpu().numpy()
        per = [L.rel_l2(got[:, :, i], ref[:, :, i]) for i in range(len(rows))]
        print(json.dumps({"mode": ("fused-" + fam) if fuse else "per-step", "rel_l2": L.rel_l2(got, ref),
                          "median_per_seq": float(np.median(per)), "max_per_seq": float(np.max(per)),
                          "gpu_norm": adj.double().norm().item()}), flush=True)
# the forward state after n steps (no adjoint): trajectory error alone
lstm.set_kernel_family("tcgen05")
fin = ops.native.advance(0, n, s0)
sref = s0r
for k in range(n):
    sref = L.forward_step(L.long_memory_cell(d, n, 0, fb), k, sref)
print(json.dumps({"mode": "advance-tcgen05 final state", "rel_l2": L.rel_l2(fin[:, :, rows].double().cpu().numpy(), sref)}))
