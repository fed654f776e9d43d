"""Parity check run in a subprocess by tests/test_gpu_variants.py: the fused
advance / tape / reverse launches and one per-step forward + backward of the
kernel variant selected by the environment, against the float64 oracle."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1806_01117_b200.lstm as lstm  # noqa: E402
from oracle import lstm_oracle as L  # noqa: E402


def main():
    d, batch, n = int(sys.argv[1]), int(sys.argv[2]), 24
    cell, ocell = lstm.random_cell(d, n, 3), L.random_cell(d, n, 3)
    rng = np.random.default_rng(4)
    x = torch.from_numpy(rng.uniform(-1, 1, (2, d, batch)).astype(np.float32)).cuda()
    a = torch.from_numpy(rng.uniform(-1, 1, (2, d, batch)).astype(np.float32)).cuda()
    dc = lstm.device_cell(cell, batch, "f32")
    out = {}
    ref = x.double().cpu().numpy()
    refs = []
    for k in range(1, 21):
        ref = L.forward_step(ocell, k, ref)
        refs.append(ref)
    out["advance"] = L.rel_l2(dc.advance(1, 21, x).cpu().numpy(), refs[-1])
    tape = dc.forward_many(1, 20, x)
    out["tape"] = max(L.rel_l2(t.cpu().numpy(), r) for t, r in zip(tape, refs))
    states = [x] + tape[:-1]
    adj = a.double().cpu().numpy()
    for i, k in reversed(list(enumerate(range(1, 21)))):
        adj = L.backward_step(ocell, k, states[i].double().cpu().numpy(), adj)
    try:
        out["reverse"] = L.rel_l2(dc.backward_many(1, states, a).cpu().numpy(), adj)
    except ValueError:  # the generic path has no fused reverse (the engine then runs per step)
        pass
    out["forward"] = L.rel_l2(dc.forward(5, x).cpu().numpy(), L.forward_step(ocell, 5, x.double().cpu().numpy()))
    out["backward"] = L.rel_l2(dc.backward(5, x, a).cpu().numpy(),
                               L.backward_step(ocell, 5, x.double().cpu().numpy(), a.double().cpu().numpy()))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
