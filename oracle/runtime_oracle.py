"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference executor
(pkg/src/asyncckpt/runtime.py) over numpy states, used as the parity checker
for counters, peak_l1_bytes and adjoints, and as the timed CPU baseline.

  _ByteLedger         runtime.py:123-159
  _Execution          runtime.py:162-199
  run_schedule        runtime.py:201-252
  multistage sweeps   runtime.py:269-322
  execute             runtime.py:339-381
Transfers complete synchronously (an in-memory dict), so stall is 0.
"""

from __future__ import annotations

import time

import numpy as np

from . import lstm_oracle as L
from . import schedule_oracle as SO


class Stats(dict):
    pass


class _Ledger:
    def __init__(self):
        self.slot = self.tape = self.xfer = self.peak = 0

    def bump(self):
        self.peak = max(self.peak, self.slot + self.tape + self.xfer)


class _Exec:
    def __init__(self, cell, n, state_size, dtype, seed_fn):
        self.cell, self.n, self.S, self.dtype = cell, n, state_size, dtype
        self.seed_fn = seed_fn
        self.fwd = self.bwd = self.stores = self.fetches = 0
        self.ledger = _Ledger()
        self.adj = None
        self.seeded = False

    def forward(self, k, state):
        state = L.forward_step(self.cell, k, state, self.dtype)
        self.fwd += 1
        if k + 1 == self.n and not self.seeded:
            self.adj = self.seed_fn(state)
            self.seeded = True
        return state

    def backward(self, k, state):
        if self.adj is None:
            raise RuntimeError(f"Reverse {k} before the adjoint was seeded")
        self.adj = L.backward_step(self.cell, k, state, self.adj, self.dtype)
        self.bwd += 1

    def run_schedule(self, actions, offset, state, capacity):
        # slot liveness: save index -> index of its last read (schedule.py:347-362)
        last, writer = {}, {}
        for idx, a in enumerate(actions):
            if a[0] == "save":
                writer[a[2]] = idx
                last[idx] = -1
            elif a[0] == "load" and a[1] in writer:
                last[writer[a[1]]] = idx
        pool, write_idx, tape, cur = {}, {}, [], 0
        for idx, a in enumerate(actions):
            op = a[0]
            if op in ("advance", "tape"):
                assert a[1] == cur
                for rel in range(a[1], a[2]):
                    if op == "tape":
                        tape.append((rel, state))
                        self.ledger.tape += self.S
                        self.ledger.bump()
                    state = self.forward(offset + rel, state)
                cur = a[2]
            elif op == "save":
                assert 0 <= a[2] < capacity
                pool[a[2]] = (offset + cur, state)
                write_idx[a[2]] = idx
                self.ledger.slot = len(pool) * self.S
                self.ledger.bump()
            elif op == "load":
                step, state = pool[a[1]]
                cur = step - offset
                if last.get(write_idx.get(a[1], -1), -2) == idx:
                    del pool[a[1]]
                    self.ledger.slot = len(pool) * self.S
                    self.ledger.bump()
            elif op == "reverse":
                rel, taped = tape.pop()
                assert rel == a[1]
                self.ledger.tape -= self.S
                self.backward(offset + a[1], taped)
            else:
                break
        self.ledger.slot = 0
        self.ledger.bump()
        return state


def execute(kind, cell, state0, *, slots=0, interval=None, dtype=np.float64, seed=None):
    """kind in {"full", "revolve", "multistage"}; returns (adjoint, stats).

    state0: (2, d, B) array.  seed: None -> loss-gradient seed (lstm.py:161-163),
    else a concrete adjoint array.  Counters follow runtime.py exactly."""
    n = cell.n_steps
    S = state0.size * np.dtype(dtype).itemsize
    seed_fn = (lambda fin: L.seed(cell, fin).astype(dtype)) if seed is None else (lambda fin: seed)
    ex = _Exec(cell, n, S, dtype, seed_fn)
    state0 = state0.astype(dtype)
    # plans are built outside the timed window, like runtime.py:359-363
    if kind == "full":
        acts = SO.taped(n)
    elif kind == "revolve":
        acts = SO.revolve(n, slots)
    elif kind == "multistage":
        bounds, segs, fallback = SO.plan_multistage(n, slots, interval)
    t0 = time.perf_counter()
    if kind == "full":
        ex.run_schedule(acts, 0, state0, 0)
    elif kind == "revolve":
        ex.run_schedule(acts, 0, state0, slots)
    elif kind == "multistage":
        if fallback:
            ex.run_schedule(segs[0][2], 0, state0, slots)
        else:
            store = {}
            state = state0
            inflight = False
            for idx, b in enumerate(bounds):  # runtime.py:281-293
                if inflight:
                    ex.ledger.xfer -= S
                store[b] = state
                ex.stores += 1
                ex.ledger.xfer += S
                ex.ledger.bump()
                inflight = True
                end = bounds[idx + 1] if idx + 1 < len(bounds) else n
                for k in range(b, end):
                    state = ex.forward(k, state)
            if inflight:
                ex.ledger.xfer -= S
            # backward with one-interval-ahead prefetch (runtime.py:311-322)
            ex.fetches += 1
            ex.ledger.xfer += S
            ex.ledger.bump()
            for j in range(len(segs) - 1, -1, -1):
                start, end, acts = segs[j]
                payload = store[start]
                if j > 0:
                    ex.fetches += 1
                    ex.ledger.xfer += S
                    ex.ledger.bump()
                ex.ledger.xfer -= S
                ex.run_schedule(acts, start, payload, slots)
    else:
        raise ValueError(kind)
    wall = time.perf_counter() - t0
    stats = Stats(
        forward_evals=ex.fwd,
        backward_evals=ex.bwd,
        stores_issued=ex.stores,
        prefetches_issued=ex.fetches,
        stall_seconds=0.0,
        peak_l1_bytes=ex.ledger.peak,
        wall_seconds=wall,
    )
    return ex.adj, stats

