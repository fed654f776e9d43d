"""TEST INFRASTRUCTURE ONLY: plain-Python restatement of the reference
scheduler (pkg/src/asyncckpt/schedule.py) for small sizes.

  cost table      schedule.py:139-155  (c[s][n], INF = 2**40)
  _best_split     schedule.py:177-181  (smallest argmin)
  revolve emit    schedule.py:188-235  (right part recursive, lowest free slot)
  taped_schedule  schedule.py:279-285
  plan_multistage schedule.py:288-329
Actions are tuples: ("advance", a, b) ("save", step, slot) ("load", slot)
("tape", a, b) ("reverse", step) ("done",).
"""

from __future__ import annotations

import heapq
import json
from fractions import Fraction
import math

INF = 1 << 40


def cost_table(n_max: int, s_max: int):
    c = [[INF] * (n_max + 1) for _ in range(s_max + 1)]
    for s in range(s_max + 1):
        c[s][0] = 0
        if n_max >= 1:
            c[s][1] = 1
        for n in range(2, min(s + 1, n_max) + 1):
            c[s][n] = n
        if s == 0:
            continue
        prev, row = c[s - 1], c[s]
        for n in range(s + 2, n_max + 1):
            row[n] = min(k + prev[n - k] + row[k] for k in range(1, n))
    return c


def best_split(length: int, slots: int, c) -> int:
    best_k, best = 1, None
    for k in range(1, length):
        v = k + c[slots - 1][length - k] + c[slots][k]
        if best is None or v < best:
            best, best_k = v, k
    return best_k


def revolve(n: int, s: int):
    if n < 1 or s < 0:
        raise ValueError("bad params")
    if n > 1 and s == 0:
        raise ValueError("infeasible")
    c = cost_table(n, min(s, n))
    free = list(range(s))
    heapq.heapify(free)
    out = []

    def emit(lo, hi, slots):
        while True:
            length = hi - lo
            if length == 0:
                return
            if length <= slots + 1:
                out.append(("tape", lo, hi))
                out.extend(("reverse", k) for k in range(hi - 1, lo - 1, -1))
                return
            k = best_split(length, slots, c)
            slot = heapq.heappop(free)
            out.append(("save", lo, slot))
            out.append(("advance", lo, lo + k))
            emit(lo + k, hi, slots - 1)
            out.append(("load", slot))
            heapq.heappush(free, slot)
            hi = lo + k

    emit(0, n, s)
    out.append(("done",))
    return out


def taped(length: int):
    return [("tape", 0, length)] + [("reverse", k) for k in range(length - 1, -1, -1)] + [("done",)]


def plan_multistage(n: int, s: int, interval: int):
    """(boundaries, [(start, end, actions)], fallback)"""
    if interval >= n:
        return (0,), [(0, n, revolve(n, s))], True
    bounds = tuple(range(0, n, interval))
    segs = []
    for start in bounds:
        end = min(start + interval, n)
        L = end - start
        segs.append((start, end, taped(L) if L <= s + 1 else revolve(L, s)))
    return bounds, segs, False


def forward_executions(actions) -> int:
    return sum(a[2] - a[1] for a in actions if a[0] in ("advance", "tape"))


def to_json(actions) -> str:
    """The reference's actions_to_json format (schedule.py:486-520)."""
    objs = []
    for a in actions:
        if a[0] == "advance":
            objs.append({"op": "advance", "from": a[1], "to": a[2]})
        elif a[0] == "save":
            objs.append({"op": "save", "step": a[1], "slot": a[2]})
        elif a[0] == "load":
            objs.append({"op": "load", "slot": a[1]})
        elif a[0] == "tape":
            objs.append({"op": "tape", "from": a[1], "to": a[2]})
        elif a[0] == "reverse":
            objs.append({"op": "reverse", "step": a[1]})
        else:
            objs.append({"op": "done"})
    return json.dumps(objs)


def interval_length(t_t: float, t_a: float) -> int:
    """perfmodel.py:56-64"""
    return max(1, math.ceil(Fraction(t_t) / Fraction(t_a)))
