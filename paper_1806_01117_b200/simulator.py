"""Discrete-event timeline of one forward/backward pass on a virtual clock
(the reference's simulator.py API: TimelineEvent, simulate, timeline_to_json).

Two lanes: "compute" (forward / backward steps and stalls, strictly serial)
and "transfer" (stores and fetches, one at a time).  Times are exact
Fractions, so with the calibrated interval the totals reproduce the closed
forms of perfmodel (t_infinity, t_revolve, t_async) exactly.  Semantics
(simulator.py:1-26 of the reference):

* FullStorage / Revolve / a multistage fallback: one compute event per
  forward step (t_a) and per reverse step (t_b) of the schedule.
* Multistage: the forward sweep issues each boundary's store on arrival,
  stalling compute while the previous store is still on the transfer lane;
  the backward issues the first fetch at the end of the sweep and the fetch
  of interval j-1 when interval j starts reversing (fetches never block
  compute), and charges each interval only the part of its inner schedule
  from the first Reverse on (its first traversal was booked in the sweep).

The engine's measured timeline (``execute(..., timeline=True)``) uses the
same event vocabulary, so the two can be compared event for event on the
transfer lane and in total time (the executor additionally re-runs each
interval's first traversal, n t_a more compute, runtime.py:23-27).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, List, Sequence, Tuple

from .perfmodel import PerfParams, interval_length
from .runtime import FullStorage, Multistage, Revolve
from .schedule import Advance, Reverse, ScheduleParams, TapeForward, plan_multistage, revolve_schedule, taped_schedule

FORWARD = "forward_compute"
BACKWARD = "backward_compute"
STORE = "store"
FETCH = "fetch"
STALL = "stall"

COMPUTE_LANE = "compute"
TRANSFER_LANE = "transfer"


@dataclass(frozen=True)
class TimelineEvent:
    kind: str
    from_step: int
    to_step: int
    start: Fraction
    end: Fraction
    lane: str


class _Lanes:
    """Virtual clock of the compute lane plus the transfer lane's free time."""

    def __init__(self, p: PerfParams):
        self.t_a, self.t_b, self.t_t = Fraction(p.t_a), Fraction(p.t_b), Fraction(p.t_t)
        self.now = Fraction(0)
        self.link_free = Fraction(0)
        self.out: List[TimelineEvent] = []

    def compute(self, kind: str, step: int, cost: Fraction) -> None:
        end = self.now + cost
        self.out.append(TimelineEvent(kind, step, step + 1, self.now, end, COMPUTE_LANE))
        self.now = end

    def replay(self, actions: Iterable, offset: int = 0) -> None:
        for act in actions:
            if isinstance(act, (Advance, TapeForward)):
                for k in range(act.from_step, act.to_step):
                    self.compute(FORWARD, offset + k, self.t_a)
            elif isinstance(act, Reverse):
                self.compute(BACKWARD, offset + act.step, self.t_b)

    def wait_link(self, step: int) -> None:
        if self.link_free > self.now:
            self.out.append(TimelineEvent(STALL, step, step, self.now, self.link_free, COMPUTE_LANE))
            self.now = self.link_free

    def transfer(self, kind: str, key: int) -> None:
        begin = max(self.now, self.link_free)
        self.link_free = begin + self.t_t
        self.out.append(TimelineEvent(kind, key, key, begin, self.link_free, TRANSFER_LANE))


def _from_first_reverse(actions: Sequence) -> Sequence:
    for i, act in enumerate(actions):
        if isinstance(act, Reverse):
            return actions[i:]
    return ()


def simulate(strategy, p: PerfParams) -> Tuple[List[TimelineEvent], float]:
    """Events and total (compute-lane) seconds of one pass."""
    lanes = _Lanes(p)
    if isinstance(strategy, FullStorage):
        lanes.replay(taped_schedule(p.n))
    elif isinstance(strategy, Revolve):
        lanes.replay(revolve_schedule(ScheduleParams(p.n, strategy.slots)))
    elif isinstance(strategy, Multistage):
        interval = strategy.interval if strategy.interval is not None else interval_length(p.t_t, p.t_a)
        plan = plan_multistage(p.n, strategy.slots, interval)
        if plan.fallback:
            lanes.replay(plan.segments[0].actions)
        else:
            bounds = list(plan.boundaries)
            for i, b in enumerate(bounds):
                lanes.wait_link(b)
                lanes.transfer(STORE, b)
                stop = bounds[i + 1] if i + 1 < len(bounds) else plan.n
                for k in range(b, stop):
                    lanes.compute(FORWARD, k, lanes.t_a)
            segs = plan.segments
            lanes.transfer(FETCH, segs[-1].start)
            for j in reversed(range(len(segs))):
                if j > 0:
                    lanes.transfer(FETCH, segs[j - 1].start)
                lanes.replay(_from_first_reverse(segs[j].actions), segs[j].start)
    else:
        raise TypeError(f"unknown strategy {strategy!r}")
    return lanes.out, float(lanes.now)


def strategy_name(strategy) -> str:
    for kind, name in ((FullStorage, "full"), (Revolve, "revolve"), (Multistage, "multistage")):
        if isinstance(strategy, kind):
            return name
    raise TypeError(f"unknown strategy {strategy!r}")


def timeline_to_obj(strategy, events: Sequence[TimelineEvent], total: float) -> dict:
    return {
        "strategy": strategy_name(strategy),
        "total": total,
        "events": [
            {"kind": e.kind, "from": e.from_step, "to": e.to_step, "start": float(e.start), "end": float(e.end),
             "lane": e.lane}
            for e in events
        ],
    }


def timeline_to_json(strategy, events: Sequence[TimelineEvent], total: float) -> str:
    return json.dumps(timeline_to_obj(strategy, events, total))


def coarsen(events: Sequence[TimelineEvent]) -> List[TimelineEvent]:
    """Merge runs of back-to-back compute events of one kind over consecutive
    steps (forward k, k+1, ... or reverse k, k-1, ...) into one event
    spanning the steps, the granularity of a fused launch."""
    out: List[TimelineEvent] = []
    for e in events:
        if out and e.lane == COMPUTE_LANE and e.kind in (FORWARD, BACKWARD):
            last = out[-1]
            if last.kind == e.kind and last.lane == COMPUTE_LANE and last.end == e.start:
                if e.kind == FORWARD and last.to_step == e.from_step:
                    out[-1] = TimelineEvent(e.kind, last.from_step, e.to_step, last.start, e.end, e.lane)
                    continue
                if e.kind == BACKWARD and last.from_step == e.to_step:
                    out[-1] = TimelineEvent(e.kind, e.from_step, last.to_step, last.start, e.end, e.lane)
                    continue
        out.append(e)
    return out
