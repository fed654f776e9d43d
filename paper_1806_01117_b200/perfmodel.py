"""Timing model used for the interval choice and for reporting.

``interval_length`` is on the hot path (it sets I from calibrated times) and
is computed natively with exact rational arithmetic: ceil(t_t / t_a) over
the exact binary values of the two doubles, like the reference's
ceil(Fraction(t_t) / Fraction(t_a)) (perfmodel.py:56-64).  The closed forms
below (perfmodel.py:45-75) are kept for reporting the measured recompute
factor against the paper's constant-overhead model.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

from . import _native as N
from .schedule import recompute_factor


@dataclass(frozen=True)
class PerfParams:
    """n steps, s slots, per-step forward t_a, backward t_b and per-state
    Level-2 transfer time t_t (seconds, positive)."""

    n: int
    s: int
    t_a: float
    t_b: float
    t_t: float

    def __post_init__(self) -> None:
        if self.n < 1:
            raise ValueError(f"n must be >= 1, got {self.n}")
        if self.s < 0:
            raise ValueError(f"s must be >= 0, got {self.s}")
        for name in ("t_a", "t_b", "t_t"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


def interval_length(t_t: float, t_a: float) -> int:
    """max(1, ceil(t_t / t_a)) computed exactly (saturates at 2^63 - 1)."""
    if t_t <= 0 or t_a <= 0:
        raise ValueError("t_t and t_a must be positive")
    out = C.c_int64(0)
    N.check(N.lib.ackpt_interval_length(float(t_t), float(t_a), C.byref(out)))
    return out.value


def t_infinity(p: PerfParams) -> float:
    """Store-all time n (t_a + t_b)."""
    return float(p.n * (Fraction(p.t_a) + Fraction(p.t_b)))


def t_revolve(p: PerfParams) -> float:
    """n R(n, s) t_a + n t_b."""
    return float(p.n * recompute_factor(p.n, p.s) * Fraction(p.t_a) + p.n * Fraction(p.t_b))


def t_async(p: PerfParams) -> float:
    """n R(I, s) t_a + n t_b with I = interval_length(t_t, t_a); revolve when I >= n.

    Counts the recompute inside intervals only, as the reference model does;
    the executor's measured factor additionally includes the forward sweep
    (runtime.py:23-27), i.e. 1 + R(I, s)."""
    interval = interval_length(p.t_t, p.t_a)
    if interval >= p.n:
        return t_revolve(p)
    return float(p.n * recompute_factor(interval, p.s) * Fraction(p.t_a) + p.n * Fraction(p.t_b))


def overhead_model(n: int, s: int, interval: int, t_a: float, t_b: float) -> dict:
    """Predicted wall and overhead vs store-all of the executor's multistage
    run (sweep + taped/revolved intervals + backward) and of plain revolve."""
    t_inf = n * (t_a + t_b)
    if interval >= n:
        ms = forward_cost_total = None
    else:
        full, rem = divmod(n, interval)
        from .schedule import forward_cost

        inner = full * forward_cost(interval, s) + (forward_cost(rem, s) if rem else 0)
        forward_cost_total = n + inner
        ms = forward_cost_total * t_a + n * t_b
    rv = float(recompute_factor(n, s)) * n * t_a + n * t_b if s > 0 or n == 1 else None
    return {
        "t_infinity": t_inf,
        "multistage_seconds": ms,
        "multistage_overhead": (ms / t_inf) if ms else None,
        "multistage_forward_evals": forward_cost_total,
        "revolve_seconds": rv,
        "revolve_overhead": (rv / t_inf) if rv else None,
    }


def emit_curves(s: int, intervals, n_max: int) -> list:
    """Recompute-factor curves over n = 1, 2, 4, ... <= n_max: the single-level
    Revolve(s) factor and, per interval I, the two-level factor R(min(I, n), s)
    (flat once n passes I) -- the reference's emit_curves (perfmodel.py)."""
    if n_max < 1:
        raise ValueError(f"n_max must be >= 1, got {n_max}")
    rows = []
    n = 1
    while n <= n_max:
        row = {"n": n, "revolve": recompute_factor(n, s)}
        for interval in intervals:
            row[f"async_I{interval}"] = recompute_factor(min(interval, n), s)
        rows.append(row)
        n *= 2
    return rows


def curves_to_csv(rows) -> str:
    """CSV of emit_curves rows, factors with 6 significant digits."""
    rows = list(rows)
    if not rows:
        return ""
    cols = list(rows[0])
    body = [",".join(cols)]
    body += [",".join([str(r["n"])] + [f"{float(r[c]):.6g}" for c in cols[1:]]) for r in rows]
    return "\n".join(body) + "\n"
