"""Executes a forward/backward operator pair under a reversal strategy on
the GPU.  Same API as the reference runtime (pkg/src/asyncckpt/runtime.py):
``OperatorPair``, ``ExecutionStats``, ``FullStorage`` / ``Revolve`` /
``Multistage``, ``execute``, ``run_forward_sweep``, ``run_backward_sweep``,
``calibrate``.

The action interpreter, the multistage sweeps, the byte ledger and all waits
run in C++ (csrc/engine.cpp) on CUDA streams; Python only prepares the call.
States are torch CUDA tensors of ``state_size`` bytes (``bytes`` inputs are
staged to the device and the adjoint is returned as ``bytes`` then).

Operators come in two kinds:
  * native (``OperatorPair.native`` set, e.g. ``lstm.operator_pair``): the
    engine launches the sm_100a step kernels directly;
  * Python callables over CUDA tensors: wrapped as C callbacks of the
    ackpt_operator plugin interface (one GIL round trip per step).

Setting CKPT_DISABLE_PREFETCH=1 issues each fetch right before its interval
(runtime.py:19-21, 302); results are unchanged, only stalls grow.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import asdict, dataclass, field
from typing import Any, Callable, Optional, Union

import torch

from . import _native as N
from .errors import SizeMismatch
from .perfmodel import interval_length
from .schedule import MultistagePlan
from .storage import Level2Backend, as_device_bytes, as_host_bytes, nbytes_of

ForwardStep = Callable[[int, Any], Any]
BackwardStep = Callable[[int, Any, Any], Any]
SeedSource = Union[bytes, torch.Tensor, Callable[[Any], Any]]


@dataclass(frozen=True)
class OperatorPair:
    """Deterministic forward and backward operators over fixed-size states.

    forward_step(k, state_k) -> state_{k+1}; backward_step(k, state_k,
    adjoint_{k+1}) -> adjoint_k; adjoint_seed: adjoint at step n, concrete or
    a callable of the final state (runtime.py:62-87).  ``native`` optionally
    carries the device operator the engine calls without Python.
    """

    forward_step: ForwardStep
    backward_step: BackwardStep
    state_size: int
    n_steps: int
    adjoint_seed: SeedSource
    native: Any = field(default=None, compare=False, repr=False)

    def __post_init__(self) -> None:
        if self.n_steps < 1:
            raise ValueError(f"n_steps must be >= 1, got {self.n_steps}")
        if self.state_size <= 0:
            raise ValueError(f"state_size must be positive, got {self.state_size}")

    def seed_for(self, final_state):
        if callable(self.adjoint_seed):
            return self.adjoint_seed(final_state)
        return self.adjoint_seed


@dataclass
class ExecutionStats:
    """The reference's seven counters (runtime.py:90-101).  B200 extras
    (gpu_seconds, kernel_launches, interval, ...) are in ``.device``."""

    forward_evals: int = 0
    backward_evals: int = 0
    stores_issued: int = 0
    prefetches_issued: int = 0
    stall_seconds: float = 0.0
    peak_l1_bytes: int = 0
    wall_seconds: float = 0.0

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass(frozen=True)
class FullStorage:
    pass


@dataclass(frozen=True)
class Revolve:
    slots: int


@dataclass(frozen=True)
class Multistage:
    slots: int
    interval: Optional[int] = None  # None: calibrate, then ceil(t_t / t_a)


Strategy = Union[FullStorage, Revolve, Multistage]


def _stats_from(st: N.Stats) -> ExecutionStats:
    out = ExecutionStats(
        forward_evals=st.forward_evals,
        backward_evals=st.backward_evals,
        stores_issued=st.stores_issued,
        prefetches_issued=st.prefetches_issued,
        stall_seconds=st.stall_seconds,
        peak_l1_bytes=st.peak_l1_bytes,
        wall_seconds=st.wall_seconds,
    )
    out.timeline = None
    out.device = {
        "gpu_seconds": st.gpu_seconds,
        "kernel_launches": st.kernel_launches,
        "interval": st.interval,
        "fallback": bool(st.fallback),
        "device_buffers": st.device_buffers,
        "link_bytes": st.link_bytes,
        "fused_advances": st.fused_advances,
        "fwd_sample_seconds": st.fwd_sample_seconds,
        "fwd_samples": st.fwd_samples,
        "bwd_sample_seconds": st.bwd_sample_seconds,
        "bwd_samples": st.bwd_samples,
        "host_enqueue_seconds": st.host_enqueue_seconds,
    }
    return out


# ---------------------------------------------------------------------------
# Python-callable operators through the C plugin interface


class _DevBuf:
    """__cuda_array_interface__ view of a raw device pointer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,),
            "typestr": "|u1",
            "data": (ptr, False),
            "version": 3,
            "strides": None,
            "stream": None,
        }


def _view(ptr: int, nbytes: int) -> torch.Tensor:
    return torch.as_tensor(_DevBuf(ptr, nbytes), device="cuda")


class _CallbackOperator:
    """ackpt_operator whose functions call the OperatorPair's Python callables
    on the engine's stream.  Callables see uint8 CUDA tensors of state_size
    bytes and may return tensors (any dtype, same byte size) or bytes."""

    def __init__(self, ops: OperatorPair):
        # the callables only: no reference back to `ops`, which owns this object
        forward_step, backward_step, adjoint_seed = ops.forward_step, ops.backward_step, ops.adjoint_seed
        S = ops.state_size
        pending: list = []  # raised exception, shared with the closures (no self-cycle)
        self._pending = pending

        def put(ptr: int, value) -> None:
            dst = _view(ptr, S)
            src = as_device_bytes(value)
            if src.numel() != S:
                raise SizeMismatch(f"operator returned {src.numel()} bytes, expected {S}")
            dst.copy_(src)

        def guard(fn):
            def call(*args):
                stream = args[-1]
                try:
                    with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                        fn(*args[:-1])
                    return N.OK
                except BaseException as exc:  # reported through the status code
                    pending.append(exc)
                    return N.EXECUTION_ERROR

            return call

        def fwd(ctx, step, inp, out):
            put(out, forward_step(step, _view(inp, S)))

        def bwd(ctx, step, state, adj_in, adj_out):
            put(adj_out, backward_step(step, _view(state, S), _view(adj_in, S)))

        def seed(ctx, final, adj_out):
            put(adj_out, adjoint_seed(_view(final, S)) if callable(adjoint_seed) else adjoint_seed)

        self._fns = (
            N.FORWARD_FN(guard(fwd)),
            N.BACKWARD_FN(guard(bwd)),
            N.SEED_FN(guard(seed)) if callable(ops.adjoint_seed) else N.SEED_FN(),
        )
        self.op = N.Operator(None, self._fns[0], self._fns[1], self._fns[2], N.ADVANCE_FN(), S, ops.n_steps,
                             N.FORWARD_MANY_FN(), N.BACKWARD_MANY_FN())

    def raise_pending(self) -> None:
        if self._pending:
            exc = self._pending[0]
            self._pending.clear()
            raise exc


class _Engine:
    """Native engine (HBM slot pool, events, streams).  ``owner`` keeps the
    operator's context alive; the engine itself is cached ON that context
    (or on the OperatorPair for callbacks), never the other way round, so
    dropping the operator pair frees the pool immediately by refcount."""

    def __init__(self, op: N.Operator, owner=None):
        self.owner = owner
        self.plan_key = None
        self._stable = {}
        h = C.c_void_p()
        N.check(N.lib.ackpt_engine_create(C.byref(op), C.byref(h)))
        self.handle = h.value

    def stable(self, name: str, like: torch.Tensor) -> torch.Tensor:
        """Engine-owned device buffer shaped like `like`, reused across calls."""
        buf = self._stable.get(name)
        if buf is None or buf.shape != like.shape or buf.dtype != like.dtype or buf.device != like.device:
            buf = torch.empty_like(like, memory_format=torch.contiguous_format)
            self._stable[name] = buf
        return buf

    def __del__(self):
        try:
            if self.handle:
                N.lib.ackpt_engine_destroy(self.handle)
        except Exception:
            pass


def _engine_for(ops: OperatorPair) -> tuple:
    """(engine, callback wrapper or None), cached per operator pair."""
    if ops.native is not None:
        eng = getattr(ops.native, "_engine", None)
        if eng is None:
            eng = _Engine(ops.native.operator())  # no back-reference: ops.native owns it
            ops.native._engine = eng
        return eng, None
    hit = ops.__dict__.get("_ackpt_engine")
    if hit is None:
        cb = _CallbackOperator(ops)
        hit = (_Engine(cb.op, cb), cb)
        object.__setattr__(ops, "_ackpt_engine", hit)  # frozen dataclass: cache only
    return hit


def release(ops: OperatorPair) -> None:
    """Free the engine (HBM slot pool, events) cached for ``ops`` now rather
    than when ``ops`` is dropped."""
    if ops.native is not None:
        if getattr(ops.native, "_engine", None) is not None:
            ops.native._engine = None
    else:
        ops.__dict__.pop("_ackpt_engine", None)


class _PaddedNative:
    """Native operator whose steps also hold the compute stream (test support)."""

    def __init__(self, base, forward_delay: float, backward_delay: float):
        self.base = base
        self._op = N.Operator()
        N.check(N.lib.ackpt_pad_operator_create(C.byref(base.operator()), forward_delay, backward_delay, C.byref(self._op)))

    def operator(self) -> N.Operator:
        return self._op

    def __del__(self):
        try:
            self._engine = None
            N.lib.ackpt_pad_operator_destroy(C.byref(self._op))
        except Exception:
            pass


def pad_operator(ops: OperatorPair, forward_delay: float, backward_delay: float) -> OperatorPair:
    """Stretch every forward / backward step of a native operator pair by a
    device-side delay (the reference tests' pad_operators, test_runtime.py:33-52,
    which sleep on the compute thread).  Results are unchanged."""
    if ops.native is None:
        raise TypeError("pad_operator needs a native operator pair")
    return OperatorPair(
        forward_step=ops.forward_step,
        backward_step=ops.backward_step,
        state_size=ops.state_size,
        n_steps=ops.n_steps,
        adjoint_seed=ops.adjoint_seed,
        native=_PaddedNative(ops.native, forward_delay, backward_delay),
    )


def _tier(backend: Optional[Level2Backend], state_size: int) -> Optional[int]:
    if backend is None:
        return None
    if not isinstance(backend, Level2Backend):
        raise TypeError("backend must be a paper_1806_01117_b200 Level2Backend")
    return backend._ensure(state_size)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _seed_ptr(ops: OperatorPair, cb) -> tuple:
    """Device buffer of a concrete seed, or (None, None) when a seed function runs."""
    if callable(ops.adjoint_seed):
        return None, None
    buf = as_device_bytes(ops.adjoint_seed)
    if buf.numel() != ops.state_size:
        raise SizeMismatch(f"adjoint seed is {buf.numel()} bytes, expected {ops.state_size}")
    return buf.data_ptr(), buf


def _output_like(state) -> torch.Tensor:
    if isinstance(state, torch.Tensor):
        return torch.empty_like(state, device=state.device if state.is_cuda else "cuda",
                                memory_format=torch.contiguous_format)
    return torch.empty(nbytes_of(state), dtype=torch.uint8, device="cuda")


def _finish(out: torch.Tensor, like):
    return out if isinstance(like, torch.Tensor) else as_host_bytes(out)


def _prepare(engine: _Engine, strategy_code: int, slots: int, interval: int, tier) -> None:
    N.check(N.lib.ackpt_engine_prepare(engine.handle, strategy_code, slots, interval, tier))


def _device_state(initial_state) -> torch.Tensor:
    if isinstance(initial_state, torch.Tensor):
        t = initial_state.detach()
        return (t if t.is_cuda else t.cuda()).contiguous()
    return as_device_bytes(initial_state)


def _resolve_interval(strategy: Multistage, ops, backend, initial_state, fuse: bool) -> int:
    # runtime.py:325-336
    if strategy.interval is not None:
        if strategy.interval < 1:
            raise ValueError(f"interval must be >= 1, got {strategy.interval}")
        return strategy.interval
    t_a, _, t_t = calibrate(ops, backend, 5, initial_state, fuse=fuse)
    return interval_length(t_t, t_a)


def execute(
    strategy: Strategy,
    ops: OperatorPair,
    initial_state,
    backend: Optional[Level2Backend] = None,
    *,
    fuse: bool = False,
    sample_kernels: int = 0,
    timeline: bool = False,
    graph: bool = False,
):
    """One forward/backward pass; returns (step-0 adjoint, stats).

    The adjoint is bit-identical across strategies (deterministic kernels,
    no atomics).  Multistage requires a backend.  ``fuse=True`` runs each
    Advance action as one fused launch (counters unchanged).  Planning,
    calibration and HBM pool allocation happen before the timed window
    (runtime.py:355-363).  ``timeline=True`` also records the measured event
    timeline (``stats.timeline``: simulator.TimelineEvent list, seconds since
    the run's start; one compute event per launch) at two CUDA events per
    launch -- a reporting mode, not for headline timing.  ``graph=True``
    replays the pass as a captured CUDA graph (captured on the second call
    with the same plan; inputs and outputs go through engine-owned buffers):
    for launch-bound passes such as the per-step contract on small states.
    Native operator pairs only.
    """
    if nbytes_of(initial_state) != ops.state_size:
        raise SizeMismatch(
            f"initial state is {nbytes_of(initial_state)} bytes, expected {ops.state_size}"
        )
    tier = None
    if isinstance(strategy, Multistage):
        if backend is None:
            raise ValueError("Multistage requires a Level-2 backend")
        interval = _resolve_interval(strategy, ops, backend, initial_state, fuse)
        tier = _tier(backend, ops.state_size)
        code, slots = N.MULTISTAGE, strategy.slots
    elif isinstance(strategy, Revolve):
        code, slots, interval = N.REVOLVE, strategy.slots, 0
    elif isinstance(strategy, FullStorage):
        code, slots, interval = N.FULL_STORAGE, 0, 0
    else:
        raise TypeError(f"unknown strategy {strategy!r}")
    engine, cb = _engine_for(ops)
    if graph and cb is not None:
        raise ValueError("graph=True needs a native operator pair")
    # fusion first (calibrate may have changed it), then re-plan only when the
    # plan changed: a prepare drops a captured graph
    N.check(N.lib.ackpt_engine_set_fusion(engine.handle, 1 if fuse else 0))
    plan_key = (code, slots, interval, tier, int(sample_kernels), bool(timeline), bool(fuse))
    if getattr(engine, "plan_key", None) != plan_key:
        N.check(N.lib.ackpt_engine_set_kernel_sampling(engine.handle, int(sample_kernels)))
        N.check(N.lib.ackpt_engine_set_timeline(engine.handle, 1 if timeline else 0))
        _prepare(engine, code, slots, interval, tier)
        engine.plan_key = plan_key
    N.check(N.lib.ackpt_engine_set_graph(engine.handle, 1 if graph else 0))
    if graph:  # stable buffers: a captured graph holds their addresses
        src = _device_state(initial_state)
        state = engine.stable("in", src)
        state.copy_(src)
        out = engine.stable("out", _output_like(initial_state))
    else:
        state = _device_state(initial_state)
        out = _output_like(initial_state)
    seed_ptr, seed_keep = _seed_ptr(ops, cb)
    st = N.Stats()
    rc = N.lib.ackpt_engine_run(engine.handle, state.data_ptr(), seed_ptr, out.data_ptr(), C.byref(st), _stream())
    if cb is not None:
        cb.raise_pending()
    N.check(rc)
    stats = _stats_from(st)
    if timeline:
        stats.timeline = _timeline(engine)
    return _finish(out.clone() if graph else out, initial_state), stats


def _timeline(engine: _Engine) -> list:
    from .simulator import TimelineEvent

    count = C.c_int64(0)
    N.check(N.lib.ackpt_engine_timeline(engine.handle, None, 0, C.byref(count)))
    buf = (N.TimelineEvent * max(1, count.value))()
    N.check(N.lib.ackpt_engine_timeline(engine.handle, buf, count.value, C.byref(count)))
    return [TimelineEvent(N.EV_KINDS[e.kind], int(e.from_step), int(e.to_step), float(e.start), float(e.end),
                          N.LANES[e.lane]) for e in buf[:count.value]]


def _sweep_engine(plan: MultistagePlan, ops: OperatorPair, backend) -> _Engine:
    if plan.fallback:
        raise ValueError("fallback plans have no Level-2 phase; use execute()")
    engine, cb = _engine_for(ops)
    _prepare(engine, N.MULTISTAGE, plan.s, plan.interval, _tier(backend, ops.state_size))
    engine.plan_key = None  # execute() re-plans
    return engine, cb


def run_forward_sweep(plan: MultistagePlan, ops: OperatorPair, backend, initial_state):
    """Store every boundary state of a non-fallback plan; returns the stored
    keys and the final state (runtime.py:384-399)."""
    engine, cb = _sweep_engine(plan, ops, backend)
    state = _device_state(initial_state)
    final = _output_like(initial_state)
    st = N.Stats()
    rc = N.lib.ackpt_engine_forward_sweep(engine.handle, state.data_ptr(), final.data_ptr(), C.byref(st), _stream())
    if cb is not None:
        cb.raise_pending()
    N.check(rc)
    return list(plan.boundaries), _finish(final, initial_state)


def run_backward_sweep(plan: MultistagePlan, ops: OperatorPair, backend, adjoint_seed):
    """Reverse all intervals from boundary states already in the backend;
    MissingKey propagates for a boundary never stored (runtime.py:402-417)."""
    engine, cb = _sweep_engine(plan, ops, backend)
    seed = _device_state(adjoint_seed)
    if seed.numel() * seed.element_size() != ops.state_size:
        raise SizeMismatch("adjoint seed does not match state_size")
    out = _output_like(adjoint_seed)
    st = N.Stats()
    rc = N.lib.ackpt_engine_backward_sweep(engine.handle, seed.data_ptr(), out.data_ptr(), C.byref(st), _stream())
    if cb is not None:
        cb.raise_pending()
    N.check(rc)
    return _finish(out, adjoint_seed)


def calibrate(ops: OperatorPair, backend, trial_steps: int, initial_state, *, fuse: bool = False) -> tuple:
    """Median (t_a, t_b, t_t) in seconds over trial_steps forward steps,
    backward steps and store round trips, timed with CUDA events
    (runtime.py:420-466).  Keys 0..trial_steps-1 are overwritten.  With
    ``fuse`` t_a is the per-step cost of a fused Advance launch, the rate at
    which a fused forward sweep runs."""
    if trial_steps < 3:
        raise ValueError(f"trial_steps must be >= 3, got {trial_steps}")
    if nbytes_of(initial_state) != ops.state_size:
        raise SizeMismatch("initial state does not match state_size")
    engine, cb = _engine_for(ops)
    N.check(N.lib.ackpt_engine_set_fusion(engine.handle, 1 if fuse else 0))
    tier = _tier(backend, ops.state_size)
    state = _device_state(initial_state)
    t_a, t_b, t_t = C.c_double(), C.c_double(), C.c_double()
    torch.cuda.current_stream().synchronize()
    rc = N.lib.ackpt_engine_calibrate(
        engine.handle, tier, trial_steps, state.data_ptr(), C.byref(t_a), C.byref(t_b), C.byref(t_t)
    )
    if cb is not None:
        cb.raise_pending()
    N.check(rc)
    return t_a.value, t_b.value, t_t.value
