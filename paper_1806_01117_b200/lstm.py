"""LSTM benchmark operator on the GPU: the reference cell (lstm.py) with an
added batch axis of independent sequences sharing the weights.

Reference: pkg/src/asyncckpt/lstm.py.  Gates f, i, o = sigmoid(W [h; x] + b),
g = tanh(W_c [h; x] + b_c); c' = f c + i g; h' = o tanh(c'); loss = sum (h_n -
target)^2; the backward step is the exact state adjoint (lstm.py:132-152).

Device state layout (include/ackpt.h): a tensor of shape (2, d, B) holding
[h; c] with the batch index fastest, dtype float32 or float64.  For B=1 and
float64 its bytes are exactly the reference's state image [h(d), c(d)]
little-endian f64 (lstm.py:99-107), so ``bytes`` states work unchanged.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import tempfile
from dataclasses import asdict, dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .runtime import (
    ExecutionStats,
    FullStorage,
    Multistage,
    OperatorPair,
    Revolve,
    Strategy,
    execute,
)
from .storage import FileBackend, Level2Backend, PinnedHostBackend, SimulatedBackend, as_host_bytes

_F8 = np.dtype("<f8")

_DTYPES = {
    "f32": torch.float32,
    "float32": torch.float32,
    torch.float32: torch.float32,
    "f64": torch.float64,
    "float64": torch.float64,
    torch.float64: torch.float64,
}


def _torch_dtype(dtype) -> torch.dtype:
    try:
        return _DTYPES[dtype]
    except KeyError:
        raise ValueError(f"dtype must be float32 or float64, got {dtype!r}") from None


@dataclass
class LstmCell:
    """Weights (d x 2d acting on [h; x]), biases, the input sequence xs (n, d)
    and the loss target (d,), float64 like the reference (lstm.py:39-69)."""

    w_f: np.ndarray
    w_i: np.ndarray
    w_o: np.ndarray
    w_c: np.ndarray
    b_f: np.ndarray
    b_i: np.ndarray
    b_o: np.ndarray
    b_c: np.ndarray
    xs: np.ndarray
    target: np.ndarray
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def hidden_size(self) -> int:
        return self.b_f.shape[0]

    @property
    def n_steps(self) -> int:
        return self.xs.shape[0]

    @property
    def state_size(self) -> int:
        """Bytes of one reference state (B=1, float64)."""
        return 2 * self.hidden_size * 8

    def state_bytes(self, batch: int = 1, dtype="f64") -> int:
        return 2 * self.hidden_size * batch * torch.empty((), dtype=_torch_dtype(dtype)).element_size()


def random_cell(d: int, n: int, seed: int) -> LstmCell:
    """Reproducible cell: every array uniform in [-0.1, 0.1) from
    default_rng(seed), drawn in the reference's order (lstm.py:72-91)."""
    rng = np.random.default_rng(seed)
    draw = lambda *shape: rng.uniform(-0.1, 0.1, size=shape)  # noqa: E731
    w = [draw(d, 2 * d) for _ in range(4)]
    b = [draw(d) for _ in range(4)]
    xs = draw(n, d)
    return LstmCell(*w, *b, xs=xs, target=draw(d))


def long_memory_cell(d: int, n: int, seed: int, forget_bias: float = 5.0) -> LstmCell:
    """random_cell(d, n, seed) with ``forget_bias`` added to b_f: the forget
    gate sits near 1 (sigmoid(5) = 0.993), so the state adjoint stays far above
    fp32 underflow at n = 10^4 (d = 8, seed 0: per-sequence norms 8e-4 ..
    1.8e-3), where the reference cell's adjoint is exactly 0 past n ~ 190.
    The chain is well conditioned (a 1-ulp fp32 perturbation of the weights
    moves the float64 adjoint by 2e-6 rel-L2; bias 6 has rows 30x more
    sensitive).  Same timing as random_cell; the workload of the long-chain
    parity checks (tests, bench.py's parity leg)."""
    cell = random_cell(d, n, seed)
    cell.b_f = cell.b_f + forget_bias
    return cell


def pack_state(h: np.ndarray, c: np.ndarray) -> bytes:
    """Reference byte image [h, c] as little-endian float64 (lstm.py:99-100)."""
    return np.ascontiguousarray(np.concatenate([h, c]), dtype=_F8).tobytes()


def unpack_state(state, d: int):
    flat = np.frombuffer(as_host_bytes(state), dtype=_F8)
    if flat.shape[0] != 2 * d:
        raise ValueError(f"state holds {flat.shape[0]} floats, expected {2 * d}")
    return flat[:d].copy(), flat[d:].copy()


def random_state(d: int, seed: int) -> bytes:
    """Reference initial state (B=1, float64 bytes; lstm.py:94-96)."""
    rng = np.random.default_rng(seed)
    return pack_state(rng.uniform(-0.1, 0.1, d), rng.uniform(-0.1, 0.1, d))


def random_states(d: int, seed: int, batch: int, dtype="f32", device="cuda") -> torch.Tensor:
    """Batched initial states, shape (2, d, batch): h then c drawn as
    uniform(-0.1, 0.1, (batch, d)) from default_rng(seed).  Row b equals
    random_state(d, seed) for batch == 1."""
    rng = np.random.default_rng(seed)
    h = rng.uniform(-0.1, 0.1, (batch, d))
    c = rng.uniform(-0.1, 0.1, (batch, d))
    host = np.stack([h.T, c.T])  # (2, d, B), batch fastest
    return torch.from_numpy(np.ascontiguousarray(host)).to(device=device, dtype=_torch_dtype(dtype))


class DeviceCell:
    """The cell uploaded to the GPU for one (batch, dtype): native ackpt_lstm."""

    def __init__(self, cell: LstmCell, batch: int, dtype):
        # no reference back to `cell`: the cell caches this object (cell._device),
        # and a cycle would keep the engine's HBM pool alive until a GC round
        self.n_steps = cell.n_steps
        self.batch = int(batch)
        self.dtype = _torch_dtype(dtype)
        self.d = cell.hidden_size
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (
            cell.w_f, cell.w_i, cell.w_o, cell.w_c, cell.b_f, cell.b_i, cell.b_o, cell.b_c, cell.xs, cell.target)]
        ptrs = [a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs]
        h = C.c_void_p()
        code = N.F32 if self.dtype == torch.float32 else N.F64
        N.check(N.lib.ackpt_lstm_create(self.d, cell.n_steps, self.batch, code, *ptrs, C.byref(h)))
        self.handle = h.value
        self.state_bytes = int(N.lib.ackpt_lstm_state_bytes(self.handle))
        self._op = None

    def operator(self) -> N.Operator:
        if self._op is None:
            op = N.Operator()
            N.check(N.lib.ackpt_lstm_operator(self.handle, C.byref(op)))
            self._op = op
        return self._op

    def __del__(self):
        try:
            if getattr(self, "_engine", None) is not None:
                self._engine = None
            if self.handle:
                N.lib.ackpt_lstm_destroy(self.handle)
        except Exception:
            pass

    # -- single calls -------------------------------------------------------
    def _tensor(self, state) -> torch.Tensor:
        if isinstance(state, torch.Tensor):
            t = state.detach()
            t = t if t.is_cuda else t.cuda()
            t = t.contiguous()
            if t.numel() * t.element_size() != self.state_bytes:
                raise ValueError("state tensor does not match the cell's state size")
            return t.view(self.dtype).reshape(2, self.d, self.batch)
        raw = torch.frombuffer(bytearray(state), dtype=self.dtype)
        if raw.numel() * raw.element_size() != self.state_bytes:
            raise ValueError("state bytes do not match the cell's state size")
        return raw.reshape(2, self.d, self.batch).cuda()

    def forward(self, step: int, state) -> torch.Tensor:
        x = self._tensor(state)
        out = torch.empty_like(x)
        N.check(N.lib.ackpt_lstm_forward(self.handle, step, x.data_ptr(), out.data_ptr(), _stream()))
        return out

    def advance(self, from_step: int, to_step: int, state) -> torch.Tensor:
        x = self._tensor(state)
        out = torch.empty_like(x)
        N.check(N.lib.ackpt_lstm_advance(self.handle, from_step, to_step, x.data_ptr(), out.data_ptr(), _stream()))
        return out

    def forward_many(self, from_step: int, count: int, state) -> list:
        """Fused TapeForward: the states after steps from_step .. from_step+count-1."""
        x = self._tensor(state)
        outs = [torch.empty_like(x) for _ in range(count)]
        ptrs = (C.c_void_p * count)(*[o.data_ptr() for o in outs])
        N.check(N.lib.ackpt_lstm_forward_many(self.handle, from_step, count, x.data_ptr(), ptrs, _stream()))
        return outs

    def backward_many(self, from_step: int, states: list, adjoint) -> torch.Tensor:
        """Fused Reverse run over steps from_step+len(states)-1 .. from_step;
        states[i] is the state of step from_step+i."""
        xs = [self._tensor(s) for s in states]
        a = self._tensor(adjoint)
        out = torch.empty_like(a)
        ptrs = (C.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
        N.check(N.lib.ackpt_lstm_backward_many(self.handle, from_step, len(xs), ptrs, a.data_ptr(),
                                               out.data_ptr(), _stream()))
        return out

    def backward(self, step: int, state, adjoint) -> torch.Tensor:
        x = self._tensor(state)
        a = self._tensor(adjoint)
        out = torch.empty_like(x)
        N.check(N.lib.ackpt_lstm_backward(self.handle, step, x.data_ptr(), a.data_ptr(), out.data_ptr(), _stream()))
        return out

    def seed(self, final_state) -> torch.Tensor:
        x = self._tensor(final_state)
        out = torch.empty_like(x)
        N.check(N.lib.ackpt_lstm_seed(self.handle, x.data_ptr(), out.data_ptr(), _stream()))
        return out

    def losses(self, final_state) -> torch.Tensor:
        x = self._tensor(final_state)
        out = torch.empty(self.batch, dtype=self.dtype, device=x.device)
        N.check(N.lib.ackpt_lstm_loss(self.handle, x.data_ptr(), out.data_ptr(), _stream()))
        return out


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def set_kernel_family(name: str) -> None:
    """Kernel family of the fused d=8 fp32 launches: "tcgen05" (default:
    tensor cores, 3xTF32 gate products) or "ffma2" (packed fp32 FMA, the
    documented fallback).  Both meet the fp32 tolerance; they round
    differently, so switch only between executions."""
    N.check(N.lib.ackpt_set_fused_family(KERNEL_FAMILIES.index(name)))


KERNEL_FAMILIES = ("ffma2", "tcgen05")


def kernel_family() -> str:
    return KERNEL_FAMILIES[N.lib.ackpt_get_fused_family()]


def device_cell(cell: LstmCell, batch: int = 1, dtype="f64") -> DeviceCell:
    key = (int(batch), _torch_dtype(dtype))
    dc = cell._device.get(key)
    if dc is None:
        dc = DeviceCell(cell, batch, dtype)
        cell._device[key] = dc
    return dc


def _like(result: torch.Tensor, like):
    if isinstance(like, torch.Tensor):
        return result.view(like.dtype).reshape(like.shape) if result.dtype != like.dtype else result.reshape(like.shape)
    return as_host_bytes(result)


def _infer(cell: LstmCell, state) -> DeviceCell:
    """Device cell matching a state: tensors carry (2, d, B) and dtype; bytes are B=1 f64."""
    if isinstance(state, torch.Tensor) and state.dtype in (torch.float32, torch.float64):
        batch = state.numel() // (2 * cell.hidden_size)
        return device_cell(cell, batch, state.dtype)
    return device_cell(cell, 1, "f64")


def lstm_forward_step(cell: LstmCell, step: int, state):
    """state_k -> state_{k+1} on the GPU (lstm.py:123-129)."""
    return _like(_infer(cell, state).forward(step, state), state)


def lstm_backward_step(cell: LstmCell, step: int, state, adjoint):
    """adjoint_{k+1} -> adjoint_k, gates recomputed from state_k (lstm.py:132-152)."""
    return _like(_infer(cell, state).backward(step, state, adjoint), state)


def loss(cell: LstmCell, final_state) -> float:
    """Sum over the batch of sum_j (h_j - target_j)^2 (lstm.py:155-158)."""
    return float(_infer(cell, final_state).losses(final_state).double().sum().item())


def loss_gradient_seed(cell: LstmCell, final_state):
    """[2 (h - target), 0] (lstm.py:161-163)."""
    return _like(_infer(cell, final_state).seed(final_state), final_state)


def operator_pair(cell: LstmCell, batch: int = 1, dtype="f64") -> OperatorPair:
    """Operator pair over (2, d, batch) device states; the executor runs its
    native step kernels without Python in the loop."""
    dc = device_cell(cell, batch, dtype)
    return OperatorPair(
        forward_step=lambda k, s: _like(dc.forward(k, s), s),
        backward_step=lambda k, s, a: _like(dc.backward(k, s, a), s),
        state_size=dc.state_bytes,
        n_steps=cell.n_steps,
        adjoint_seed=lambda final: _like(dc.seed(final), final),
        native=dc,
    )


@dataclass
class BenchReport:
    n: int
    strategy: str
    wall_seconds: float
    forward_evals: int
    recompute_factor_measured: float
    peak_l1_bytes: int
    stall_seconds: float
    gradient_checksum: str

    def to_json(self) -> str:
        return json.dumps(asdict(self))


def _strategy_label(strategy: Strategy) -> str:
    for kind, label in ((FullStorage, "full"), (Revolve, "revolve"), (Multistage, "multistage")):
        if isinstance(strategy, kind):
            return label
    raise TypeError(f"unknown strategy {strategy!r}")


def make_backend(config: Optional[dict], slot_bytes: Optional[int] = None) -> Optional[Level2Backend]:
    """{"kind": "sim", "bandwidth", "latency"} -> throttled pinned tier;
    {"kind": "pinned"} -> PinnedHostBackend; {"kind": "file", "dir"} ->
    FileBackend; None -> no backend (lstm.py:201-216)."""
    if config is None:
        return None
    kind = config["kind"]
    if kind == "sim":
        return SimulatedBackend(
            bandwidth=config.get("bandwidth", 1e9), latency=config.get("latency", 0.0), slot_bytes=slot_bytes
        )
    if kind == "pinned":
        return PinnedHostBackend(slot_bytes=slot_bytes)
    if kind == "file":
        return FileBackend(config.get("dir") or tempfile.mkdtemp(prefix="ckpt_"), slot_bytes=slot_bytes)
    raise ValueError(f"unknown backend kind {kind!r}")


def bench(
    strategy: Strategy,
    n: int,
    d: int,
    s: int,
    backend_config: Optional[dict] = None,
    seed: int = 0,
    runs: int = 5,
    batch: int = 1,
    dtype="f64",
    fuse: bool = False,
    timeline_path: Optional[str] = None,
    graph: bool = False,
) -> BenchReport:
    """One forward/backward iteration timed as the minimum over ``runs``
    (lstm.py:219-254); batch=1/f64 reproduces the reference's workload.
    ``timeline_path``: also write the fastest run's measured event timeline
    there (simulator JSON format; total = the compute stream's time).
    ``graph``: replay the pass as a captured CUDA graph (runtime.execute)."""
    cell = random_cell(d, n, seed)
    ops = operator_pair(cell, batch, dtype)
    if batch == 1 and _torch_dtype(dtype) == torch.float64:
        state0 = random_state(d, seed + 1)
    else:
        state0 = random_states(d, seed + 1, batch, dtype)
    backend = make_backend(backend_config, ops.state_size)
    try:
        best: Optional[ExecutionStats] = None
        adjoint = b""
        for _ in range(max(1, runs)):
            adjoint, stats = execute(strategy, ops, state0, backend, fuse=fuse, timeline=timeline_path is not None,
                                    graph=graph)
            if best is None or stats.wall_seconds < best.wall_seconds:
                best = stats
        if timeline_path is not None:
            from .simulator import timeline_to_json

            with open(timeline_path, "w") as fh:
                fh.write(timeline_to_json(strategy, best.timeline, best.device["gpu_seconds"]))
        return BenchReport(
            n=n,
            strategy=_strategy_label(strategy),
            wall_seconds=best.wall_seconds,
            forward_evals=best.forward_evals,
            recompute_factor_measured=best.forward_evals / n,
            peak_l1_bytes=best.peak_l1_bytes,
            stall_seconds=best.stall_seconds,
            gradient_checksum=hashlib.sha256(as_host_bytes(adjoint)).hexdigest(),
        )
    finally:
        if backend is not None:
            backend.close()
