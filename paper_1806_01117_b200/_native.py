"""ctypes binding of libackpt.so, the C ABI declared in include/ackpt.h.

There is no fallback: if the shared library is missing the import fails
loudly (build it with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_1806_01117_b200/csrc``).  ctypes.CDLL releases the GIL for
the duration of every foreign call.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libackpt.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libackpt.so not found at {LIB_PATH}: build the CUDA extension first "
        "(make -C paper_1806_01117_b200/csrc); there is no CPU fallback"
    )

lib = C.CDLL(LIB_PATH)

# ---- status codes (include/ackpt.h) ----
OK = 0
INFEASIBLE_SCHEDULE = 1
SIZE_MISMATCH = 2
SLOT_OUT_OF_RANGE = 3
SLOT_UNWRITTEN = 4
MISSING_KEY = 5
CHECKSUM_MISMATCH = 6
STORAGE_FULL = 7
EXECUTION_ERROR = 8
VALUE_ERROR = 9
CUDA_ERROR = 10
NOT_READY = 11

_EXC = {
    INFEASIBLE_SCHEDULE: errors.InfeasibleSchedule,
    SIZE_MISMATCH: errors.SizeMismatch,
    SLOT_OUT_OF_RANGE: errors.SlotOutOfRange,
    SLOT_UNWRITTEN: errors.SlotUnwritten,
    MISSING_KEY: errors.MissingKey,
    CHECKSUM_MISMATCH: errors.ChecksumMismatch,
    STORAGE_FULL: errors.StorageFull,
    EXECUTION_ERROR: errors.ExecutionError,
    VALUE_ERROR: ValueError,
    CUDA_ERROR: errors.ExecutionError,
}

# ---- action ops ----
ADVANCE, SAVE, LOAD, TAPE, REVERSE, DONE = range(6)
F32, F64 = 0, 1
FULL_STORAGE, REVOLVE, MULTISTAGE = 0, 1, 2


class Action(C.Structure):
    _fields_ = [("op", C.c_int32), ("reserved", C.c_int32), ("a", C.c_int64), ("b", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [
        ("forward_evals", C.c_int64),
        ("backward_evals", C.c_int64),
        ("stores_issued", C.c_int64),
        ("prefetches_issued", C.c_int64),
        ("stall_seconds", C.c_double),
        ("peak_l1_bytes", C.c_int64),
        ("wall_seconds", C.c_double),
        ("gpu_seconds", C.c_double),
        ("kernel_launches", C.c_int64),
        ("interval", C.c_int64),
        ("fallback", C.c_int64),
        ("device_buffers", C.c_int64),
        ("link_bytes", C.c_int64),
        ("fused_advances", C.c_int64),
        ("fwd_sample_seconds", C.c_double),
        ("fwd_samples", C.c_int64),
        ("bwd_sample_seconds", C.c_double),
        ("bwd_samples", C.c_int64),
        ("host_enqueue_seconds", C.c_double),
    ]


class CascadeStats(C.Structure):
    _fields_ = [("dram_slots", C.c_int64), ("spills", C.c_int64), ("spill_bytes", C.c_int64),
                ("spill_seconds", C.c_double), ("reads", C.c_int64), ("read_bytes", C.c_int64),
                ("read_seconds", C.c_double), ("dram_hits", C.c_int64), ("ring_hits", C.c_int64),
                ("ring_misses", C.c_int64)]


class TimelineEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lane", C.c_int32), ("from_step", C.c_int64), ("to_step", C.c_int64),
                ("start", C.c_double), ("end", C.c_double)]


EV_KINDS = ("forward_compute", "backward_compute", "store", "fetch", "stall")
LANES = ("compute", "transfer")

FORWARD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p)
BACKWARD_FN = C.CFUNCTYPE(
    C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p
)
SEED_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
ADVANCE_FN = C.CFUNCTYPE(
    C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p
)


FORWARD_MANY_FN = C.CFUNCTYPE(
    C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p
)
BACKWARD_MANY_FN = C.CFUNCTYPE(
    C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p, C.c_void_p
)
MAX_FUSED = 64


class Operator(C.Structure):
    _fields_ = [
        ("ctx", C.c_void_p),
        ("forward", FORWARD_FN),
        ("backward", BACKWARD_FN),
        ("seed", SEED_FN),
        ("advance", ADVANCE_FN),
        ("state_bytes", C.c_int64),
        ("n_steps", C.c_int64),
        ("forward_many", FORWARD_MANY_FN),
        ("backward_many", BACKWARD_MANY_FN),
    ]


_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

_SIGS = {
    "ackpt_last_error": ([], C.c_char_p),
    "ackpt_version": ([], C.c_char_p),
    "ackpt_forward_cost": ([C.c_int64, C.c_int64, _i64p], C.c_int),
    "ackpt_best_split": ([C.c_int64, C.c_int64, _i64p], C.c_int),
    "ackpt_revolve_schedule": ([C.c_int64, C.c_int64, C.POINTER(Action), C.c_int64, _i64p], C.c_int),
    "ackpt_taped_schedule": ([C.c_int64, C.POINTER(Action), C.c_int64, _i64p], C.c_int),
    "ackpt_interval_length": ([C.c_double, C.c_double, _i64p], C.c_int),
    "ackpt_set_schedule_threads": ([C.c_int32], C.c_int),
    "ackpt_lstm_create": (
        [C.c_int32, C.c_int64, C.c_int64, C.c_int32] + [_dp] * 10 + [C.POINTER(_vp)],
        C.c_int,
    ),
    "ackpt_lstm_destroy": ([_vp], C.c_int),
    "ackpt_lstm_state_bytes": ([_vp], C.c_int64),
    "ackpt_lstm_forward": ([_vp, C.c_int64, _vp, _vp, _vp], C.c_int),
    "ackpt_lstm_advance": ([_vp, C.c_int64, C.c_int64, _vp, _vp, _vp], C.c_int),
    "ackpt_lstm_backward": ([_vp, C.c_int64, _vp, _vp, _vp, _vp], C.c_int),
    "ackpt_lstm_forward_many": ([_vp, C.c_int64, C.c_int64, _vp, C.POINTER(_vp), _vp], C.c_int),
    "ackpt_lstm_backward_many": ([_vp, C.c_int64, C.c_int64, C.POINTER(_vp), _vp, _vp, _vp], C.c_int),
    "ackpt_lstm_seed": ([_vp, _vp, _vp, _vp], C.c_int),
    "ackpt_lstm_loss": ([_vp, _vp, _vp, _vp], C.c_int),
    "ackpt_lstm_operator": ([_vp, C.POINTER(Operator)], C.c_int),
    "ackpt_set_fused_family": ([C.c_int32], C.c_int),
    "ackpt_get_fused_family": ([], C.c_int32),
    "ackpt_pad_operator_create": ([C.POINTER(Operator), C.c_double, C.c_double, C.POINTER(Operator)], C.c_int),
    "ackpt_pad_operator_destroy": ([C.POINTER(Operator)], C.c_int),
    "ackpt_tier_create": ([C.c_int64, C.c_int64, C.POINTER(_vp)], C.c_int),
    "ackpt_tier_create_file": ([C.c_char_p, C.c_int64, C.POINTER(_vp)], C.c_int),
    "ackpt_tier_create_cascade": ([C.c_char_p, C.c_int64, C.c_int32, C.POINTER(_vp)], C.c_int),
    "ackpt_tier_cascade_stats": ([_vp, C.POINTER(CascadeStats)], C.c_int),
    "ackpt_tier_destroy": ([_vp], C.c_int),
    "ackpt_tier_set_throttle": ([_vp, C.c_double, C.c_double], C.c_int),
    "ackpt_tier_begin_store": ([_vp, C.c_int64, C.c_int64, _vp, C.c_int64, _vp, _i64p], C.c_int),
    "ackpt_tier_begin_fetch": ([_vp, C.c_int64, _vp, C.c_int64, _vp, _i64p], C.c_int),
    "ackpt_tier_wait": ([_vp, C.c_int64, _i64p], C.c_int),
    "ackpt_tier_streams": ([_vp, C.POINTER(_vp), C.POINTER(_vp)], C.c_int),
    "ackpt_tier_stream_wait": ([_vp, C.c_int64, _vp], C.c_int),
    "ackpt_tier_poll": ([_vp, C.c_int64], C.c_int),
    "ackpt_tier_contains": ([_vp, C.c_int64, C.POINTER(C.c_int32)], C.c_int),
    "ackpt_tier_key_bytes": ([_vp, C.c_int64, _i64p], C.c_int),
    "ackpt_tier_host_ptr": ([_vp, C.c_int64, C.POINTER(_vp)], C.c_int),
    "ackpt_tier_clear": ([_vp], C.c_int),
    "ackpt_engine_create": ([C.POINTER(Operator), C.POINTER(_vp)], C.c_int),
    "ackpt_engine_destroy": ([_vp], C.c_int),
    "ackpt_engine_prepare": ([_vp, C.c_int32, C.c_int64, C.c_int64, _vp], C.c_int),
    "ackpt_engine_set_fusion": ([_vp, C.c_int32], C.c_int),
    "ackpt_engine_set_prefetch": ([_vp, C.c_int32], C.c_int),
    "ackpt_engine_set_kernel_sampling": ([_vp, C.c_int64], C.c_int),
    "ackpt_engine_run": ([_vp, _vp, _vp, _vp, C.POINTER(Stats), _vp], C.c_int),
    "ackpt_engine_forward_sweep": ([_vp, _vp, _vp, C.POINTER(Stats), _vp], C.c_int),
    "ackpt_engine_backward_sweep": ([_vp, _vp, _vp, C.POINTER(Stats), _vp], C.c_int),
    "ackpt_engine_calibrate": ([_vp, _vp, C.c_int64, _vp, _dp, _dp, _dp], C.c_int),
    "ackpt_engine_interval": ([_vp], C.c_int64),
    "ackpt_engine_set_timeline": ([_vp, C.c_int32], C.c_int),
    "ackpt_engine_set_graph": ([_vp, C.c_int32], C.c_int),
    "ackpt_engine_timeline": ([_vp, C.POINTER(TimelineEvent), C.c_int64, _i64p], C.c_int),
    "ackpt_crc32c": ([_vp, C.c_int64, C.c_uint32], C.c_uint32),
    "ackpt_chain_selftest": ([], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    msg = lib.ackpt_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int) -> None:
    """Raise the Python exception mirroring a non-OK status (errors.py)."""
    if rc != OK:
        raise _EXC.get(rc, errors.ExecutionError)(last_error())
