"""TEST INFRASTRUCTURE ONLY: ctypes loader of the C cost-table restatement."""

import ctypes as C
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "librevolve_dp.so")


def available() -> bool:
    return os.path.exists(_LIB)


def cost_table(n_max: int, s_max: int) -> np.ndarray:
    lib = C.CDLL(_LIB)
    out = np.empty((s_max + 1, n_max + 1), dtype=np.int64)
    lib.oracle_cost_table.argtypes = [C.c_int64, C.c_int64, C.c_void_p]
    lib.oracle_cost_table(n_max, s_max, out.ctypes.data)
    return out
