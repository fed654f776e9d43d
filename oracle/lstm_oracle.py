"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference LSTM cell,
batched over independent sequences.

States are arrays of shape (2, d, B) = [h; c] with the batch index fastest
(the product's HBM layout); B=1 float64 is the reference byte image.
Follows pkg/src/asyncckpt/lstm.py:
  _gates              lstm.py:114-120
  lstm_forward_step   lstm.py:123-129
  lstm_backward_step  lstm.py:132-152
  loss / seed         lstm.py:155-163
  random_cell/state   lstm.py:72-96
"""

from __future__ import annotations

import numpy as np


class Cell:
    """Weights of one cell (float64 masters), optionally rounded to dtype."""

    def __init__(self, w, b, xs, target, dtype=np.float64):
        # w: 4 x (d, 2d) in gate order f, i, o, c; b: 4 x (d,)
        self.dtype = np.dtype(dtype)
        self.d = b[0].shape[0]
        self.w = [np.asarray(m, np.float64) for m in w]
        self.b = [np.asarray(v, np.float64) for v in b]
        self.xs = np.asarray(xs, np.float64)
        self.target = np.asarray(target, np.float64)

    @property
    def n_steps(self):
        return self.xs.shape[0]


def random_cell(d: int, n: int, seed: int) -> Cell:
    """Same draws, same order as lstm.py:72-91."""
    rng = np.random.default_rng(seed)
    u = lambda *shape: rng.uniform(-0.1, 0.1, size=shape)  # noqa: E731
    w = [u(d, 2 * d) for _ in range(4)]
    b = [u(d) for _ in range(4)]
    xs = u(n, d)
    target = u(d)
    return Cell(w, b, xs, target)


def long_memory_cell(d: int, n: int, seed: int, forget_bias: float = 5.0) -> Cell:
    """random_cell plus forget_bias on b_f (mirror of the product's
    lstm.long_memory_cell): non-vacuous adjoints at long n."""
    cell = random_cell(d, n, seed)
    cell.b[0] = cell.b[0] + forget_bias
    return cell


def random_states(d: int, seed: int, batch: int) -> np.ndarray:
    """(2, d, B) float64; batch=1 equals random_state(d, seed) (lstm.py:94-96)."""
    rng = np.random.default_rng(seed)
    h = rng.uniform(-0.1, 0.1, (batch, d))
    c = rng.uniform(-0.1, 0.1, (batch, d))
    return np.ascontiguousarray(np.stack([h.T, c.T]))


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def _gates(cell: Cell, h: np.ndarray, k: int, dtype):
    # z = [h; x_k] per sequence; W @ z + b  (lstm.py:114-120).  h: (d, B)
    d = cell.d
    x = cell.xs[k].astype(dtype)[:, None]
    z = np.concatenate([h, np.broadcast_to(x, (d, h.shape[1]))], axis=0)
    pre = [cell.w[g].astype(dtype) @ z + cell.b[g].astype(dtype)[:, None] for g in range(4)]
    return _sigmoid(pre[0]), _sigmoid(pre[1]), _sigmoid(pre[2]), np.tanh(pre[3])


def forward_step(cell: Cell, k: int, state: np.ndarray, dtype=np.float64) -> np.ndarray:
    """state_k (2, d, B) -> state_{k+1}  (lstm.py:123-129)."""
    dtype = np.dtype(dtype)
    h, c = state[0].astype(dtype), state[1].astype(dtype)
    f, i, o, g = _gates(cell, h, k, dtype)
    c2 = f * c + i * g
    h2 = o * np.tanh(c2)
    return np.stack([h2, c2]).astype(dtype)


def backward_step(cell: Cell, k: int, state: np.ndarray, adjoint: np.ndarray, dtype=np.float64):
    """adjoint_{k+1} -> adjoint_k, gates recomputed from state_k (lstm.py:132-152)."""
    dtype = np.dtype(dtype)
    d = cell.d
    h, c = state[0].astype(dtype), state[1].astype(dtype)
    dh_n, dc_n = adjoint[0].astype(dtype), adjoint[1].astype(dtype)
    f, i, o, g = _gates(cell, h, k, dtype)
    c2 = f * c + i * g
    t = np.tanh(c2)
    do = dh_n * t
    dc = dc_n + dh_n * o * (1.0 - t * t)
    da = [dc * c * f * (1.0 - f), dc * g * i * (1.0 - i), do * o * (1.0 - o), dc * i * (1.0 - g * g)]
    dz = sum(cell.w[q].astype(dtype).T @ da[q] for q in range(4))
    return np.stack([dz[:d], dc * f]).astype(dtype)


def loss(cell: Cell, final_state: np.ndarray) -> np.ndarray:
    """Per-sequence sum_j (h_j - target_j)^2 (lstm.py:155-158)."""
    diff = final_state[0] - cell.target[:, None]
    return (diff * diff).sum(axis=0)


def seed(cell: Cell, final_state: np.ndarray) -> np.ndarray:
    """[2 (h - target), 0]  (lstm.py:161-163)."""
    h = final_state[0]
    return np.stack([2.0 * (h - cell.target.astype(h.dtype)[:, None]), np.zeros_like(h)])


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
