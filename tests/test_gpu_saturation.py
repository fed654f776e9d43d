"""Saturating pre-activations on every batch-tiled fast path (VERDICT r1
item 2).

The fp32 kernels evaluate sigmoid / tanh from pre-scaled exponent arguments
with one shared reciprocal per hidden unit (lstm_f32_math.cuh): the product
of the four 1 + 2^t terms overflows once pre-activations pass ~22, which takes
a separate-reciprocal branch, and the Newton-reciprocal tanh clamps its ex2
argument at 64.  The reference (lstm.py:110-120) saturates exactly through
np.exp / np.tanh.  These tests drive pre-activations to +-60 and beyond +-90
(biases uniform in +-100, weights x4, |h| < 1, |c| up to 60; large weights
would make the trajectory chaotic, amplifying fp32 rounding past any fp32
tolerance in a few steps) at B = 4096 -- above the
CTA-per-sequence crossover (kSbFirstBatch = 2048), so dispatch reaches:

* d = 4 / 8 per-step K1 / K2 (packed FFMA2, lstm_f32.cuh),
* d = 8 fused advance / tape / reverse of both families (tcgen05 3xTF32,
  lstm_f32_tc.cuh; FFMA2 fallback),
* d = 16 / 32 / 64 tensor-core kernels (lstm_f32_tcd.cuh), per step and fused,

and compare every sampled sequence with the float64 oracle (rel-L2 <= 1e-5,
2e-5 per sequence like test_gpu_kernels.py).
"""

import numpy as np
import pytest
import torch

from oracle import lstm_oracle as L

pytestmark = pytest.mark.gpu

TOL = 1e-5
WSCALE = 4.0
BIAS = 100.0
BATCH = 4096


@pytest.fixture(scope="module")
def P():
    import paper_1806_01117_b200.lstm as lstm

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return lstm


def _scaled_cells(P, d, n, seed):
    cell, ocell = P.random_cell(d, n, seed), L.random_cell(d, n, seed)
    rng = np.random.default_rng(seed + 1000)
    biases = [rng.uniform(-BIAS, BIAS, d) for _ in range(4)]
    for name in ("w_f", "w_i", "w_o", "w_c"):
        setattr(cell, name, getattr(cell, name) * WSCALE)
    for name, b in zip(("b_f", "b_i", "b_o", "b_c"), biases):
        setattr(cell, name, b.copy())
    ocell.w = [w * WSCALE for w in ocell.w]
    ocell.b = [b.copy() for b in biases]
    return cell, ocell


def _states(d, seed, hscale=1.0, cscale=60.0):
    rng = np.random.default_rng(seed)
    return np.stack([rng.uniform(-hscale, hscale, (d, BATCH)), rng.uniform(-cscale, cscale, (d, BATCH))])


def _preact_range(ocell, k, x):
    d = ocell.d
    z = np.concatenate([x[0], np.broadcast_to(ocell.xs[k][:, None], (d, x.shape[2]))])
    return max(np.abs(ocell.w[g] @ z + ocell.b[g][:, None]).max() for g in range(4))


def _check(got, ref, what):
    assert np.isfinite(got).all(), what
    assert L.rel_l2(got, ref) <= TOL, (what, L.rel_l2(got, ref))
    for b in np.linspace(0, BATCH - 1, 64).astype(int):
        assert L.rel_l2(got[:, :, b], ref[:, :, b]) <= 2 * TOL, (what, b, L.rel_l2(got[:, :, b], ref[:, :, b]))


@pytest.fixture(params=["tcgen05", "ffma2"])
def family(request, P):
    before = P.kernel_family()
    P.set_kernel_family(request.param)
    yield request.param
    P.set_kernel_family(before)


@pytest.mark.parametrize("d", [4, 8, 16, 32, 64])
def test_per_step_saturating(P, d):
    cell, ocell = _scaled_cells(P, d, 4, 21 + d)
    x = _states(d, 5).astype(np.float32).astype(np.float64)
    a = _states(d, 6, 1.0, 1.0).astype(np.float32).astype(np.float64)
    assert _preact_range(ocell, 2, x) > 90  # beyond the shared-reciprocal overflow and the ex2 clamp
    dc = P.device_cell(cell, BATCH, "f32")
    xt, at = torch.from_numpy(x).float().cuda(), torch.from_numpy(a).float().cuda()
    _check(dc.forward(2, xt).cpu().numpy(), L.forward_step(ocell, 2, x), f"fwd d={d}")
    _check(dc.backward(2, xt, at).cpu().numpy(), L.backward_step(ocell, 2, x, a), f"bwd d={d}")


def test_fused_d8_saturating(P, family):
    d, n = 8, 12
    cell, ocell = _scaled_cells(P, d, n, 40)
    x = _states(d, 7).astype(np.float32).astype(np.float64)
    dc = P.device_cell(cell, BATCH, "f32")
    xt = torch.from_numpy(x).float().cuda()
    # advance / tape: the forward trajectory from a saturated start
    refs, ref = [], x
    for k in range(n):
        ref = L.forward_step(ocell, k, ref)
        refs.append(ref)
    _check(dc.advance(0, n, xt).cpu().numpy(), refs[-1], f"advance {family}")
    outs = dc.forward_many(0, n, xt)
    for k in (0, n // 2, n - 1):
        _check(outs[k].cpu().numpy(), refs[k], f"tape {family} step {k}")
    # reverse over states with saturating pre-activations at every step
    states = [_states(d, 100 + k).astype(np.float32).astype(np.float64) for k in range(n)]
    adj0 = _states(d, 99, 1.0, 1.0).astype(np.float32).astype(np.float64)
    ref_a = adj0
    for k in range(n - 1, -1, -1):
        ref_a = L.backward_step(ocell, k, states[k], ref_a)
    got = dc.backward_many(0, [torch.from_numpy(s).float().cuda() for s in states],
                           torch.from_numpy(adj0).float().cuda()).cpu().numpy()
    _check(got, ref_a, f"reverse {family}")


@pytest.mark.parametrize("d", [16, 32, 64])
def test_fused_large_d_saturating(P, d):
    n = 6
    cell, ocell = _scaled_cells(P, d, n, 50 + d)
    dc = P.device_cell(cell, BATCH, "f32")
    x = _states(d, 8).astype(np.float32).astype(np.float64)
    xt = torch.from_numpy(x).float().cuda()
    refs, ref = [], x
    for k in range(n):
        ref = L.forward_step(ocell, k, ref)
        refs.append(ref)
    _check(dc.advance(0, n, xt).cpu().numpy(), refs[-1], f"advance d={d}")
    outs = dc.forward_many(0, n, xt)
    _check(outs[n - 1].cpu().numpy(), refs[n - 1], f"tape d={d}")
    states = [_states(d, 200 + k).astype(np.float32).astype(np.float64) for k in range(n)]
    adj0 = _states(d, 199, 1.0, 1.0).astype(np.float32).astype(np.float64)
    ref_a = adj0
    for k in range(n - 1, -1, -1):
        ref_a = L.backward_step(ocell, k, states[k], ref_a)
    got = dc.backward_many(0, [torch.from_numpy(s).float().cuda() for s in states],
                           torch.from_numpy(adj0).float().cuda()).cpu().numpy()
    _check(got, ref_a, f"reverse d={d}")
