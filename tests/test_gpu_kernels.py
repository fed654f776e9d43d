"""Per-step parity of the sm_100a kernels (K1 forward, K2 adjoint, K3 seed,
K4 loss, fused advance) against the CPU oracle and the reference's golden
steps.  SURVEY §8(c) protocol 1: fp32 rel-L2 <= 1e-5 against the float64
oracle evaluated on the same (fp32-rounded) inputs; the f64 build <= 1e-12.
"""

import numpy as np
import pytest
import torch

from oracle import lstm_oracle as L

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5  # rel-L2, fp32 kernels vs float64 oracle
F64_TOL = 1e-12  # rel-L2, float64 kernels vs reference


@pytest.fixture(scope="module")
def P():
    import paper_1806_01117_b200.lstm as lstm

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return lstm


def _cells(P, d, n, seed):
    return P.random_cell(d, n, seed), L.random_cell(d, n, seed)


def _states(d, seed, batch, scale=1.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, (2, d, batch))


@pytest.mark.parametrize(
    "d,batch",
    # B <= 2048: CTA-per-sequence kernels; above: 4096/4100 float2 kernels
    # (full / partial last tile), 2052/4098 ragged float2 tails, 4101 odd
    # (CTA per sequence), d = 16 / 32 tensor-core tiles (2500, 3000 ragged)
    [(8, 4096), (8, 4100), (8, 516), (8, 2), (8, 1002), (4, 1024), (8, 1001), (5, 64), (16, 300), (32, 17),
     (16, 4096), (32, 1000), (32, 256), (64, 40), (8, 2052), (8, 4098), (8, 4101), (4, 4100), (16, 2500),
     (32, 3000), (64, 3000)],
)
def test_forward_backward_f32_vs_oracle(P, d, batch):
    cell, ocell = _cells(P, d, 6, 11 + d)
    x = _states(d, 3, batch).astype(np.float32)
    a = _states(d, 4, batch).astype(np.float32)
    dc = P.device_cell(cell, batch, "f32")
    for k in (0, 3, 5):
        xt = torch.from_numpy(x).cuda()
        at = torch.from_numpy(a).cuda()
        fwd = dc.forward(k, xt).cpu().numpy()
        bwd = dc.backward(k, xt, at).cpu().numpy()
        ref_f = L.forward_step(ocell, k, x.astype(np.float64))
        ref_b = L.backward_step(ocell, k, x.astype(np.float64), a.astype(np.float64))
        assert L.rel_l2(fwd, ref_f) <= F32_TOL, (k, L.rel_l2(fwd, ref_f))
        assert L.rel_l2(bwd, ref_b) <= F32_TOL, (k, L.rel_l2(bwd, ref_b))
        # every sequence individually, not just the aggregate
        for b in np.linspace(0, batch - 1, min(batch, 16)).astype(int):
            assert L.rel_l2(fwd[:, :, b], ref_f[:, :, b]) <= 2 * F32_TOL
            assert L.rel_l2(bwd[:, :, b], ref_b[:, :, b]) <= 2 * F32_TOL


def test_f32_saturating_inputs(P):
    # large pre-activations exercise the clamped shared-reciprocal path
    d, batch = 8, 512
    cell, ocell = _cells(P, d, 2, 5)
    x = _states(d, 9, batch, scale=60.0).astype(np.float32)
    a = _states(d, 10, batch).astype(np.float32)
    dc = P.device_cell(cell, batch, "f32")
    fwd = dc.forward(1, torch.from_numpy(x).cuda()).cpu().numpy()
    bwd = dc.backward(1, torch.from_numpy(x).cuda(), torch.from_numpy(a).cuda()).cpu().numpy()
    assert np.isfinite(fwd).all() and np.isfinite(bwd).all()
    assert L.rel_l2(fwd, L.forward_step(ocell, 1, x.astype(np.float64))) <= F32_TOL
    assert L.rel_l2(bwd, L.backward_step(ocell, 1, x.astype(np.float64), a.astype(np.float64))) <= F32_TOL


@pytest.mark.parametrize("d,n,seed", [(4, 6, 5), (8, 10, 6), (6, 5, 7), (16, 4, 8), (5, 3, 9)])
def test_f64_steps_match_reference_golden(P, step_golden, d, n, seed):
    cell = P.random_cell(d, n, seed)
    for k in range(n):
        x = step_golden[f"d{d}_s{seed}_k{k}_in"].tobytes()
        a = step_golden[f"d{d}_s{seed}_k{k}_adjin"].tobytes()
        fwd = np.frombuffer(P.lstm_forward_step(cell, k, x), "<f8")
        bwd = np.frombuffer(P.lstm_backward_step(cell, k, x, a), "<f8")
        assert L.rel_l2(fwd, step_golden[f"d{d}_s{seed}_k{k}_fwd"]) <= F64_TOL
        assert L.rel_l2(bwd, step_golden[f"d{d}_s{seed}_k{k}_bwd"]) <= F64_TOL


def test_seed_and_loss(P):
    d, batch = 8, 1000
    cell, ocell = _cells(P, d, 3, 2)
    x = _states(d, 5, batch)
    for dtype, tol in (("f64", 1e-14), ("f32", 1e-6)):
        npdt = np.float64 if dtype == "f64" else np.float32
        xt = torch.from_numpy(x.astype(npdt)).cuda()
        dc = P.device_cell(cell, batch, dtype)
        seed = dc.seed(xt).cpu().numpy()
        assert L.rel_l2(seed, L.seed(ocell, x.astype(npdt).astype(np.float64))) <= tol
        assert (seed[1] == 0).all()
        losses = dc.losses(xt).cpu().numpy()
        assert L.rel_l2(losses, L.loss(ocell, x.astype(npdt).astype(np.float64))) <= tol


@pytest.fixture(params=["ffma2", "tcgen05"])
def family(request, P):
    before = P.kernel_family()
    P.set_kernel_family(request.param)
    yield request.param
    P.set_kernel_family(before)


def _tensor_core_family(P, d, batch, dtype):
    # fused d=8 fp32 forward launches (even batch above the CTA-per-sequence
    # crossover, B > 2048) run on tcgen05 / mma with the 3xTF32 split
    return (P.kernel_family() == "tcgen05" and d == 8 and dtype == "f32" and batch % 2 == 0
            and batch > 2048)


@pytest.mark.parametrize("d,batch,dtype", [(8, 4096, "f32"), (4, 512, "f32"), (8, 7, "f32"), (6, 64, "f64"),
                                           (4, 4100, "f32"), (8, 2306, "f32")])
def test_fused_advance(P, family, d, batch, dtype):
    cell, ocell = _cells(P, d, 12, 21)
    npdt = np.float64 if dtype == "f64" else np.float32
    x = torch.from_numpy(_states(d, 8, batch).astype(npdt)).cuda()
    dc = P.device_cell(cell, batch, dtype)
    fused = dc.advance(2, 11, x)
    if _tensor_core_family(P, d, batch, dtype):
        ref = x.double().cpu().numpy()
        for k in range(2, 11):
            ref = L.forward_step(ocell, k, ref)
        assert L.rel_l2(fused.cpu().numpy(), ref) <= F32_TOL
        # same family: the fused tape's last output is the fused advance, bit for bit
        assert torch.equal(dc.forward_many(2, 9, x)[-1], fused)
    else:
        chain = x
        for k in range(2, 11):
            chain = dc.forward(k, chain)
        assert torch.equal(fused, chain)  # identical arithmetic per step


@pytest.mark.parametrize("d,batch", [(8, 4096), (4, 512), (8, 1002), (8, 300), (8, 2), (8, 258),
                                     (4, 4100), (8, 4098), (8, 2300), (8, 2050), (8, 2306)])
def test_fused_tape_and_reverse(P, family, d, batch):
    cell, ocell = _cells(P, d, 70, 22)
    x = torch.from_numpy(_states(d, 9, batch).astype(np.float32)).cuda()
    a = torch.from_numpy(_states(d, 10, batch).astype(np.float32)).cuda()
    dc = P.device_cell(cell, batch, "f32")
    outs = dc.forward_many(3, 64, x)
    states = [x] + outs[:-1]  # input state of steps 3..66
    fused = dc.backward_many(3, states, a)
    if _tensor_core_family(P, d, batch, "f32"):
        ref = x.double().cpu().numpy()
        for i, k in enumerate(range(3, 67)):
            ref = L.forward_step(ocell, k, ref)
            assert L.rel_l2(outs[i].cpu().numpy(), ref) <= F32_TOL, (k, L.rel_l2(outs[i].cpu().numpy(), ref))
        adj = a.double().cpu().numpy()
        for i, k in reversed(list(enumerate(range(3, 67)))):
            adj = L.backward_step(ocell, k, states[i].double().cpu().numpy(), adj)
        assert L.rel_l2(fused.cpu().numpy(), adj) <= F32_TOL
        assert torch.equal(dc.advance(3, 67, x), outs[-1])
    else:
        chain = x
        for k in range(3, 67):
            chain = dc.forward(k, chain)
            assert torch.equal(outs[k - 3], chain)
        adj = a
        for k in range(66, 2, -1):
            adj = dc.backward(k, states[k - 3], adj)
        assert torch.equal(fused, adj)


def test_c2_shape_kernels_on_sampled_rows(P):
    # BASELINE config 2 shape: d=8, B=2^20 fp32 -> 64 MiB states
    d, batch = 8, 1 << 20
    cell, ocell = _cells(P, d, 4, 0)
    x = P.random_states(d, 1, batch, "f32")
    assert x.numel() * x.element_size() == 64 << 20
    dc = P.device_cell(cell, batch, "f32")
    y = dc.forward(2, x)
    a = dc.seed(y)
    g = dc.backward(2, x, a)
    idx = torch.tensor([0, 1, 2, 3, 12345, batch // 2, batch - 2, batch - 1], device="cuda")
    xs = x[:, :, idx].double().cpu().numpy()
    assert L.rel_l2(y[:, :, idx].cpu().numpy(), L.forward_step(ocell, 2, xs)) <= F32_TOL
    ys = y[:, :, idx].double().cpu().numpy()
    a_ref = L.seed(ocell, ys)
    assert L.rel_l2(g[:, :, idx].cpu().numpy(), L.backward_step(ocell, 2, xs, a_ref)) <= F32_TOL


@pytest.mark.parametrize("d,batch", [(16, 4096), (16, 2178), (32, 2100), (32, 4224), (64, 2200), (64, 4096)])
def test_large_d_tensor_core_fused(P, d, batch):
    # d in {16, 32, 64}, B > 2048 (below, the CTA-per-sequence kernels win):
    # tcgen05 kernels (lstm_f32_tcd.cuh) for the per-step operators and the
    # fused advance / tape / reverse launches (d = 64: forward kernels only,
    # its reverse runs CTA per sequence), full and ragged tiles
    cell, ocell = _cells(P, d, 40, 30 + d)
    x = torch.from_numpy(_states(d, 31, batch).astype(np.float32)).cuda()
    a = torch.from_numpy(_states(d, 32, batch).astype(np.float32)).cuda()
    dc = P.device_cell(cell, batch, "f32")
    ref = x.double().cpu().numpy()
    refs = []
    for k in range(2, 34):
        ref = L.forward_step(ocell, k, ref)
        refs.append(ref)
    adv = dc.advance(2, 34, x).cpu().numpy()
    assert L.rel_l2(adv, refs[-1]) <= F32_TOL, L.rel_l2(adv, refs[-1])
    outs = dc.forward_many(2, 32, x)
    for i in (0, 7, 31):
        assert L.rel_l2(outs[i].cpu().numpy(), refs[i]) <= F32_TOL
    assert torch.equal(outs[-1], dc.advance(2, 34, x))  # same kernel, same bits
    states = [x] + outs[:-1]
    fused = dc.backward_many(2, states, a).cpu().numpy()
    adj = a.double().cpu().numpy()
    for i, k in reversed(list(enumerate(range(2, 34)))):
        adj = L.backward_step(ocell, k, states[i].double().cpu().numpy(), adj)
    assert L.rel_l2(fused, adj) <= F32_TOL, L.rel_l2(fused, adj)
    # the per-step operator chain equals the fused launches bit for bit
    chain = a
    for i, k in reversed(list(enumerate(range(2, 34)))):
        chain = dc.backward(k, states[i], chain)
    assert torch.equal(chain.cpu(), torch.from_numpy(fused))


@pytest.mark.parametrize("d,batch,dtype", [(32, 1, "f64"), (16, 3, "f64"), (5, 37, "f32"), (8, 1, "f32"),
                                           (128, 2, "f64"), (128, 3, "f32"), (96, 2, "f64"), (8, 3000, "f64"),
                                           (24, 2100, "f32"), (32, 64, "f32"), (8, 512, "f32")])
def test_small_batch_kernels(P, d, batch, dtype):
    # one CTA per sequence (lstm_small.cu): every fp32 batch <= 2048 and every
    # shape outside the fp32 fast paths; W in shared memory (padded rows) or,
    # for d = 96 / 128, read from global memory (transposed copy); per-step
    # (programmatic dependent launches) and fused launches, float64 within 1e-12
    cell, ocell = _cells(P, d, 30, 40 + d)
    npdt = np.float64 if dtype == "f64" else np.float32
    tol = 1e-12 if dtype == "f64" else F32_TOL
    x = torch.from_numpy(_states(d, 41, batch).astype(npdt)).cuda()
    a = torch.from_numpy(_states(d, 42, batch).astype(npdt)).cuda()
    dc = P.device_cell(cell, batch, dtype)
    ref = x.double().cpu().numpy()
    refs = []
    for k in range(3, 23):
        ref = L.forward_step(ocell, k, ref)
        refs.append(ref)
    assert L.rel_l2(dc.advance(3, 23, x).cpu().numpy(), refs[-1]) <= tol
    outs = dc.forward_many(3, 20, x)
    assert max(L.rel_l2(o.cpu().numpy(), r) for o, r in zip(outs, refs)) <= tol
    chain = x
    for k in range(3, 23):
        chain = dc.forward(k, chain)
    assert torch.equal(chain, outs[-1])
    states = [x] + outs[:-1]
    adj = a.double().cpu().numpy()
    for i, k in reversed(list(enumerate(range(3, 23)))):
        adj = L.backward_step(ocell, k, states[i].double().cpu().numpy(), adj)
    fused = dc.backward_many(3, states, a)
    assert L.rel_l2(fused.cpu().numpy(), adj) <= tol
    per_step = a
    for i, k in reversed(list(enumerate(range(3, 23)))):
        per_step = dc.backward(k, states[i], per_step)
    assert torch.equal(per_step, fused)


@pytest.mark.parametrize("batch", [1 << 24, (1 << 24) + 6])
def test_c4_per_gpu_shape_on_sampled_rows(P, batch):
    # BASELINE config 4's per-GPU shard (8 GiB over 8 GPUs: d=8, B=2^24 fp32,
    # 1 GiB states) and a ragged variant: 64-bit indexing at scale through the
    # per-step and fused kernels, checked on sampled rows (incl. the last)
    d = 8
    cell, ocell = _cells(P, d, 6, 1)
    x = P.random_states(d, 1, batch, "f32")
    dc = P.device_cell(cell, batch, "f32")
    idx = torch.tensor([0, 1, 777, batch // 3, batch // 2 + 1, batch - 2, batch - 1], device="cuda")
    xs = x[:, :, idx].double().cpu().numpy()
    y = dc.forward(1, x)
    assert L.rel_l2(y[:, :, idx].cpu().numpy(), L.forward_step(ocell, 1, xs)) <= F32_TOL
    a = dc.seed(y)
    g = dc.backward(1, x, a)
    a_s = a[:, :, idx].double().cpu().numpy()
    assert L.rel_l2(g[:, :, idx].cpu().numpy(), L.backward_step(ocell, 1, xs, a_s)) <= F32_TOL
    del g
    outs = dc.forward_many(1, 2, x)
    adv = dc.advance(1, 3, x)
    ref2 = L.forward_step(ocell, 2, L.forward_step(ocell, 1, xs))
    assert L.rel_l2(outs[1][:, :, idx].cpu().numpy(), ref2) <= F32_TOL
    assert torch.equal(outs[1], adv)
    rev = dc.backward_many(1, [x, outs[0]], a)
    want = L.backward_step(ocell, 1, xs, L.backward_step(ocell, 2, outs[0][:, :, idx].double().cpu().numpy(), a_s))
    assert L.rel_l2(rev[:, :, idx].cpu().numpy(), want) <= F32_TOL
