import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1806_01117_b200 as pkg, paper_1806_01117_b200.lstm as lstm
from oracle import lstm_oracle as L
for d in (16, 32):
    n, batch = 30, 512
    cell = lstm.random_cell(d, n, 4); dc = lstm.device_cell(cell, batch, "f32")
    x = lstm.random_states(d, 5, batch, "f32"); a = lstm.random_states(d, 6, batch, "f32")
    f1 = dc.forward(3, x); f2 = dc.forward(3, x)
    b1 = dc.backward(3, x, a); b2 = dc.backward(3, x, a)
    oc = L.random_cell(d, n, 4)
    rf = L.forward_step(oc, 3, x.double().cpu().numpy()); rb = L.backward_step(oc, 3, x.double().cpu().numpy(), a.double().cpu().numpy())
    print(d, "fwd det", torch.equal(f1, f2), "bwd det", torch.equal(b1, b2), "fwd err", L.rel_l2(f1.double().cpu().numpy(), rf), "bwd err", L.rel_l2(b1.double().cpu().numpy(), rb))
    adv = dc.advance(3, 10, x); chain = x
    for k in range(3, 10): chain = dc.forward(k, chain)
    print(d, "adv==chain", torch.equal(adv, chain), (adv-chain).abs().max().item())
    ops = lstm.operator_pair(cell, batch, "f32")
    r = [pkg.execute(s, ops, x, fuse=fz)[0] for fz in (False, True) for s in (pkg.FullStorage(), pkg.FullStorage(), pkg.Revolve(5))]
    print(d, [torch.equal(r[0], q) for q in r[:3]], [torch.equal(r[3], q) for q in r[3:]], [(r[0]-q).abs().max().item() for q in r])
