import sys
import torch
sys.path.insert(0, '.')
import paper_1806_01117_b200.lstm as lstm
from oracle import lstm_oracle as L
d = int(sys.argv[1]); batch = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cell = lstm.random_cell(d, 30, 4); dc = lstm.device_cell(cell, batch, "f32")
x = lstm.random_states(d, 5, batch, "f32")
oc = L.random_cell(d, 30, 4)
rf = L.forward_step(oc, 3, x.double().cpu().numpy())
for r in range(reps):
    f = dc.forward(3, x)
    torch.cuda.synchronize()
    e = L.rel_l2(f.double().cpu().numpy(), rf)
    bad = (abs(f.double().cpu().numpy() - rf) > 1e-4).any(axis=(0, 1)).nonzero()[0]
    print(d, batch, r, f"{e:.3e}", "bad seqs", bad[:10], len(bad))
