"""HBM write-only vs read-only vs copy bandwidth on the box (CUDA events,
best of 10): the tape kernel writes 64 MiB per step and reads almost
nothing, so its HBM ceiling is the write-only rate, not the copy rate."""
import json
import torch

n = 1 << 30  # floats: 4 GiB
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) * 1e-3)
    return min(t)


a.fill_(1.0)
res = {
    "write_gbs": 4 * n / best(lambda: a.fill_(2.0)) / 1e9,
    "read_gbs": 4 * n / best(lambda: a.sum()) / 1e9,
    "copy_gbs (read+write)": 8 * n / best(lambda: b.copy_(a)) / 1e9,
}
print(json.dumps(res))
