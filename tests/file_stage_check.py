"""Run by tests/test_gpu_variants.py in a subprocess (the file-stage path is
chosen once per process): Multistage over the CKPT file tier, per-step and
fused, equals FullStorage bit for bit with the reference's counters."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1806_01117_b200 as pkg  # noqa: E402
import paper_1806_01117_b200.lstm as lstm  # noqa: E402


def main():
    scratch = sys.argv[1]
    ok = True
    for d, batch, dtype in ((32, 1, "f64"), (8, 4096, "f32")):
        n = 60
        ops = lstm.operator_pair(lstm.random_cell(d, n, 5), batch, dtype)
        s0 = lstm.random_state(d, 6) if batch == 1 else lstm.random_states(d, 6, batch, dtype)
        with pkg.FileBackend(scratch) as fb:
            for fuse in (False, True):  # same kernel family per mode -> same bits
                want, _ = pkg.execute(pkg.FullStorage(), ops, s0, fuse=fuse)
                got, st = pkg.execute(pkg.Multistage(4, interval=8), ops, s0, fb, fuse=fuse)
                same = got == want if batch == 1 else torch.equal(got, want)
                good = same and st.stores_issued == st.prefetches_issued > 0
                if not good:
                    print(json.dumps({"d": d, "fuse": fuse, "same": bool(same), "stores": st.stores_issued,
                                      "prefetches": st.prefetches_issued}), file=sys.stderr)
                ok = ok and good
    print(json.dumps({"ok": bool(ok)}))


if __name__ == "__main__":
    main()
