"""Two ranks, one GPU: torchrun --nproc-per-node 2 with
gloo, both ranks on cuda:0, each running the real engine on its batch shard
(tests/multirank_worker.py).  The ranks never wait on each other's kernels
(no collective inside the pass), so sharing the device is safe.  Checks: the
interval is agreed, the shards tile the batch, and every sequence's adjoint
is bit-identical to the unsharded run (long-memory cell: non-zero)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("fuse", ["1", "0"], ids=["fused", "per-step"])
def test_two_ranks_bit_identical_to_unsharded(fuse):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "multirank_worker.py")]
    out = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, MR_FUSE=fuse), capture_output=True, text=True,
                         timeout=540)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["world"] == 2 and line["intervals_agreed"] and line["covers_batch"]
    assert line["bit_identical_to_unsharded"] and line["forward_evals_equal"]
    assert line["adjoint_norm"] > 1e-20 and len(set(line["digests"])) == 2
