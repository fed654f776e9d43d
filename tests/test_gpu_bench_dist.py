"""bench.py under torchrun with the NCCL process group initialised (one rank,
ACKPT_BENCH_DIST=1): the multi-GPU plumbing -- interval agreement
(all_reduce MAX), barriers, max-over-ranks timing -- runs on the real
device and prints the contract's JSON line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_bench_under_torchrun_with_nccl_process_group():
    env = dict(os.environ, ACKPT_BENCH_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--n-steps", "600", "--steps", "1", "--warmup", "3", "--full-n", "100",
           "--no-c1", "--no-cpu", "--no-revolve", "--no-other-mode", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=540)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["unit"] == "steps/s"
    assert line["scaling"] == "weak" and line["gpu_launches"] > 0
