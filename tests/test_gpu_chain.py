"""Chained tensor-core launches (programmatic dependent launch + per-tile
completion flags, csrc/chain.cuh; d = 8 fused and d = 16 / 32 / 64 fused and
per-step) produce bit-identical results to
plain launches: tools/chain_probe.py with ACKPT_TC_CHAIN=0 (never chain),
default (the launches the executor marks chain) and force (every back-to-back
launch of the cell chains)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(mode):
    env = dict(os.environ)
    env.pop("ACKPT_TC_CHAIN", None)
    if mode is not None:
        env["ACKPT_TC_CHAIN"] = mode
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "chain_probe.py")], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("chain_probe ok")][-1].split()
    return line[line.index("direct") + 1], line[line.index("engine") + 1]


@pytest.mark.gpu
def test_chained_launches_bit_identical():
    plain_direct, plain_engine = _run("0")
    direct, engine = _run(None)
    assert (direct, engine) == (plain_direct, plain_engine)
    forced_direct, _ = _run("force")
    assert forced_direct == plain_direct
