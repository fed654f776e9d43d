"""Every environment-selected kernel path (selected by environment variables that are
read once per process) stays within the fp32 parity tolerance: each runs
tests/variant_check.py in its own subprocess."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = [
    # d = 8 at B > 2048 (below that the CTA-per-sequence kernels run)
    ({"ACKPT_TC": "0"}, 8, 4096),                       # FFMA2 fused family (the documented fallback)
    ({"ACKPT_TC": "0"}, 8, 4002),                       # ... ragged tail
    ({}, 8, 4002),                                      # tcgen05 reverse without the bulk prefetch (B % 4 != 0)
    ({"ACKPT_TCD": "0"}, 16, 4096),                     # CTA-per-sequence kernels for d = 16 at large B
    ({"ACKPT_SB_MAX": "0", "ACKPT_TCD": "0"}, 16, 4096),  # thread-per-sequence generic kernels
    ({}, 32, 4100),                                     # tensor-core d = 32, ragged tile
    ({"ACKPT_SB_FIRST": "0"}, 32, 1000),                # tensor-core d = 32 below the crossover
    ({"ACKPT_PDL": "0"}, 32, 3),                        # CTA-per-sequence without dependent launches
    ({"ACKPT_SB_FIRST": "0"}, 8, 1000),                 # tcgen05 d = 8 family below the crossover
]


@pytest.mark.parametrize("env,d,batch", VARIANTS, ids=lambda v: json.dumps(v) if isinstance(v, dict) else str(v))
def test_variant_parity(env, d, batch):
    full_env = dict(os.environ, **env)
    out = subprocess.run([sys.executable, os.path.join(HERE, "variant_check.py"), str(d), str(batch)],
                         env=full_env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    errs = json.loads(out.stdout.strip().splitlines()[-1])
    assert max(errs.values()) <= 1e-5, errs


def test_file_stage_host_function_path(tmp_path):
    # ACKPT_FILE_HOSTFN=1: the file stage through cudaLaunchHostFunc instead
    # of the tier I/O threads -- same adjoints and counters
    out = subprocess.run([sys.executable, os.path.join(HERE, "file_stage_check.py"), str(tmp_path)],
                         env=dict(os.environ, ACKPT_FILE_HOSTFN="1"), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1])["ok"]
