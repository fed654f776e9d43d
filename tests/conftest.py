import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def sched_golden():
    with open(os.path.join(GOLDEN, "schedule_golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def runtime_golden():
    with open(os.path.join(GOLDEN, "runtime_golden.json")) as fh:
        cfgs = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, "runtime_golden.npz")))
    return cfgs, arrays


@pytest.fixture(scope="session")
def step_golden():
    return dict(np.load(os.path.join(GOLDEN, "step_golden.npz")))


@pytest.fixture(scope="session")
def storage_golden():
    with open(os.path.join(GOLDEN, "storage_golden.json")) as fh:
        return json.load(fh)
