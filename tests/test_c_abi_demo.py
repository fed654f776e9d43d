"""The C boundary used from C: examples/c_abi_demo.c compiles against
include/ackpt.h + libackpt.so with gcc alone (CPU) and, on the GPU, runs
FullStorage / Revolve / Multistage with bit-identical adjoints and the
schedule's counters."""

import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1806_01117_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", f"-I{ROOT}/include", f"-I{CUDA}/include",
           os.path.join(ROOT, "examples", "c_abi_demo.c"), f"-L{LIB}", "-lackpt", f"-L{CUDA}/lib64", "-lcudart",
           "-lm", f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_demo_compiles_against_header_and_library(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs_on_device(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rep = json.loads(out.stdout.strip().splitlines()[-1])
    assert rep["bit_identical"] and rep["finite"] and rep["counters_ok"], rep
    assert rep["forward_evals"][2] == 80
