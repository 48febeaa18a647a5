"""tcgen05 kind::tf32 operand-layout probe (tests/cuda/umma_probe.cu) on the GPU:
pins the K-major interleaved layout the tensor-core evaluator uses."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_umma_probe_layouts():
    src = os.path.join(ROOT, "tests", "cuda", "umma_probe.cu")
    exe = os.path.join(ROOT, "tests", "cuda", "umma_probe")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                        "-o", exe, src], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("<== OK") == 9
