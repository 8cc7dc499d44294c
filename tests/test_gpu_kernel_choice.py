"""Both single-GPU MBGMV kernels pass the whole parity suite on their own.

The library serves a fused call with the ring-pipelined kernel (kernels.cu)
or the warp-task kernel (mbgmv8.cu) depending on the call's projection count
(api.cpp fused_kc, ring by default); SLORA_MBGMV=warp forces the warp-task kernel for every call, =auto for the o call.
The choice is read once per process, so each forced run is a subprocess that
re-runs the parity and MBGMM suites.  Mark: gpu.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kernel", ["warp", "auto"])
def test_parity_suite_with_forced_kernel(kernel):
    env = dict(os.environ, SLORA_MBGMV=kernel)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_mbgmm.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
