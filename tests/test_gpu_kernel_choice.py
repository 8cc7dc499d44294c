"""Both single-GPU fused MBGMV kernels pass the parity suite on their own.

The library serves a fused call with the ring-pipelined kernel (kernels.cu,
the default) or, with SLORA_MBGMV=group, the cluster kernel (mbgmv.cu:
K-split clusters exchanging partial v through distributed shared memory,
dynamic item claiming).  The choice is read once per process, so each forced
run is a subprocess that re-runs the parity and MBGMM suites.  Mark: gpu.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kernel", ["group"])
def test_parity_suite_with_forced_kernel(kernel):
    env = dict(os.environ, SLORA_MBGMV=kernel)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_mbgmm.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
