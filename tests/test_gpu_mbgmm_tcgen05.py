"""The tcgen05 MBGMM shrink (mbgmm.cu mbgmm_shrink_tc_kernel: TMA-swizzled x
tiles, cp.async-gathered canonical A k-blocks, tcgen05.mma into TMEM, k-split
parts summed in order by the expand) passes the MBGMM suite -- bit-exact in
the integer regime, within tolerance on random inputs.  SLORA_MBGMM_TC is read
once per process, so the suite runs in a subprocess.  Mark: gpu.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_mbgmm_suite_on_tcgen05_shrink():
    env = dict(os.environ, SLORA_MBGMM_TC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_mbgmm.py"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
