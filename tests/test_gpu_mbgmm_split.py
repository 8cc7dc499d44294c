"""GPU parity of the MBGMM shrink's K-split / unit-height variants.

The mma.sync shrink holds R stored A rows (8, 16 or 32) over one of `split`
parts of K ("K-split shrink units"); the expand adds the
parts in order.  The defaults (whole K at h = 4096, two 4096-column parts at
h = 8192) run in the other MBGMM suites.  The choice is read once per process
from SLORA_MG_SPLIT / SLORA_MG_SROWS, so each setting re-runs the MBGMM parity
suites (bit-exact integer regime + tolerance cases, against the fp64 oracle)
in a fresh interpreter.  Mark: gpu.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("split,srows", [(2, 32), (4, 16), (4, 0), (8, 0), (1, 8)])
def test_mbgmm_suites_under_split(split, srows):
    env = dict(os.environ, SLORA_MG_SPLIT=str(split), SLORA_MG_SROWS=str(srows))
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
         "tests/test_gpu_mbgmm.py", "tests/test_gpu_mbgmm_gather.py"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
