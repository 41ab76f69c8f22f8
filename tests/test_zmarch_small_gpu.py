"""The z-marching line-Jacobi kernel is chosen only for large plane groups
(PSM_ZMARCH_MIN_CELLS, default 2^21 cells); the fused multi-GPU halo forces it
on slabs of any size.  Re-run the golden line-Jacobi parity cases in a child
process with the threshold at 0, so every specialised nx (here 64) goes
through the z-marching kernel at small, ragged shapes."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_golden_line_jacobi_through_zmarch():
    env = dict(os.environ, PSM_ZMARCH_MIN_CELLS="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_parity_gpu.py"), "-k", "line_jac or multi_line_jac"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout
