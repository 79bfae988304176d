"""GPU parity of the multi-sweep Gauss-Seidel wavefront (K sweeps in flight per
warp, gauss_seidel2d_ms.cu) against the sequential oracle — bitwise, for every
sweep depth K = 1..4 (one process each: the depth is read once per process)."""
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_gs_multisweep_bitwise(cuda_lib, k):
    env = dict(os.environ, ST_GS_MS_K=str(k), ST_GS_MS="1")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "gs_ms_cases.py"), str(k)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
