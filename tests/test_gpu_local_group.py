"""GPU tests of the decomposed path on ONE B200: P ranks in one process (LOCAL
transport) run the real kernels, the shared schedule (boundary rows, async
copy-engine swap, interior rows, join) and temporal blocking across ranks; the
gathered results equal the oracle bitwise."""
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = pathlib.Path(__file__).resolve().parent


@pytest.mark.parametrize("case", ["j2_h1", "j2_p3_h1", "j2_h4_t4", "j2_p4_h6_t6", "j2_p3_h3_t1", "j3_h1", "j3_p3_h2",
                                  "j3_p3_h2_t1", "j3_p2_h2_t2", "j3_p4_h3_t2", "j3_p2_h4_t2",
                                  "pw_p2", "pw_p4", "pen_j3_2x1", "pen_j3_1x2", "pen_j3_2x2", "pen_j3_3x2",
                                  "pen_j3t2_2x1", "pen_j3t2_1x2", "pen_j3t2_2x2", "pen_j3t2_3x2", "pen_j3t2_2x3_thin",
                                  "pen_j3h2_t1_2x2", "pen_pw_2x2", "pen_pw_3x2", "pen_pw_1x3"])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_local_group_equals_oracle(cuda_lib, case, fused):
    # fused=1: boundary sweeps store straight into the neighbours' ghost rows (NEXT #3);
    # fused=0: copy-engine swap after the boundary sweeps
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", ST_FUSED_HALO=fused)
    r = subprocess.run([sys.executable, str(HERE / "local_group_cases.py"), case], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "CASES OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_late_rank_is_detected_not_hung(cuda_lib):
    # st_comm_wait: a rank that never joins a swap surfaces as ST_ETIMEDOUT
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    r = subprocess.run([sys.executable, str(HERE / "local_group_cases.py"), "late_rank"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "CASES OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_shared_device_needs_enough_connections(cuda_lib):
    # k LOCAL ranks on one device deadlock if their 2k streams share hardware
    # queues; st_comm_init_local refuses k=4 under the default 8 connections
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    r = subprocess.run([sys.executable, str(HERE / "local_group_cases.py"), "connections"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "CASES OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
