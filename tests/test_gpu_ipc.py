"""GPU tests of the IPC transport: P processes (torchrun-style env, gloo for the
out-of-band blob exchange) share the available GPU(s); the halo swap runs on
CUDA-IPC mappings with device-side flags (fused and copy-engine). Bitwise vs the oracle."""
import os
import pathlib
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = pathlib.Path(__file__).resolve().parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [(w, c, f) for w in (2, 3) for c in ("j2_h1", "j2_h4_t4", "pw", "j3_h1", "j3_h2_t1", "j3_h2_t2", "j3_h3_t2")
         for f in ("1", "0")]
CASES += [(w, c, "1") for w in (2, 3, 4) for c in ("pen_j3", "pen_j3t2", "pen_pw")]  # pencils: y-z process grids


def _run(world, case, fused, timeout=240):
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), ST_FUSED_HALO=fused)
        procs.append(subprocess.Popen([sys.executable, str(HERE / "ipc_cases.py"), case], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("IPC case timed out")
        outs.append((p.returncode, o, e))
    assert all(rc == 0 for rc, _, _ in outs), [(rc, o[-500:], e[-1500:]) for rc, o, e in outs]
    assert "OK" in outs[0][1]


@pytest.mark.parametrize("world,case,fused", CASES)
def test_ipc_multiprocess_equals_oracle(cuda_lib, world, case, fused):
    _run(world, case, fused)


@pytest.mark.slow
@pytest.mark.parametrize("case", ["c4_bands", "c5_planes"])
def test_ipc_preflight_full_width_shapes(cuda_lib, case):
    # the launch shapes of the 8-GPU scaling run (C4 width, 4096-row slabs, H = T = 8;
    # C5 slabs) with 4 processes on one GPU: bitwise on the bands/planes at every slab edge
    _run(4, case, "1", timeout=900)
