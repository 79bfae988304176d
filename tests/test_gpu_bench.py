"""The bench.py contract at N > 1, run as the driver launches it (torchrun, one
process per rank) with both ranks on the one GPU of the box (--same-gpu, IPC
transport): every leg runs its decomposed path (2-D slabs with 8 ghost rows,
3-D slabs with 2 ghost planes = two sweeps per pass across ranks, PW ghost
planes) and rank 0 prints one JSON line with the contract's keys. Functional
only: two ranks time-slicing one GPU say nothing about scaling."""
import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = pathlib.Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_same_gpu_contract(cuda_lib):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--same-gpu", "--steps", "1", "--warmup", "3", "--sweeps", "16", "--pw-apps", "2",
           "--j3-sweeps", "6", "--gs-sweeps", "4", "--no-e2e", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 2 and d["steps"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    j3 = d["jacobi3d"]
    assert j3["workload"].endswith("_zslabs2") and j3["value"] > 0
    assert j3["roofline"]["kernel"] == "jacobi3d_t2_kernel"  # T = 2 across ranks
    assert d["pw_advect3d"]["value"] > 0
