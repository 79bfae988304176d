"""The bench.py contract, run as the driver launches it.

* N = 2 (torchrun, one process per rank) with both ranks on the one GPU of the box
  (--same-gpu, IPC transport): the strong-scaling legs (C4 row slabs with 8 ghost
  rows and T = 8 across ranks, C5 z-slabs) run their decomposed paths, rank 0 times
  the same workload alone, and the one JSON line carries the scaling keys (per-GPU,
  aggregate, efficiency, transport, phase profile). Functional only: two ranks
  time-slicing one GPU say nothing about scaling.
* N = 1 with few sweeps: the headline line carries the single-GPU C4/C5 legs and the
  T = 1 sweep leg, each with its roofline.
"""
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


def _json_line(r):
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


CONTRACT = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "dtype", "config", "roofline", "gpu_launches", "clocks")


def test_bench_two_ranks_same_gpu_contract(cuda_lib):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--same-gpu", "--steps", "1", "--warmup", "3", "--sweeps", "16", "--pw-apps", "2",
           "--scale-steps", "1", "--j3-sweeps", "6", "--no-e2e", "--no-cpu"]
    d = _json_line(subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                                  env=dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")))
    for k in CONTRACT + ("per_gpu", "aggregate", "efficiency", "phases", "c5"):
        assert k in d, k
    assert d["n_gpus"] == 2 and d["steps"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("jacobi2d_32768x32768") and "rowslabs2" in d["config"]["workload"]
    assert d["config"]["transport"] == "ipc-fused" and d["config"]["ipc_probe"] == "ok"
    assert abs(d["per_gpu"] * 2 - d["aggregate"]) < 1e-2 * d["aggregate"] and d["aggregate"] == d["value"]
    assert d["efficiency"] > 0 and d["t1_ms_per_step"] > 0
    ph = d["phases"]
    assert len(ph["ranks"]) == 2 and all(r["boundary"] > 0 and r["interior"] > 0 for r in ph["ranks"])
    c5 = d["c5"]
    assert "zslabs2" in c5["workload"] and c5["per_gpu"] > 0 and c5["efficiency"] > 0
    assert len(c5["phases"]["ranks"]) == 2 and all(r["swap"] > 0 for r in c5["phases"]["ranks"])
    j3 = d["jacobi3d"]
    assert j3["workload"].endswith("_zslabs2") and j3["value"] > 0
    assert j3["roofline"]["kernel"] == "jacobi3d_t2_kernel"  # T = 2 across ranks


def test_bench_one_gpu_contract(cuda_lib):
    cmd = [sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3", "--sweeps", "16",
           "--pw-apps", "2", "--scale-steps", "1", "--j3-sweeps", "6", "--gs-sweeps", "4", "--no-e2e", "--no-cpu"]
    d = _json_line(subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900))
    for k in CONTRACT + ("c4", "c5", "jacobi2d_t1", "pw_advect3d"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["config"]["workload"].startswith("jacobi2d_16384x16384")
    assert d["c4"]["workload"].startswith("jacobi2d_32768x32768") and d["c4"]["roofline"]["frac"] > 0
    assert d["c5"]["workload"].startswith("pw_advect3d_1024x1024x512") and d["c5"]["roofline"]["frac"] > 0
    t1 = d["jacobi2d_t1"]
    assert t1["roofline"]["kernel"] == "jacobi2d_stream_kernel" and t1["roofline"]["sweeps_per_launch"] == [1]
