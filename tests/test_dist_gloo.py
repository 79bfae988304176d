"""World-size-2 (and 3) gloo runs of the decomposed Jacobi schedule on CPU:
real torch.distributed processes exchange halos per st_halo_plan and execute
st_jacobi2d_schedule / st_jacobi3d_schedule; the gathered result is bitwise the
oracle's."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import torch.distributed as dist
    import oracle
    import stencil_inputs as si
    from slab_sim import run_gloo_rank
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if len(cfg) == 6:  # 3-D: (nx, ny, nz, h, iters, tblock), z slabs
            nx, ny, nz, h, iters, tblock = cfg
            a = si.jacobi3d_grid(nx, ny, nz)
            want = lambda: oracle.jacobi3d(a, iters, nx=nx)
        else:
            nx, ny, h, iters, tblock = cfg
            a = si.jacobi2d_grid(nx, ny)
            want = lambda: oracle.jacobi2d(a, iters, nx=nx)
        got = run_gloo_rank(a, nx, h, iters, tblock)
        if rank == 0:
            q.put(bool(np.array_equal(got, want())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, (33, 40, 1, 9, 1)),   # one ghost row, swap every sweep, overlap split
    (2, (33, 40, 4, 11, 4)),  # temporal blocking across ranks, 4-deep ghosts
    (3, (20, 31, 2, 7, 2)),   # odd split (remainder to the high rank), middle rank
    (2, (65, 24, 3, 8, 1)),   # deep ghosts with single sweeps
    (2, (9, 6, 14, 2, 7, 0)),  # 3-D z slabs, two sweeps per pass (auto with 2 ghost planes)
    (3, (7, 5, 16, 3, 6, 2)),  # 3-D, middle rank, slab of 5 planes < 2*halo (no overlap split)
])
def test_gloo_schedule_equals_oracle(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
