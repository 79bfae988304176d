"""GPU tests of the communicator path.

* A real NCCL communicator of size 1 drives st_jacobi2d_run / st_pw_advect3d
  through their slab code path (ghost depth > 1, schedule ops, comm stream,
  events) on one B200 — bitwise vs the oracle.
* With >= 2 GPUs (not available in this round's 1-GPU runs), P ranks run the
  decomposed Jacobi and PW over NCCL and the gathered result must equal the
  oracle bitwise; the test skips on 1-GPU boxes.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import stencil_inputs as si

pytestmark = pytest.mark.gpu


def slab_with_ghosts(a_glob, h):
    """Single-rank slab with h ghost rows per side; the Dirichlet rows sit next to the owned rows."""
    ny = a_glob.shape[0] - 2
    out = np.zeros((ny + 2 * h, a_glob.shape[1]))
    out[h - 1:h + ny + 1] = a_glob
    return out


@pytest.fixture(scope="module")
def comm1(cuda_lib):
    import torch
    torch.cuda.set_device(0)
    c = cuda_lib.Comm.create(0, 1, cuda_lib.Comm.unique_id(), 0)
    yield c
    c.close()


@pytest.mark.parametrize("h,tblock,iters", [(1, 1, 5), (2, 1, 7), (2, 2, 9), (4, 4, 13), (4, 0, 10), (8, 8, 17)])
def test_single_rank_comm_jacobi(cuda_lib, comm1, h, tblock, iters):
    import torch
    nx, ny = 200, 300
    a_glob = si.jacobi2d_grid(nx, ny)
    a = torch.from_numpy(slab_with_ghosts(a_glob, h)).cuda()
    b = torch.full_like(a, float("nan"))
    r = cuda_lib.st_jacobi2d_run(a, b, iters, tblock=tblock, halo=h, comm=comm1, nx=nx)
    got = r.cpu().numpy()[h - 1:h + ny + 1, :nx + 2]
    want = oracle.jacobi2d(a_glob, iters, nx=nx)[:, :nx + 2]
    assert np.array_equal(got, want)


def test_single_rank_comm_pw(cuda_lib, comm1):
    import torch
    nx, ny, nz = 96, 20, 33
    d = si.pw_inputs(nx, ny, nz)
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    g = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    cuda_lib.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"],
                            g["tzd2"], comm=comm1)
    for o, w in zip(outs, want):
        assert np.array_equal(o.cpu().numpy(), w)


def test_halo_exchange_single_rank_is_noop(cuda_lib, comm1):
    import torch
    f = torch.arange(60, dtype=torch.float64, device="cuda").reshape(6, 10)
    before = f.clone()
    cuda_lib.st_halo_exchange(comm1, [f], 4, 10, 1)
    torch.cuda.synchronize()
    assert torch.equal(f, before)


# ------------------------------------------------------------------ >= 2 GPUs
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _multi_worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    import paper_2310_01882_b200 as st
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = st.Comm.from_process_group(rank)
    ok = True
    # Jacobi: global 64+ring x (nx) grid, row slabs, ghost depth 4, T = 4
    nx, ny, h, iters = 130, 257, 4, 23
    a_glob = si.jacobi2d_grid(nx, ny)
    start, n = st.st_block_split(ny, world, rank)
    loc = np.zeros((n + 2 * h, a_glob.shape[1]))
    for l in range(n + 2 * h):
        gr = start + 1 + (l - h)
        if 0 <= gr <= ny + 1:
            loc[l] = a_glob[gr]
    for tblock in (1, 4):
        a = torch.from_numpy(loc).cuda()
        b = torch.empty_like(a)
        r = st.st_jacobi2d_run(a, b, iters, tblock=tblock, halo=h, comm=comm, nx=nx)
        rows = [None] * world
        dist.all_gather_object(rows, (start, r.cpu().numpy()[h:h + n]))
        if rank == 0:
            want = oracle.jacobi2d(a_glob, iters, nx=nx)
            for s0, blk in rows:
                ok &= bool(np.array_equal(blk[:, :nx + 2], want[s0 + 1:s0 + 1 + blk.shape[0], :nx + 2]))
    # PW: z slabs, one ghost plane, exchanged by the library
    nxp, nyp, nzp = 70, 18, 41
    d = si.pw_inputs(nxp, nyp, nzp)
    z0, nzl = st.st_block_split(nzp, world, rank)
    dl = si.pw_inputs(nxp, nyp, nzp, plane0=z0, planes=nzl + 2)
    g = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in dl.items()}
    for k in "uvw":  # ghost planes must come from the neighbours: poison them
        if rank > 0:
            g[k][0] = float("nan")
        if rank < world - 1:
            g[k][-1] = float("nan")
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"],
                      comm=comm)
    parts = [None] * world
    dist.all_gather_object(parts, (z0, [o.cpu().numpy()[1:nzl + 1] for o in outs]))
    if rank == 0:
        want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
        for s0, blks in parts:
            for blk, w in zip(blks, want):
                ok &= bool(np.array_equal(blk, w[s0 + 1:s0 + 1 + blk.shape[0]]))
        q.put(ok)
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_gpu_decomposed_equals_oracle(cuda_lib, world):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_multi_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


_BORROW_SCRIPT = r"""
import os, sys
sys.path.insert(0, os.environ["REPO"])
import numpy as np, torch, torch.distributed as dist
import oracle, stencil_inputs as si
import paper_2310_01882_b200 as st
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
t = torch.ones(4, device="cuda")
dist.all_reduce(t)  # materialise torch's communicator
comm = st.Comm.from_torch_nccl(0)
assert (comm.rank, comm.nranks, comm.device) == (0, 1, 0)
nx, ny, h = 150, 90, 2
a_glob = si.jacobi2d_grid(nx, ny)
slab = np.zeros((ny + 2 * h, a_glob.shape[1])); slab[h - 1:h + ny + 1] = a_glob
a = torch.from_numpy(slab).cuda(); b = torch.full_like(a, float("nan"))
r = st.st_jacobi2d_run(a, b, 7, tblock=2, halo=h, comm=comm, nx=nx)
ok = np.array_equal(r.cpu().numpy()[h - 1:h + ny + 1, :nx + 2], oracle.jacobi2d(a_glob, 7, nx=nx)[:, :nx + 2])
comm.close()
dist.all_reduce(t)  # torch's communicator is still alive (borrowed, not destroyed)
dist.destroy_process_group()
print("BORROW_OK" if ok else "BORROW_MISMATCH")
"""


def test_borrowed_torch_nccl_communicator(cuda_lib, tmp_path):
    # st_comm_from_nccl: torch's ProcessGroupNCCL communicator drives the slab path
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, REPO=repo, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    out = subprocess.run([sys.executable, "-c", _BORROW_SCRIPT], env=env, capture_output=True, text=True,
                         timeout=300)
    assert "BORROW_OK" in out.stdout, out.stdout + out.stderr
