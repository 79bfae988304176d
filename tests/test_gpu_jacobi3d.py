"""GPU parity of st_jacobi3d_run (the paper's 7-point benchmark, PAPER.md:214;
SURVEY.md §8(f) NEXT #1) against the CPU oracle — bitwise."""
import numpy as np
import pytest

import oracle
import stencil_inputs as si

pytestmark = pytest.mark.gpu


def run_gpu(st, a_np, iters, tblock=0, nx=None, halo=1, comm=None):
    import torch
    a = torch.from_numpy(a_np).cuda()
    b = torch.full_like(a, float("nan"))
    r = st.st_jacobi3d_run(a, b, iters, tblock=tblock, nx=nx, halo=halo, comm=comm)
    torch.cuda.synchronize()
    assert (r is b) == bool(iters & 1)
    return r.cpu().numpy()


SHAPES = [  # (nx, ny, nz, ldx, iters): tiles of 32 x 32 (2 rows/thread), ragged in every dim
    (1, 1, 1, 4, 3), (2, 3, 5, 4, 2), (31, 33, 7, 34, 5), (32, 32, 64, 34, 4), (33, 31, 65, 36, 3),
    (64, 70, 9, 66, 6), (100, 45, 130, 102, 7), (257, 9, 11, 260, 2),
]


@pytest.mark.parametrize("nx,ny,nz,ldx,iters", SHAPES)
def test_ragged_shapes_bitwise(cuda_lib, nx, ny, nz, ldx, iters):
    a = si.jacobi3d_grid(nx, ny, nz, ldx=ldx)
    want = oracle.jacobi3d(a, iters, nx=nx)
    got = run_gpu(cuda_lib, a, iters, nx=nx)
    assert np.array_equal(got[:, :, :nx + 2], want[:, :, :nx + 2])
    if iters & 1:  # result in b: its pitch padding was never written
        assert np.all(np.isnan(got[:, :, nx + 2:]))


def test_integer_linear_fixed_point_many_sweeps(cuda_lib):
    nz, ny, nx = 40, 66, 70
    z, y, x = np.meshgrid(np.arange(nz + 2), np.arange(ny + 2), np.arange(nx + 2), indexing="ij")
    a = np.ascontiguousarray((3 * x + 2 * y + 5 * z + 7).astype(np.float64))
    assert np.array_equal(run_gpu(cuda_lib, a, 200), a)


@pytest.mark.slow
def test_512cubed_5_sweeps_bitwise(cuda_lib):
    a = si.jacobi3d_grid(512, 512, 512)
    assert np.array_equal(run_gpu(cuda_lib, a, 5), oracle.jacobi3d(a, 5))


def test_tblock_rejected(cuda_lib):
    import torch
    a = torch.zeros(6, 6, 6, dtype=torch.float64, device="cuda")
    with pytest.raises(cuda_lib.StencilError) as e:
        cuda_lib.st_jacobi3d_run(a, a.clone(), 3, tblock=3)
    assert e.value.code == cuda_lib.ST_ENOTSUP


@pytest.mark.parametrize("iters", [2, 3, 4, 5, 6, 9])
@pytest.mark.parametrize("shape", [(45, 37, 21), (130, 17, 70), (1, 1, 1), (300, 9, 3)])
def test_two_sweep_passes_equal_single_sweeps(cuda_lib, iters, shape):
    # temporal blocking T = 2 (tblock 0 = auto, 2 = forced) is bitwise T = 1 and the oracle,
    # for every parity of the pass count
    import torch
    nx, ny, nz = shape
    g = si.jacobi3d_grid(nx, ny, nz)
    want = oracle.jacobi3d(g, iters)
    for tb in (1, 2, 0):
        a = torch.from_numpy(g).cuda()
        r = cuda_lib.st_jacobi3d_run(a, torch.full_like(a, float("nan")), iters, tblock=tb)
        torch.cuda.synchronize()
        assert np.array_equal(r.cpu().numpy(), want), f"tblock={tb}"


@pytest.mark.parametrize("h", [1, 3])
def test_single_rank_comm(cuda_lib, h):
    import torch
    torch.cuda.set_device(0)
    comm = cuda_lib.Comm.create(0, 1, cuda_lib.Comm.unique_id(), 0)
    try:
        nx, ny, nz, iters = 40, 30, 20, 7
        g = si.jacobi3d_grid(nx, ny, nz)
        loc = np.zeros((nz + 2 * h, ny + 2, g.shape[2]))
        loc[h - 1:h + nz + 1] = g
        got = run_gpu(cuda_lib, loc, iters, halo=h, comm=comm)
        assert np.array_equal(got[h - 1:h + nz + 1], oracle.jacobi3d(g, iters))
    finally:
        comm.close()


def test_fast_div6_is_correctly_rounded(cuda_lib):
    # the 3-D kernel divides by 6 with 1 DMUL + 2 DFMA (common.cuh ddiv6); it must equal
    # IEEE division bit for bit: random significands over all exponents, signs, and the
    # special values, plus the values the stencil actually produces
    import torch
    g = torch.Generator(device="cuda").manual_seed(1234)
    n = 1 << 26
    bits = torch.randint(0, 2 ** 62, (n,), device="cuda", generator=g, dtype=torch.int64)
    top = torch.randint(0, 2, (n,), device="cuda", generator=g, dtype=torch.int64) << 62  # exponents >= 1024 too
    sign = torch.randint(0, 2, (n,), device="cuda", generator=g, dtype=torch.int64) << 63
    x = (bits | top | sign).view(torch.float64)
    assert cuda_lib.st_selftest_div6(x) == 0
    sums = torch.rand(n, device="cuda", generator=g, dtype=torch.float64) * 6 + 3  # six values in [0.5, 1.5)
    assert cuda_lib.st_selftest_div6(sums) == 0
    special = torch.tensor([0.0, -0.0, float("inf"), float("-inf"), float("nan"), 5e-324, 2.2250738585072014e-308,
                            1.7976931348623157e308, 6.0, -6.0, 3.0, 1.0], dtype=torch.float64, device="cuda")
    assert cuda_lib.st_selftest_div6(special) == 0
    # both ends of ddiv6's fast range (biased exponents 24 .. 2022) and their neighbours
    import numpy as np
    edge = []
    for e in (22, 23, 24, 25, 2021, 2022, 2023, 2024):
        for m in (0, 1, 2 ** 51, 2 ** 52 - 1):
            edge += [(e << 52) | m, (1 << 63) | (e << 52) | m]
    ev = torch.from_numpy(np.array(edge, dtype=np.uint64).view(np.float64)).cuda()
    assert cuda_lib.st_selftest_div6(ev) == 0


@pytest.mark.parametrize("tblock", [1, 2])
@pytest.mark.parametrize("shape", [(150, 37, 23), (129, 17, 40)])
def test_quotients_outside_the_fast_division_range(cuda_lib, tblock, shape):
    # sums that leave ddiv6's fast range (zero, subnormal/tiny, huge, non-finite) take the
    # exact division: per quotient (T = 1) or by the deferred per-plane check of the
    # two-sweep kernel, which recomputes a plane when any quotient of the CTA was out of range
    import torch
    nx, ny, nz = shape
    g = si.jacobi3d_grid(nx, ny, nz).copy()
    g[3:6, 2:9, 10:40] = 0.0                       # zero sums
    g[8:11, 5:15, 60:100] *= 2.0 ** -1040          # subnormal neighbourhoods
    g[12:14, 20:30, 5:30] *= 2.0 ** 1021           # near overflow (sums overflow to inf)
    g[15, 3, 7] = float("inf")
    g[16, 4, 8] = -0.0
    want = oracle.jacobi3d(g, 4)
    a = torch.from_numpy(g).cuda()
    r = cuda_lib.st_jacobi3d_run(a, torch.full_like(a, float("nan")), 4, tblock=tblock)
    torch.cuda.synchronize()
    got = r.cpu().numpy()
    assert np.array_equal(got, want, equal_nan=True)
