"""GPU parity of the in-place lexicographic Gauss-Seidel (Listing 1 literally,
NEXT #4) against the sequential oracle — bitwise."""
import numpy as np
import pytest

import oracle
import stencil_inputs as si

pytestmark = pytest.mark.gpu


def run_gs(st, a_np, iters, nx=None):
    import torch
    a = torch.from_numpy(a_np).cuda()
    st.st_gauss_seidel2d_run(a, iters, nx=nx)
    torch.cuda.synchronize()
    return a.cpu().numpy()


SHAPES = [  # (nx, ny, ld, iters): strips of 32 rows, chunks of 64 columns, ragged tails
    (1, 1, 4, 3), (5, 3, 8, 4), (64, 32, 66, 2), (65, 33, 68, 3), (130, 64, 132, 5), (200, 95, 202, 7),
    (129, 200, 132, 11), (300, 257, 302, 4), (1000, 130, 1002, 3),
    # odd pitches: the register (non-tiled) kernel
    (65, 33, 67, 3), (200, 95, 203, 5),
]


@pytest.mark.parametrize("nx,ny,ld,iters", SHAPES)
def test_gs_bitwise(cuda_lib, nx, ny, ld, iters):
    a = si.jacobi2d_grid(nx, ny, ld=ld)
    want = oracle.gauss_seidel2d(a, iters, nx=nx)
    got = run_gs(cuda_lib, a, iters, nx=nx)
    assert np.array_equal(got, want)


def test_gs_many_sweeps_large(cuda_lib):
    a = si.jacobi2d_grid(1500, 1100)
    assert np.array_equal(run_gs(cuda_lib, a, 25), oracle.gauss_seidel2d(a, 25))


def test_gs_linear_fixed_point(cuda_lib):
    nx, ny = 700, 333
    y, x = np.mgrid[0:ny + 2, 0:nx + 2]
    a = np.ascontiguousarray((4 * x - 3 * y + 11).astype(np.float64))
    assert np.array_equal(run_gs(cuda_lib, a, 50), a)
