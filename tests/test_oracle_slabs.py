"""Pin D1: the decomposed CPU oracle ("halo swap
between iterations", SPEC.md:399 block split remainder-to-high, SPEC.md:465
ranks-sim bitwise equal to serial) equals the undecomposed oracle bitwise."""
import numpy as np
import pytest

import oracle
import stencil_inputs as si


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("ny", [32, 37])
def test_D1_jacobi_slabs_h1(p, ny):
    a = si.jacobi2d_grid(19, ny, ld=22)
    ref = oracle.jacobi2d(a, 23, nx=19)
    assert np.array_equal(oracle.jacobi2d_slabs(a, 23, p, 1, nx=19), ref)


@pytest.mark.parametrize("p,h,iters", [(2, 2, 9), (3, 4, 13), (4, 3, 12), (8, 2, 7), (2, 4, 1)])
def test_D1_jacobi_slabs_deep_ghosts(p, h, iters):
    # H-deep ghosts swapped every H sweeps (temporal blocking across ranks), iters % H != 0 included
    a = si.jacobi2d_grid(26, 45)
    assert np.array_equal(oracle.jacobi2d_slabs(a, iters, p, h), oracle.jacobi2d(a, iters))


def test_slabs_reject_thin_slabs():
    a = si.jacobi2d_grid(8, 6)
    with pytest.raises(ValueError):
        oracle.jacobi2d_slabs(a, 3, 4, 2)  # 6 rows / 4 ranks -> 1 row < H=2


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
def test_D1_pw_slabs(p):
    nz, ny, nx = 17, 6, 9
    d = si.pw_inputs(nx, ny, nz, ldx=12)
    ref = oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx)
    got = oracle.pw_slabs(d["u"], d["v"], d["w"], d, p, nx=nx)
    for r, g in zip(ref, got):
        assert np.array_equal(r, g)


@pytest.mark.parametrize("py,pz", [(1, 1), (2, 1), (1, 3), (2, 2), (3, 2), (4, 3)])
def test_D1_pencils_jacobi3d(py, pz):
    # 2-D (y, z) process grid, "decompose the 3D space into two dimensions"
    a = si.jacobi3d_grid(11, 13, 14)
    assert np.array_equal(oracle.pencils_jacobi3d(a, 7, py, pz), oracle.jacobi3d(a, 7))


@pytest.mark.parametrize("py,pz", [(2, 1), (1, 2), (2, 2), (3, 3), (2, 4)])
def test_D1_pencils_pw_needs_corner_ghosts(py, pz):
    # PW reads (z+1, y-1) and (z-1, y+1): the y-then-z swap must fill the corner ghosts
    nz, ny, nx = 13, 11, 9
    d = si.pw_inputs(nx, ny, nz, ldx=12)
    ref = oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx)
    got = oracle.pencils_pw(d["u"], d["v"], d["w"], d, py, pz, nx=nx)
    for r, g in zip(ref, got):
        assert np.array_equal(r, g)
