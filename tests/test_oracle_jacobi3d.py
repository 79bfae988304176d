"""Pins of the 3-D 7-point Jacobi oracle (the paper's benchmark 1, PAPER.md:214;
readings R20/R21: sum z-,z+,y-,y+,x-,x+ then / 6.0) against things other than itself."""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
import stencil_inputs as si
from oracle import numpy_ref, scalar

U = 2.0 ** -53


def field(nz, ny, nx, f, ldx=None):
    ldx = nx + 2 if ldx is None else ldx
    z, y, x = np.meshgrid(np.arange(nz + 2), np.arange(ny + 2), np.arange(ldx), indexing="ij")
    a = f(z, y, x).astype(np.float64)
    a[:, :, nx + 2:] = 0.0
    return np.ascontiguousarray(a)


def test_single_cell_average():
    a = np.zeros((3, 3, 3))
    vals = {(0, 1, 1): 1.0, (2, 1, 1): 2.0, (1, 0, 1): 3.0, (1, 2, 1): 4.0, (1, 1, 0): 5.0, (1, 1, 2): 9.0}
    for k, v in vals.items():
        a[k] = v
    for n in (1, 4):
        assert oracle.jacobi3d(a, n)[1, 1, 1] == 24.0 / 6.0


@pytest.mark.parametrize("n", [0, 1, 3, 10, 40])
def test_2x2x2_closed_form(n):
    a = np.ones((4, 4, 4))
    a[1:3, 1:3, 1:3] = 0.0
    r = oracle.jacobi3d(a, n)
    assert np.all(r[1:3, 1:3, 1:3] == 1.0 - 2.0 ** -n)


@pytest.mark.parametrize("shape,iters", [((1, 1, 1), 3), ((5, 7, 9), 6), ((12, 3, 33), 11)])
def test_integer_linear_fixed_point(shape, iters):
    nz, ny, nx = shape
    a = field(nz, ny, nx, lambda z, y, x: 3 * x + 2 * y + 5 * z + 7, ldx=nx + 3)
    assert np.array_equal(oracle.jacobi3d(a, iters, nx=nx), a)


def test_sine_eigenmode():
    nz, ny, nx = 14, 12, 16
    a = field(nz, ny, nx, lambda z, y, x: np.sin(np.pi * x / (nx + 1)) * np.sin(np.pi * y / (ny + 1))
              * np.sin(np.pi * z / (nz + 1)))
    a[0] = a[-1] = 0.0
    a[:, 0] = a[:, -1] = 0.0
    a[:, :, 0] = a[:, :, -1] = 0.0
    n = 30
    lam = (math.cos(math.pi / (nx + 1)) + math.cos(math.pi / (ny + 1)) + math.cos(math.pi / (nz + 1))) / 3
    r = oracle.jacobi3d(a, n)
    assert np.abs(r - lam ** n * a).max() <= 1e-14


def test_exact_rational_brute_force():
    rng = random.Random(3)
    nz, ny, nx, n = 4, 5, 6, 12
    vals = [[[Fraction(rng.randrange(-2 ** 16, 2 ** 16), 2 ** 16) for _ in range(nx + 2)] for _ in range(ny + 2)]
            for _ in range(nz + 2)]
    exact = scalar.jacobi3d(vals, n, Fraction(6))
    a = np.array([[[float(v) for v in row] for row in pl] for pl in vals])
    r = oracle.jacobi3d(a, n)
    amax = max(abs(v) for pl in vals for row in pl for v in row)
    err = max(abs(Fraction(float(r[z, y, x])) - exact[z][y][x])
              for z in range(nz + 2) for y in range(ny + 2) for x in range(nx + 2))
    assert err <= 6 * Fraction(U) * n * amax


def test_z_mirror_symmetry():
    a = si.jacobi3d_grid(9, 8, 11)
    r = oracle.jacobi3d(a, 5)
    rf = oracle.jacobi3d(np.ascontiguousarray(a[::-1]), 5)
    assert np.array_equal(rf[::-1], r)


def test_numpy_transcription_bitwise():
    a = si.jacobi3d_grid(13, 7, 9, ldx=16)
    assert np.array_equal(oracle.jacobi3d(a, 7, nx=13), numpy_ref.jacobi3d(a, 7, nx=13))


def test_flop_count_six():
    tally = [0]
    vals = [scalar.FlopCounter(float(i), tally) for i in range(6)]
    scalar.jacobi3d_point(*vals, 6.0)
    assert tally[0] == 6  # PAPER.md:214 "six floating point operations required per grid cell"


def test_divide_is_not_reciprocal_multiply():
    # R21: "/ 6.0" and "* (1/6)" differ in the last bit for some sums; the oracle divides
    s = 0.1 + 0.2 + 0.3 + 0.4 + 0.5 + 0.7
    a = np.zeros((3, 3, 3))
    for k, v in zip([(0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)], [0.1, 0.2, 0.3, 0.4, 0.5, 0.7]):
        a[k] = v
    got = oracle.jacobi3d(a, 1)[1, 1, 1]
    assert got == s / 6.0
    diffs = sum(1 for i in range(1, 2000) if (i * 0.1) / 6.0 != (i * 0.1) * (1.0 / 6.0))
    assert diffs > 0


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_slabs_equal_undecomposed(p):
    a = si.jacobi3d_grid(10, 6, 17)
    assert np.array_equal(oracle.jacobi3d_slabs(a, 9, p), oracle.jacobi3d(a, 9))


@pytest.mark.parametrize("threads", [1, 4])
def test_threads_bitwise(threads):
    a = si.jacobi3d_grid(20, 11, 13)
    assert np.array_equal(oracle.jacobi3d(a, 4, threads=threads), oracle.jacobi3d(a, 4, threads=1))
