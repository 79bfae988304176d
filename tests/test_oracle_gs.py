"""Pins of the in-place (lexicographic) Gauss-Seidel oracle — Listing 1 taken
literally (the loop nest overwrites `data` in place, i outer,
j inner). SURVEY.md §8(f) NEXT #4."""
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
import stencil_inputs as si
from oracle import scalar

U = 2.0 ** -53


def test_first_sweep_2x2_by_hand():
    # interior 0, ring 1; lexicographic: (1,1) sees old neighbours, (1,2) sees new (1,1), ...
    a = np.ones((4, 4))
    a[1:3, 1:3] = 0.0
    r = oracle.gauss_seidel2d(a, 1)
    assert r[1, 1] == 0.5          # ((1 + 0) + 1) + 0 = 2   -> 0.5
    assert r[1, 2] == 0.625        # ((1 + 0) + 0.5) + 1     -> 0.625
    assert r[2, 1] == 0.625        # ((0.5 + 1) + 1) + 0     -> 0.625
    assert r[2, 2] == 0.8125       # ((0.625 + 1) + 0.625) + 1 -> 0.8125


def test_single_cell_and_constant():
    a = np.zeros((3, 3))
    a[0, 1], a[2, 1], a[1, 0], a[1, 2] = 1.0, 2.0, 3.0, 4.0
    assert oracle.gauss_seidel2d(a, 5)[1, 1] == 2.5
    c = np.full((9, 12), 3.0)
    assert np.array_equal(oracle.gauss_seidel2d(c, 7), c)


@pytest.mark.parametrize("shape,iters", [((5, 7), 9), ((33, 20), 25)])
def test_integer_linear_fixed_point(shape, iters):
    ny, nx = shape
    y, x = np.mgrid[0:ny + 2, 0:nx + 2]
    a = (4 * x - 3 * y + 11).astype(np.float64)
    assert np.array_equal(oracle.gauss_seidel2d(a, iters), a)


def test_exact_rational_brute_force():
    rng = random.Random(5)
    ny, nx, n = 9, 12, 30
    vals = [[Fraction(rng.randrange(-2 ** 20, 2 ** 20), 2 ** 20) for _ in range(nx + 2)] for _ in range(ny + 2)]
    exact = scalar.gauss_seidel2d(vals, n, Fraction(1, 4))
    r = oracle.gauss_seidel2d(np.array([[float(v) for v in row] for row in vals]), n)
    amax = max(abs(v) for row in vals for v in row)
    err = max(abs(Fraction(float(r[y, x])) - exact[y][x]) for y in range(ny + 2) for x in range(nx + 2))
    assert err <= 3 * Fraction(U) * n * amax


def test_python_transcription_bitwise():
    a = si.jacobi2d_grid(14, 11)
    want = scalar.gauss_seidel2d(a.tolist(), 6, 0.25)
    assert np.array_equal(oracle.gauss_seidel2d(a, 6), np.array(want))


def test_differs_from_jacobi_and_converges_faster():
    # GS is not Jacobi: same fixed point, faster convergence (spectral radius ~ lambda_J^2)
    nx = ny = 30
    a = np.zeros((ny + 2, nx + 2))
    a[0, :] = 1.0
    gs = oracle.gauss_seidel2d(a, 200)
    ja = oracle.jacobi2d(a, 200)
    assert not np.array_equal(gs, ja)
    ref = oracle.gauss_seidel2d(a, 5000)
    assert np.abs(gs - ref).max() < np.abs(ja - ref).max()
