"""Pins of the 2-D Jacobi oracle against things other than itself.

The oracle follows PAPER.md:98-104 (Listing 1) under the value semantics of
stencil.apply. Each pin below is a closed form, an invariant,
a special case, exact-rational brute force or an independent transcription.
"""
import json
import math
import pathlib
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
import stencil_inputs as si
from oracle import numpy_ref, scalar

FACTS = json.loads((pathlib.Path(__file__).parent / "golden" / "paper_facts.json").read_text())
U = 2.0 ** -53  # unit roundoff, binary64


def grid(ny, nx, f):
    return np.array([[f(y, x) for x in range(nx + 2)] for y in range(ny + 2)], dtype=np.float64)


def test_listing_bounds_give_one_cell_ring():
    # PAPER.md:99-101 loops 2..255 over a 1-based array whose bounds (Listing 2,
    # PAPER.md:122) are one cell wider than the output: 254 interior + 1-cell ring.
    l1, l2 = FACTS["listing1"], FACTS["listing2"]
    n_interior = l1["loop_hi"] - l1["loop_lo"] + 1
    assert n_interior == l2["output_ub"] - l2["output_lb"] == 254 - 0
    assert l2["input_ub"] - l2["input_lb"] == n_interior + 2
    assert max(abs(d) for o in l1["offsets_ji"] for d in o) == 1  # halo width 1


def test_J1_single_cell():
    # 1x1 interior; ring N=1 (row 0), S=2 (row 2), W=3 (col 0), E=4 (col 2)
    a = np.zeros((3, 3))
    a[0, 1], a[2, 1], a[1, 0], a[1, 2] = 1.0, 2.0, 3.0, 4.0
    for n in (1, 2, 7):
        r = oracle.jacobi2d(a, n)
        assert r[1, 1] == 2.5
        r[1, 1] = 0.0
        assert np.array_equal(r, a)


@pytest.mark.parametrize("n", [0, 1, 2, 5, 17, 52])
def test_J2_two_by_two_closed_form(n):
    a = np.ones((4, 4))
    a[1:3, 1:3] = 0.0
    r = oracle.jacobi2d(a, n)
    assert np.all(r[1:3, 1:3] == 1.0 - 2.0 ** -n)


@pytest.mark.parametrize("shape,iters", [((1, 1), 3), ((7, 5), 11), ((33, 64), 40), ((66, 3), 9)])
def test_J3_integer_linear_fixed_point(shape, iters):
    ny, nx = shape
    a = grid(ny, nx, lambda y, x: 3 * x + 2 * y + 7)
    assert np.array_equal(oracle.jacobi2d(a, iters), a)
    b = grid(ny, nx, lambda y, x: -5 * x + 11 * y - 3)
    assert np.array_equal(oracle.jacobi2d(b, iters), b)


def test_J4_noninteger_linear_drift_bound():
    a = grid(64, 64, lambda y, x: 0.1 * x + 0.3 * y)
    n = 100
    r = oracle.jacobi2d(a, n)
    # max principle: per-sweep rounding <= 3u * 4max|f| * 0.25 does not amplify
    bound = n * 3 * U * np.abs(a).max() * 2
    assert np.abs(r - a).max() <= bound


def test_J5_constant_and_spec_ones():
    ones = FACTS["spec_ones_4x4"]
    a = np.full((ones["n"], ones["n"]), 1.0)  # 4x4 grid = 2x2 interior + ring
    assert np.all(oracle.jacobi2d(a, 1)[1:-1, 1:-1] == ones["value"])
    c = np.full((20, 31), 6.0)
    assert np.array_equal(oracle.jacobi2d(c, 13), c)


def test_J6_sine_eigenmode_C1():
    nx = ny = 64
    sx = [math.sin(math.pi * x / (nx + 1)) for x in range(nx + 2)]
    sy = [math.sin(math.pi * y / (ny + 1)) for y in range(ny + 2)]
    a = grid(ny, nx, lambda y, x: sy[y] * sx[x])
    a[0, :] = a[-1, :] = a[:, 0] = a[:, -1] = 0.0
    n = 100
    lam = (math.cos(math.pi / (nx + 1)) + math.cos(math.pi / (ny + 1))) / 2
    assert abs(lam ** n - 0.8897225961100627) < 1e-15  # SURVEY.md §8(c5) J6 value
    r = oracle.jacobi2d(a, n)
    assert np.abs(r - lam ** n * a).max() <= 1e-13


def test_J7_exact_rational_brute_force():
    rng = random.Random(7)
    ny, nx, n = 12, 16, 60
    vals = [[Fraction(rng.randrange(-2 ** 20, 2 ** 20), 2 ** 20) for _ in range(nx + 2)] for _ in range(ny + 2)]
    exact = scalar.jacobi2d(vals, n, Fraction(1, 4))
    a = np.array([[float(v) for v in row] for row in vals])
    r = oracle.jacobi2d(a, n)
    amax = max(abs(v) for row in vals for v in row)
    err = max(abs(Fraction(float(r[y, x])) - exact[y][x]) for y in range(ny + 2) for x in range(nx + 2))
    assert err <= 3 * Fraction(U) * n * amax


def test_J8_spec_6x6_seeded_direct_evaluator():
    # 6x6 `seeded:42`, 1 sweep == a 20-line direct evaluator from the snapshot
    a = si.jacobi2d_grid(6, 6)
    snap = a.tolist()
    exp = [row[:] for row in snap]
    for y in range(1, 7):
        for x in range(1, 7):
            exp[y][x] = (snap[y - 1][x] + snap[y + 1][x] + snap[y][x - 1] + snap[y][x + 1]) * 0.25
    assert np.array_equal(oracle.jacobi2d(a, 1), np.array(exp))


def test_J9_y_mirror_symmetry():
    a = si.jacobi2d_grid(23, 17)
    r = oracle.jacobi2d(a, 9)
    rf = oracle.jacobi2d(np.ascontiguousarray(a[::-1]), 9)
    assert np.array_equal(rf[::-1], r)


def test_J10_ring_identity_chunking():
    a = si.jacobi2d_grid(29, 40, ld=44)
    r100 = oracle.jacobi2d(a, 100, nx=40)
    r40 = oracle.jacobi2d(a, 40, nx=40)
    assert np.array_equal(oracle.jacobi2d(r40, 60, nx=40), r100)
    assert np.array_equal(oracle.jacobi2d(a, 0, nx=40), a)
    ring = np.ones_like(a, dtype=bool)
    ring[1:-1, 1:41] = False
    assert np.array_equal(r100[ring], a[ring])  # ring + pitch padding never written


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_threads_bitwise_independent(threads):
    a = si.jacobi2d_grid(50, 61)
    assert np.array_equal(oracle.jacobi2d(a, 7, threads=threads), oracle.jacobi2d(a, 7, threads=1))


def test_P8_numpy_transcription_bitwise():
    a = si.jacobi2d_grid(38, 45, ld=42)
    assert np.array_equal(oracle.jacobi2d(a, 25, nx=38), numpy_ref.jacobi2d(a, 25, nx=38))


def test_P9_flop_count():
    tally = [0]
    vals = [scalar.FlopCounter(float(i), tally) for i in range(4)]
    scalar.jacobi_point(*vals, 0.25)
    assert tally[0] == 4  # 3 adds + 1 multiply per point (Listing 1)
