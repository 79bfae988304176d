"""Pins of the generic linear stencil.apply oracle (reading R23 of DESIGN.md;
PAPER.md:107-126 apply/access, PAPER.md:149-191/185 offsets of the discovered
loop nest, SPEC.md:197-205 halo = max |offset|). Each pin is fixed by something
other than the oracle's own formula: exact rational arithmetic, closed forms of
special stencils, a rounding-order witness, invariants and an independent NumPy
transcription."""
from fractions import Fraction

import numpy as np
import pytest

import oracle

rng = np.random.default_rng(2310)


def padded(ny, nx, R, fill=None, ld=None):
    ld = nx + 2 * R if ld is None else ld
    if fill is None:
        return rng.standard_normal((ny + 2 * R, ld))
    return np.full((ny + 2 * R, ld), fill, dtype=np.float64)


def test_identity_stencil_is_identity():
    a = padded(7, 9, 0 + 1)
    for it in (0, 1, 4):
        assert np.array_equal(oracle.stencil2d(a, [(0, 0), (1, 1)], [1.0, 0.0], it), a)


def test_shift_stencil_closed_form():
    # out_k(y, x) = a(y, min(x + k, nx + R - 1 + 1)): the interior slides left by one column per
    # sweep; the right ring column (x = nx + R) is fixed and feeds the last interior columns
    ny, nx, R = 5, 11, 1
    a = padded(ny, nx, R)
    for k in (1, 2, 5):
        got = oracle.stencil2d(a, [(0, 1)], [1.0], k)
        want = a.copy()
        for x in range(R, R + nx):
            want[R:R + ny, x] = a[R:R + ny, min(x + k, nx + R)]
        assert np.array_equal(got, want)


def test_exact_rational_brute_force_random_stencils():
    # integer inputs and dyadic/integer coefficients keep every product and partial sum
    # exact in binary64, so the oracle must equal exact rational arithmetic bitwise —
    # any wrong offset sign, (dy, dx) transposition or dropped term fails
    for trial in range(12):
        n = int(rng.integers(1, 6))
        R = int(rng.integers(1, 3))
        offs = [(int(rng.integers(-R, R + 1)), int(rng.integers(-R, R + 1))) for _ in range(n)]
        offs[0] = (R, -R) if trial % 2 else offs[0]  # make sure the halo really is R
        coefs = [float(rng.choice([1.0, -1.0, 2.0, 0.5, -0.25])) for _ in range(n)]
        ny, nx = int(rng.integers(1, 6)), int(rng.integers(1, 7))
        Rr = oracle.stencil_halo(offs)
        a = rng.integers(-8, 9, size=(ny + 2 * Rr, nx + 2 * Rr)).astype(np.float64)
        iters = 3
        got = oracle.stencil2d(a, offs, coefs, iters)
        cur = [[Fraction(v) for v in row] for row in a.tolist()]
        for _ in range(iters):
            nxt = [row[:] for row in cur]
            for y in range(Rr, Rr + ny):
                for x in range(Rr, Rr + nx):
                    nxt[y][x] = sum(Fraction(c) * cur[y + dy][x + dx] for (dy, dx), c in zip(offs, coefs))
            cur = nxt
        assert np.array_equal(got, np.array([[float(v) for v in row] for row in cur]))


def test_left_to_right_order_witness():
    # c = (1, 1, 1) on values (1e17, 1, -1e17): the exact sum is 1, but Fortran's
    # left-to-right order rounds 1e17 + 1 to 1e17 first (ulp 16), so the stencil result is exactly 0
    b = np.zeros((5, 5))
    b[2, 0], b[2, 2], b[2, 4] = 1e17, 1.0, -1e17
    got = oracle.stencil2d(b, [(0, -2), (0, 0), (0, 2)], [1.0, 1.0, 1.0], 1)
    assert got[2, 2] == 0.0
    # the order (1e17, -1e17, 1) gives the exact 1
    got = oracle.stencil2d(b, [(0, -2), (0, 2), (0, 0)], [1.0, 1.0, 1.0], 1)
    assert got[2, 2] == 1.0


def test_ring_invariance_iters_zero_and_chunking():
    offs = [(-2, 0), (0, 1), (1, -1), (0, 0)]
    coefs = [0.3, 0.2, 0.1, 0.4]
    R = oracle.stencil_halo(offs)
    a = padded(13, 17, R)
    r5 = oracle.stencil2d(a, offs, coefs, 5)
    mask = np.ones_like(a, dtype=bool)
    mask[R:R + 13, R:R + 17] = False
    assert np.array_equal(r5[mask], a[mask])
    assert np.array_equal(oracle.stencil2d(a, offs, coefs, 0), a)
    assert np.array_equal(oracle.stencil2d(oracle.stencil2d(a, offs, coefs, 2), offs, coefs, 3), r5)


def numpy_transcription(a, offs, coefs, iters, nx=None):
    R = oracle.stencil_halo(offs)
    ny = a.shape[0] - 2 * R
    nx = a.shape[1] - 2 * R if nx is None else nx
    cur = a.copy()
    for _ in range(iters):
        nxt = cur.copy()
        acc = None
        for (dy, dx), c in zip(offs, coefs):
            t = c * cur[R + dy:R + dy + ny, R + dx:R + dx + nx]
            acc = t if acc is None else acc + t
        nxt[R:R + ny, R:R + nx] = acc
        cur = nxt
    return cur


@pytest.mark.parametrize("offs", [
    [(-1, 0), (1, 0), (0, -1), (0, 1)],
    [(0, 0), (-2, 0), (2, 0), (0, -2), (0, 2), (-1, -1), (1, 1), (-1, 1), (1, -1)],
    [(3, -2), (-1, 3), (0, 0)],
])
def test_numpy_transcription_bitwise(offs):
    coefs = list(rng.standard_normal(len(offs)))
    R = oracle.stencil_halo(offs)
    a = padded(19, 23, R, ld=23 + 2 * R + 3)
    nx = 23
    assert np.array_equal(oracle.stencil2d(a, offs, coefs, 4, nx=nx)[:, :nx + 2 * R],
                          numpy_transcription(a[:, :nx + 2 * R].copy(), offs, coefs, 4)[:, :nx + 2 * R])


def test_listing1_within_rounding_of_the_generic_form():
    # Listing 1 ((N+S)+W)+E)*0.25 and the generic 0.25N + 0.25S + 0.25W + 0.25E agree in exact
    # arithmetic; in binary64 within a few ulps per sweep (different rounding order)
    a = padded(30, 40, 1) + 2.0
    j = oracle.jacobi2d(a, 10)
    g = oracle.stencil2d(a, [(-1, 0), (1, 0), (0, -1), (0, 1)], [0.25] * 4, 10)
    assert np.max(np.abs(j - g)) <= 10 * 4 * 2.0 ** -53 * np.max(np.abs(a))
