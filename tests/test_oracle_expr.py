"""Pins of the expression-stencil oracle (reading R24): Listing 1 written as an
expression equals the pinned C Jacobi oracle bitwise; linear expressions equal
the C generic-stencil oracle bitwise; nonlinear expressions on integer data equal
exact rational evaluation; the parser rejects anything but accesses, literals,
+ - * / and parentheses."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import expr as ox

rng = np.random.default_rng(149)


def test_listing1_expression_equals_jacobi_oracle():
    # Listing 1: data(j,i-1)+data(j,i+1)+data(j-1,i)+data(j+1,i) with j = x, i = y
    e = "(a(-1,0) + a(1,0) + a(0,-1) + a(0,1)) * 0.25"
    a = rng.standard_normal((35, 41))
    assert np.array_equal(ox.stencil2d_expr(a, e, 7), oracle.jacobi2d(a, 7))


def test_linear_expression_equals_generic_oracle():
    offs = [(2, -1), (0, 0), (-1, 2), (1, 1)]
    coefs = [0.3, -0.7, 0.125, 1.5]
    e = " + ".join(f"{c!r}*a({dy},{dx})" for (dy, dx), c in zip(offs, coefs))
    a = rng.standard_normal((30, 33))
    assert np.array_equal(ox.stencil2d_expr(a, e, 4), oracle.stencil2d(a, offs, coefs, 4))


@pytest.mark.parametrize("e", [
    "a(0,1)*a(0,-1) - a(1,0)",
    "-(a(1,1) - 2*a(0,0)) * (a(-1,-1) + 3)",
    "(a(0,0) + a(2,0))*(a(0,0) - a(-2,0)) - a(0,2)*4",
])
def test_nonlinear_exact_rationals(e):
    # integer data, one sweep: every intermediate is an exact small integer in binary64
    R = ox.halo(e)
    a = rng.integers(-9, 10, size=(6 + 2 * R, 7 + 2 * R)).astype(np.float64)
    got = ox.stencil2d_expr(a, e, 1)
    want = a.copy()
    for y in range(R, R + 6):
        for x in range(R, R + 7):
            want[y, x] = float(ox.eval_exact(e, lambda dy, dx: Fraction(a[y + dy, x + dx])))
    assert np.array_equal(got, want)


def test_division_and_literals_are_binary64():
    # 1/3 is float division (not C integer division) and literals are binary64 nearest
    a = np.full((3, 3), 3.0)
    got = ox.stencil2d_expr(a, "a(0,0) * (1/3) + 0.1", 1)
    assert got[1, 1] == 3.0 * (1.0 / 3.0) + 0.1


@pytest.mark.parametrize("bad", ["a(0,0) ** 2", "a(0,0) if 1 else 0", "b(0,0)", "a(0,0); import os",
                                 "abs(a(0,0))", "a(0,0) % 2", "a(0)"])
def test_rejects_unsupported_syntax(bad):
    with pytest.raises((ValueError, SyntaxError)):
        ox.stencil2d_expr(np.zeros((5, 5)), bad, 1)


def test_ring_fixed_and_offsets_parsed():
    e = "a(-3,1) + 0.5*a(2,-2)"
    assert ox.offsets(e) == [(-3, 1), (2, -2)] and ox.halo(e) == 3
    a = rng.standard_normal((20, 18))
    got = ox.stencil2d_expr(a, e, 3)
    mask = np.ones_like(a, dtype=bool)
    mask[3:-3, 3:-3] = False
    assert np.array_equal(got[mask], a[mask])


def test_benchmark1_expression_equals_jacobi3d_oracle():
    # the paper's benchmark 1 as an expression: readings R20/R21 exactly
    e = "(a(-1,0,0) + a(1,0,0) + a(0,-1,0) + a(0,1,0) + a(0,0,-1) + a(0,0,1)) / 6"
    a = rng.standard_normal((9, 11, 14))
    assert np.array_equal(ox.stencil3d_expr(a, e, 4), oracle.jacobi3d(a, 4))


def test_3d_nonlinear_exact_rationals():
    e = "a(1,0,-1)*a(0,2,0) - 3*a(-1,-1,1)"
    R = ox.halo3(e)
    a = rng.integers(-5, 6, size=(3 + 2 * R, 4 + 2 * R, 5 + 2 * R)).astype(np.float64)
    got = ox.stencil3d_expr(a, e, 1)
    want = a.copy()
    for z in range(R, R + 3):
        for y in range(R, R + 4):
            for x in range(R, R + 5):
                want[z, y, x] = float(ox.eval_exact(e, lambda dz, dy, dx: Fraction(a[z + dz, y + dy, x + dx])))
    assert np.array_equal(got, want)


def test_fused_pw_region_equals_pw_oracle():
    # benchmark 2 written as one fused region of three expressions evaluates
    # bitwise like the hand-written C PW oracle (the expressions come from the product's helper;
    # the reference is or_pw_advect3d, so the two sides share nothing)
    import paper_2310_01882_b200 as st
    import stencil_inputs as si
    d = si.pw_inputs(23, 17, 11)
    exprs = st.pw_fused_expressions(d["tcx"], d["tcy"])
    got = ox.fused3d_expr([d["u"], d["v"], d["w"]], exprs, [d["tzc1"], d["tzc2"], d["tzd1"], d["tzd2"]], nx=23)
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    for g, w in zip(got, want):
        assert np.array_equal(g[1:-1, 1:-1, 1:24], w[1:-1, 1:-1, 1:24])


def test_fused_integer_exact_and_grammar():
    e = ["f0(1,0,0)*k1 - f1(0,-1,1)", "2*f1(0,0,0) + f0(-1,1,-1)*f0(0,0,0)*k0"]
    a = [rng.integers(-6, 7, size=(5, 6, 7)).astype(np.float64) for _ in range(2)]
    k = [rng.integers(-3, 4, size=5).astype(np.float64) for _ in range(2)]
    got = ox.fused3d_expr(a, e, k)
    for j, ej in enumerate(e):
        want = np.zeros_like(a[0])
        for z in range(1, 4):
            for y in range(1, 5):
                for x in range(1, 6):
                    env = {"f0": lambda dz, dy, dx: Fraction(a[0][z + dz, y + dy, x + dx]),
                           "f1": lambda dz, dy, dx: Fraction(a[1][z + dz, y + dy, x + dx]),
                           "k0": Fraction(k[0][z]), "k1": Fraction(k[1][z])}
                    want[z, y, x] = float(eval(ej, {"__builtins__": {}}, env))
        assert np.array_equal(got[j], want)
    for bad in ["a(0,0,0)", "f8(0,0,0)", "k9", "f0(0,0)", "f0(0,0,0)**2"]:
        with pytest.raises((ValueError, SyntaxError)):
            ox.fused3d_expr(a, [bad], k)
