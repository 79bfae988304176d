"""Pins of the PW-advection oracle.

PAPER.md:216 names the Piacsek-Williams scheme [pwadvection] as used by MONC,
"three separate stencil computations across three fields" fused into one
region, "63 floating point operations required per grid cell", but prints no
formula; R6 reads it as the MONC pwadvection form. These pins fix
that reading from outside the oracle: closed forms for linear and constant
fields, the scheme's defining discrete kinetic-energy conservation, the flop
count, exact-rational brute force and an independent transcription.
"""
import itertools
import json
import pathlib
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
import stencil_inputs as si
from oracle import numpy_ref, scalar

FACTS = json.loads((pathlib.Path(__file__).parent / "golden" / "paper_facts.json").read_text())
U = 2.0 ** -53


def coefs(nz, tcx=0.25, tcy=0.5, c1=0.125, c2=0.125, d1=0.375, d2=0.375):
    return {"tcx": tcx, "tcy": tcy, "tzc1": np.full(nz + 2, c1), "tzc2": np.full(nz + 2, c2),
            "tzd1": np.full(nz + 2, d1), "tzd2": np.full(nz + 2, d2)}


def field(nz, ny, nx, f):
    z, y, x = np.meshgrid(np.arange(nz + 2), np.arange(ny + 2), np.arange(nx + 2), indexing="ij")
    return np.ascontiguousarray(f(z, y, x).astype(np.float64))


def interior(a):
    return a[1:-1, 1:-1, 1:-1]


def test_P1_zero():
    z = np.zeros((6, 7, 8))
    for s in oracle.pw_advect3d(z, z.copy(), z.copy(), coefs(4)):
        assert np.all(s == 0) and not np.any(np.signbit(s))


def test_P2_constant_fields_exact_zero_detects_contraction():
    nz, ny, nx = 5, 6, 7
    u = np.full((nz + 2, ny + 2, nx + 2), 0.1)
    v = np.full_like(u, 0.3)
    w = np.full_like(u, 0.7)
    co = si.pw_coefficients(nz)
    co["tzc2"] = co["tzc1"].copy()
    co["tzd2"] = co["tzd1"].copy()
    for s in oracle.pw_advect3d(u, v, w, co):
        assert np.all(interior(s) == 0.0) and not np.any(np.signbit(interior(s)))
    # with unequal z coefficients the constant-field source is genuinely nonzero
    co2 = si.pw_coefficients(nz)
    su, _, _ = oracle.pw_advect3d(u, v, w, co2)
    assert np.abs(interior(su)).max() > 1e-3


@pytest.mark.parametrize("a", [1, 3, -2])
def test_P3_linear_self_advection(a):
    nz, ny, nx = 6, 5, 7
    co = coefs(nz, tcx=0.25, tcy=0.5, d1=0.375, d2=0.375)
    zero = np.zeros((nz + 2, ny + 2, nx + 2))
    X = field(nz, ny, nx, lambda z, y, x: a * x)
    Y = field(nz, ny, nx, lambda z, y, x: a * y)
    Z = field(nz, ny, nx, lambda z, y, x: a * z)
    su, sv, sw = oracle.pw_advect3d(X, zero, zero, co)
    assert np.array_equal(interior(su), interior(-6 * co["tcx"] * a * a * X / a))
    assert np.all(interior(sv) == 0) and np.all(interior(sw) == 0)
    su, sv, sw = oracle.pw_advect3d(zero, Y, zero, co)
    assert np.array_equal(interior(sv), interior(-6 * co["tcy"] * a * a * Y / a))
    assert np.all(interior(su) == 0) and np.all(interior(sw) == 0)
    su, sv, sw = oracle.pw_advect3d(zero, zero, Z, co)
    assert np.array_equal(interior(sw), interior(-6 * 0.375 * a * a * Z / a))
    assert np.all(interior(su) == 0) and np.all(interior(sv) == 0)


# (advected field A, transporting field B, coordinate d): s_A = -2*coef_d*b*c
MIXED = [("u", "v", "y"), ("u", "w", "z"), ("v", "u", "x"), ("v", "w", "z"), ("w", "u", "x"), ("w", "v", "y")]


@pytest.mark.parametrize("A,B,d", MIXED)
def test_P4_cross_field_terms(A, B, d):
    nz, ny, nx = 5, 6, 4
    c, b = 3.0, 2.0
    co = coefs(nz, tcx=0.25, tcy=0.5, c1=0.125, c2=0.125, d1=0.375, d2=0.375)
    coord = {"x": lambda z, y, x: x, "y": lambda z, y, x: y, "z": lambda z, y, x: z}[d]
    flds = {k: np.zeros((nz + 2, ny + 2, nx + 2)) for k in "uvw"}
    flds[A] = np.full((nz + 2, ny + 2, nx + 2), c)
    flds[B] = field(nz, ny, nx, lambda z, y, x: b * coord(z, y, x))
    out = dict(zip("uvw", oracle.pw_advect3d(flds["u"], flds["v"], flds["w"], co)))
    coef = {"x": co["tcx"], "y": co["tcy"], "z": 0.125}[d]
    assert np.all(interior(out[A]) == -2 * coef * b * c)


def periodic(a):
    """Fill the 1-cell halo periodically from the interior (all three axes)."""
    a = a.copy()
    for ax in range(3):
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        src_lo = [slice(None)] * 3
        src_hi = [slice(None)] * 3
        sl_lo[ax], src_lo[ax] = 0, -2
        sl_hi[ax], src_hi[ax] = -1, 1
        a[tuple(sl_lo)] = a[tuple(src_lo)]
        a[tuple(sl_hi)] = a[tuple(src_hi)]
    return a


def test_P5_kinetic_energy_conservation():
    nz, ny, nx = 6, 7, 8
    d = si.pw_inputs(nx, ny, nz, seed=5)
    u, v, w = (periodic(d[k]) for k in "uvw")
    co = coefs(nz, tcx=d["tcx"], tcy=d["tcy"], c1=0.3, c2=0.3, d1=0.3, d2=0.3)
    su, sv, sw = oracle.pw_advect3d(u, v, w, co)
    terms = interior(u * su) + interior(v * sv) + interior(w * sw)
    scale = np.abs(interior(u * su)).sum() + np.abs(interior(v * sv)).sum() + np.abs(interior(w * sw)).sum()
    assert scale > 1.0
    assert abs(terms.sum()) <= 1e-13 * scale
    # the invariant is sensitive: a perturbation of one output breaks it
    su_bad = su.copy()
    su_bad[1:-1, 1:-1, 1:-1] += 0.05 * interior(v)
    bad = (interior(u * su_bad) + interior(v * sv) + interior(w * sw)).sum()
    assert abs(bad) > 1e-6 * scale


def footprint():
    """Which input cells (field, dz, dy, dx) each output reads, by perturbation on a 5^3 grid."""
    nz = ny = nx = 3
    d = si.pw_inputs(nx, ny, nz, seed=11)
    base = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    c = (2, 2, 2)
    res = {k: set() for k in "uvw"}
    for name in "uvw":
        for dz, dy, dx in itertools.product((-1, 0, 1), repeat=3):
            pert = {k: d[k].copy() for k in "uvw"}
            pert[name][c[0] + dz, c[1] + dy, c[2] + dx] += 0.375
            out = oracle.pw_advect3d(pert["u"], pert["v"], pert["w"], d)
            for k, o, b in zip("uvw", out, base):
                if o[c] != b[c]:
                    res[k].add((name, dz, dy, dx))
    return res


def test_P6_influence_set_matches_footprint():
    fp = footprint()
    # union footprint per input field, as (dz: [(dy,dx)])
    want = {
        "u": {-1: [(0, 0)], 0: [(-1, 0), (0, -1), (0, 0), (0, 1), (1, -1), (1, 0)], 1: [(0, -1), (0, 0)]},
        "v": {-1: [(0, 0)], 0: [(-1, 0), (-1, 1), (0, -1), (0, 0), (0, 1), (1, 0)], 1: [(-1, 0), (0, 0)]},
        "w": {-1: [(0, 0), (0, 1), (1, 0)], 0: [(-1, 0), (0, -1), (0, 0), (0, 1), (1, 0)], 1: [(0, 0)]},
    }
    union = fp["u"] | fp["v"] | fp["w"]
    got = {f: {} for f in "uvw"}
    for f, dz, dy, dx in union:
        got[f].setdefault(dz, []).append((dy, dx))
    got = {f: {k: sorted(v) for k, v in g.items()} for f, g in got.items()}
    assert got == want
    assert sum(len(v) for g in want.values() for v in g.values()) == 27
    # every output depends on 15 distinct input cells
    assert [len(fp[k]) for k in "uvw"] == [15, 15, 15]


class AbsNum:
    """Evaluates |e| with every '-' turned into '+' (the forward-error scale of an expression)."""

    def __init__(self, v):
        self.v = abs(Fraction(v))

    def __add__(self, o): return AbsNum(self.v + _v(o))
    __radd__ = __add__
    def __sub__(self, o): return AbsNum(self.v + _v(o))
    def __rsub__(self, o): return AbsNum(self.v + _v(o))
    def __mul__(self, o): return AbsNum(self.v * _v(o))
    __rmul__ = __mul__


def _v(o):
    return o.v if isinstance(o, AbsNum) else abs(Fraction(o))


def test_P7_exact_rational_brute_force():
    nz, ny, nx = 4, 5, 6
    d = si.pw_inputs(nx, ny, nz, seed=3)
    su, sv, sw = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    exact = scalar.pw_advect3d(d["u"], d["v"], d["w"], d, conv=Fraction)
    scale = scalar.pw_advect3d(d["u"], d["v"], d["w"], d, conv=AbsNum)
    worst = Fraction(0)
    for (z, y, x), vals in exact.items():
        for k, (o, e) in enumerate(zip((su, sv, sw), vals)):
            err = abs(Fraction(float(o[z, y, x])) - e)
            bound = 8 * Fraction(U) * scale[(z, y, x)][k].v
            assert err <= bound
            worst = max(worst, err / bound if bound else 0)
    assert worst < 1


def test_P8_numpy_transcription_bitwise():
    nz, ny, nx = 9, 13, 11
    d = si.pw_inputs(nx, ny, nz, ldx=14)
    a = oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx)
    b = numpy_ref.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_P9_flop_count_63():
    tally = [0]
    acc = lambda dz, dy, dx: scalar.FlopCounter(0.5 + dz + 0.1 * dy + 0.01 * dx, tally)
    scalar.pw_point(acc, acc, acc, 1, 0.25, 0.5, 0.1, 0.2, 0.3, 0.4)
    assert tally[0] == FACTS["flops_per_cell"]["pw_advection"] == 63


def test_pw_points_sampled_equals_full():
    nz, ny, nx = 7, 6, 9
    d = si.pw_inputs(nx, ny, nz)
    full = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    rng = np.random.default_rng(0)
    pts = np.stack([rng.integers(1, n + 1, 40) for n in (nz, ny, nx)], axis=1)
    got = oracle.pw_points(d["u"], d["v"], d["w"], d, pts)
    for k in range(3):
        assert np.array_equal(got[:, k], full[k][pts[:, 0], pts[:, 1], pts[:, 2]])


def test_halos_of_outputs_untouched():
    nz, ny, nx = 3, 4, 5
    d = si.pw_inputs(nx, ny, nz, ldx=8)
    out = tuple(np.full_like(d["u"], 7.0) for _ in range(3))
    oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx, out=out)
    for s in out:
        m = np.ones_like(s, dtype=bool)
        m[1:-1, 1:-1, 1:nx + 1] = False
        assert np.all(s[m] == 7.0)


def test_P3b_vertical_coefficients_placement():
    # tzd1 weights the lower (z-1) flux and tzd2 the upper (z+1) one: w = a*z gives
    # sw = a^2 * (d1*(z-1)*(2z-1) - d2*(z+1)*(2z+1)) exactly (small integers, dyadic d1, d2)
    nz, ny, nx, a = 6, 3, 4, 3
    d1, d2 = 0.375, 0.625
    co = coefs(nz, d1=d1, d2=d2)
    zero = np.zeros((nz + 2, ny + 2, nx + 2))
    Z = field(nz, ny, nx, lambda z, y, x: a * z)
    _, _, sw = oracle.pw_advect3d(zero, zero, Z, co)
    z = np.arange(1, nz + 1)[:, None, None]
    want = a * a * (d1 * (z - 1) * (2 * z - 1) - d2 * (z + 1) * (2 * z + 1))
    assert np.array_equal(interior(sw), np.broadcast_to(want, (nz, ny, nx)))


@pytest.mark.parametrize("A", ["u", "v"])
def test_P4b_cross_vertical_coefficients_placement(A):
    # A == c, w = b*z: s_A = (c1*c)*(2b(z-1)) - (c2*c)*(2bz) with tzc1 != tzc2
    nz, ny, nx, b, c = 5, 4, 3, 2.0, 3.0
    c1, c2 = 0.125, 0.375
    co = coefs(nz, c1=c1, c2=c2)
    flds = {k: np.zeros((nz + 2, ny + 2, nx + 2)) for k in "uvw"}
    flds[A] = np.full((nz + 2, ny + 2, nx + 2), c)
    flds["w"] = field(nz, ny, nx, lambda z, y, x: b * z)
    out = dict(zip("uvw", oracle.pw_advect3d(flds["u"], flds["v"], flds["w"], co)))
    z = np.arange(1, nz + 1)[:, None, None]
    want = (c1 * c) * (2 * b * (z - 1)) - (c2 * c) * (2 * b * z)
    assert np.array_equal(interior(out[A]), np.broadcast_to(want, (nz, ny, nx)))
