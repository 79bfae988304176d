"""Generic per-point formulas over any number type — TEST INFRASTRUCTURE ONLY.

Used with `fractions.Fraction` for exact-rational brute force (pins J7, P7)
and with `FlopCounter` to count the floating-point operations per point
(pin P9 against PAPER.md:214/216: "six floating point operations" for the
7-point benchmark, "63 floating point operations required per grid cell" for
PW; the 2-D 5-point sweep of Listing 1 has 4). Pure-Python loops: tiny grids
only.
"""
from __future__ import annotations


class FlopCounter:
    """A number that counts every binary arithmetic op applied to it (shared tally)."""

    __slots__ = ("v", "tally")

    def __init__(self, v, tally):
        self.v = v
        self.tally = tally

    def _op(self, other, fn, reverse=False):
        self.tally[0] += 1
        ov = other.v if isinstance(other, FlopCounter) else other
        return FlopCounter(fn(ov, self.v) if reverse else fn(self.v, ov), self.tally)

    def __add__(self, o): return self._op(o, lambda a, b: a + b)
    def __radd__(self, o): return self._op(o, lambda a, b: a + b, True)
    def __sub__(self, o): return self._op(o, lambda a, b: a - b)
    def __rsub__(self, o): return self._op(o, lambda a, b: a - b, True)
    def __mul__(self, o): return self._op(o, lambda a, b: a * b)
    def __rmul__(self, o): return self._op(o, lambda a, b: a * b, True)
    def __truediv__(self, o): return self._op(o, lambda a, b: a / b)


def jacobi_point(n, s, w, e, quarter):
    """Listing 1: (data(j,i-1)+data(j,i+1)+data(j-1,i)+data(j+1,i)) * 0.25."""
    return (((n + s) + w) + e) * quarter


def jacobi3d_point(zm, zp, ym, yp, xm, xp, six):
    """average of the six orthogonal neighbours (R20/R21)."""
    return (((((zm + zp) + ym) + yp) + xm) + xp) / six


def jacobi3d(a, iters, six):
    """Exact/generic 3-D Jacobi on nested lists a[z][y][x]."""
    nz, ny, nx = len(a) - 2, len(a[0]) - 2, len(a[0][0]) - 2
    cur = [[row[:] for row in pl] for pl in a]
    for _ in range(iters):
        nxt = [[row[:] for row in pl] for pl in cur]
        for z in range(1, nz + 1):
            for y in range(1, ny + 1):
                for x in range(1, nx + 1):
                    nxt[z][y][x] = jacobi3d_point(cur[z - 1][y][x], cur[z + 1][y][x], cur[z][y - 1][x],
                                                  cur[z][y + 1][x], cur[z][y][x - 1], cur[z][y][x + 1], six)
        cur = nxt
    return cur


def jacobi2d(a, iters, quarter):
    """Exact/generic Jacobi on a list-of-lists padded grid (value semantics)."""
    ny, nx = len(a) - 2, len(a[0]) - 2
    cur = [row[:] for row in a]
    for _ in range(iters):
        nxt = [row[:] for row in cur]
        for y in range(1, ny + 1):
            for x in range(1, nx + 1):
                nxt[y][x] = jacobi_point(cur[y - 1][x], cur[y + 1][x], cur[y][x - 1], cur[y][x + 1], quarter)
        cur = nxt
    return cur


def gauss_seidel2d(a, iters, quarter):
    """Listing 1 executed literally (in place, i outer, j inner) on a list-of-lists grid."""
    ny, nx = len(a) - 2, len(a[0]) - 2
    cur = [row[:] for row in a]
    for _ in range(iters):
        for y in range(1, ny + 1):
            for x in range(1, nx + 1):
                cur[y][x] = jacobi_point(cur[y - 1][x], cur[y + 1][x], cur[y][x - 1], cur[y][x + 1], quarter)
    return cur


def pw_point(U, V, W, z, tcx, tcy, tzc1, tzc2, tzd1, tzd2):
    """PW advection at one point (R6). U(dz,dy,dx) etc. are accessors
    relative to the point; tz* are the values at plane z. Returns (su, sv, sw)."""
    su = ((tcx * (U(0, 0, -1) * (U(0, 0, 0) + U(0, 0, -1)) - U(0, 0, 1) * (U(0, 0, 0) + U(0, 0, 1)))
           + tcy * (U(0, -1, 0) * (V(0, -1, 0) + V(0, -1, 1)) - U(0, 1, 0) * (V(0, 0, 0) + V(0, 0, 1))))
          + ((tzc1 * U(-1, 0, 0)) * (W(-1, 0, 0) + W(-1, 0, 1))
             - (tzc2 * U(1, 0, 0)) * (W(0, 0, 0) + W(0, 0, 1))))
    sv = ((tcx * (V(0, 0, -1) * (U(0, 0, -1) + U(0, 1, -1)) - V(0, 0, 1) * (U(0, 0, 0) + U(0, 1, 0)))
           + tcy * (V(0, -1, 0) * (V(0, 0, 0) + V(0, -1, 0)) - V(0, 1, 0) * (V(0, 0, 0) + V(0, 1, 0))))
          + ((tzc1 * V(-1, 0, 0)) * (W(-1, 0, 0) + W(-1, 1, 0))
             - (tzc2 * V(1, 0, 0)) * (W(0, 0, 0) + W(0, 1, 0))))
    sw = ((tcx * (W(0, 0, -1) * (U(0, 0, -1) + U(1, 0, -1)) - W(0, 0, 1) * (U(0, 0, 0) + U(1, 0, 0)))
           + tcy * (W(0, -1, 0) * (V(0, -1, 0) + V(1, -1, 0)) - W(0, 1, 0) * (V(0, 0, 0) + V(1, 0, 0))))
          + ((tzd1 * W(-1, 0, 0)) * (W(0, 0, 0) + W(-1, 0, 0))
             - (tzd2 * W(1, 0, 0)) * (W(0, 0, 0) + W(1, 0, 0))))
    return su, sv, sw


def pw_advect3d(u, v, w, co, conv=lambda x: x):
    """Generic PW over nested lists / arrays u[z][y][x]; returns dict of
    {(z,y,x): (su,sv,sw)} for interior points. `conv` maps stored values into
    the number type (e.g. Fraction)."""
    nz, ny, nx = len(u) - 2, len(u[0]) - 2, len(u[0][0]) - 2
    out = {}
    tcx, tcy = conv(co["tcx"]), conv(co["tcy"])
    for z in range(1, nz + 1):
        for y in range(1, ny + 1):
            for x in range(1, nx + 1):
                def acc(f):
                    return lambda dz, dy, dx: conv(f[z + dz][y + dy][x + dx])
                out[(z, y, x)] = pw_point(acc(u), acc(v), acc(w), z, tcx, tcy,
                                          conv(co["tzc1"][z]), conv(co["tzc2"][z]),
                                          conv(co["tzd1"][z]), conv(co["tzd2"][z]))
    return out
