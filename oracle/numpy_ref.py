"""Second, independent transcription of the oracle with NumPy slicing (pin P8).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Written directly from the
paper's statements — PAPER.md:98-104 (Listing 1), PAPER.md:126 (value
semantics) and PAPER.md:216 (PW advection, formula reading R6 of DESIGN.md) —
without looking at oracle.c's loops, so that a transcription slip in either
shows up as a bitwise mismatch. NumPy elementwise ops on float64 round once
per op, in the order written, and never contract.
"""
from __future__ import annotations

import numpy as np


def jacobi2d_sweep(a: np.ndarray, nx: int) -> np.ndarray:
    """One Jacobi sweep of the padded (ny+2) x ld field; ring copied unchanged."""
    b = a.copy()
    north = a[:-2, 1:nx + 1]
    south = a[2:, 1:nx + 1]
    west = a[1:-1, 0:nx]
    east = a[1:-1, 2:nx + 2]
    b[1:-1, 1:nx + 1] = (((north + south) + west) + east) * 0.25
    return b


def jacobi2d(a0: np.ndarray, iters: int, nx: int | None = None) -> np.ndarray:
    nx = a0.shape[1] - 2 if nx is None else nx
    a = a0.copy()
    for _ in range(iters):
        a = jacobi2d_sweep(a, nx)
    return a


def pw_advect3d(u, v, w, co, nx: int | None = None):
    """Slicing form of the PW advection; returns (su, sv, sw) with zero halos."""
    nz, ny = u.shape[0] - 2, u.shape[1] - 2
    nx = u.shape[2] - 2 if nx is None else nx

    def S(f, dz, dy, dx):
        return f[1 + dz:nz + 1 + dz, 1 + dy:ny + 1 + dy, 1 + dx:nx + 1 + dx]

    tcx, tcy = co["tcx"], co["tcy"]
    c1 = co["tzc1"][1:nz + 1, None, None]
    c2 = co["tzc2"][1:nz + 1, None, None]
    d1 = co["tzd1"][1:nz + 1, None, None]
    d2 = co["tzd2"][1:nz + 1, None, None]

    # su: advection of u by u (x), v (y), w (z)
    xu = tcx * (S(u, 0, 0, -1) * (S(u, 0, 0, 0) + S(u, 0, 0, -1))
                - S(u, 0, 0, 1) * (S(u, 0, 0, 0) + S(u, 0, 0, 1)))
    yu = tcy * (S(u, 0, -1, 0) * (S(v, 0, -1, 0) + S(v, 0, -1, 1))
                - S(u, 0, 1, 0) * (S(v, 0, 0, 0) + S(v, 0, 0, 1)))
    zu = ((c1 * S(u, -1, 0, 0)) * (S(w, -1, 0, 0) + S(w, -1, 0, 1))
          - (c2 * S(u, 1, 0, 0)) * (S(w, 0, 0, 0) + S(w, 0, 0, 1)))
    # sv
    xv = tcx * (S(v, 0, 0, -1) * (S(u, 0, 0, -1) + S(u, 0, 1, -1))
                - S(v, 0, 0, 1) * (S(u, 0, 0, 0) + S(u, 0, 1, 0)))
    yv = tcy * (S(v, 0, -1, 0) * (S(v, 0, 0, 0) + S(v, 0, -1, 0))
                - S(v, 0, 1, 0) * (S(v, 0, 0, 0) + S(v, 0, 1, 0)))
    zv = ((c1 * S(v, -1, 0, 0)) * (S(w, -1, 0, 0) + S(w, -1, 1, 0))
          - (c2 * S(v, 1, 0, 0)) * (S(w, 0, 0, 0) + S(w, 0, 1, 0)))
    # sw
    xw = tcx * (S(w, 0, 0, -1) * (S(u, 0, 0, -1) + S(u, 1, 0, -1))
                - S(w, 0, 0, 1) * (S(u, 0, 0, 0) + S(u, 1, 0, 0)))
    yw = tcy * (S(w, 0, -1, 0) * (S(v, 0, -1, 0) + S(v, 1, -1, 0))
                - S(w, 0, 1, 0) * (S(v, 0, 0, 0) + S(v, 1, 0, 0)))
    zw = ((d1 * S(w, -1, 0, 0)) * (S(w, 0, 0, 0) + S(w, -1, 0, 0))
          - (d2 * S(w, 1, 0, 0)) * (S(w, 0, 0, 0) + S(w, 1, 0, 0)))

    out = []
    for xs, ys, zs in ((xu, yu, zu), (xv, yv, zv), (xw, yw, zw)):
        s = np.zeros_like(u)
        s[1:nz + 1, 1:ny + 1, 1:nx + 1] = (xs + ys) + zs
        out.append(s)
    return tuple(out)


def jacobi3d(a0: np.ndarray, iters: int, nx: int | None = None) -> np.ndarray:
    """3-D 7-point Jacobi by slicing (order z-, z+, y-, y+, x-, x+, then / 6.0)."""
    nx = a0.shape[2] - 2 if nx is None else nx
    a = a0.copy()
    for _ in range(iters):
        b = a.copy()
        s = a[:-2, 1:-1, 1:nx + 1] + a[2:, 1:-1, 1:nx + 1]
        s = s + a[1:-1, :-2, 1:nx + 1]
        s = s + a[1:-1, 2:, 1:nx + 1]
        s = s + a[1:-1, 1:-1, 0:nx]
        s = s + a[1:-1, 1:-1, 2:nx + 2]
        b[1:-1, 1:-1, 1:nx + 1] = s / 6.0
        a = b
    return a
