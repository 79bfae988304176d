"""CPU oracle for the stencil hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package. The product package
`paper_2310_01882_b200` never imports it and shares no code with it.

Contents
  liboracle.so (oracle.c)  plain C loops, -O2 -ffp-contract=off: or_jacobi2d,
                           or_pw_advect3d, or_pw_points, or_jacobi2d_slabs, or_pw_slabs
  numpy_ref.py             a second, independent NumPy-slicing transcription (pin P8)
  scalar.py                generic per-point formulas over any number type
                           (Fraction brute force J7/P7, flop counting P9)

Every function cites the passage it follows; see oracle.c's header and
DESIGN.md §3 ("Readings of the paper").
"""
from __future__ import annotations

import ctypes
import os
import pathlib

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_dp = ctypes.c_void_p
_i64 = ctypes.c_int64
_dbl = ctypes.c_double


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise RuntimeError(f"{_LIB_PATH} not built; run `make -C {_HERE.parent}`")
    lib = ctypes.CDLL(str(_LIB_PATH))
    lib.or_jacobi2d.restype = ctypes.c_int
    lib.or_jacobi2d.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, ctypes.c_int]
    lib.or_jacobi2d_slabs.restype = ctypes.c_int
    lib.or_jacobi2d_slabs.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]
    pw = [_dp] * 6 + [_i64] * 4 + [_dbl, _dbl] + [_dp] * 4
    lib.or_pw_advect3d.restype = ctypes.c_int
    lib.or_pw_advect3d.argtypes = pw + [ctypes.c_int]
    lib.or_pw_slabs.restype = ctypes.c_int
    lib.or_pw_slabs.argtypes = pw + [ctypes.c_int]
    lib.or_jacobi3d.restype = ctypes.c_int
    lib.or_jacobi3d.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int]
    lib.or_jacobi3d_slabs.restype = ctypes.c_int
    lib.or_jacobi3d_slabs.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int]
    lib.or_pencils_jacobi3d.restype = ctypes.c_int
    lib.or_pencils_jacobi3d.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]
    lib.or_pencils_pw.restype = ctypes.c_int
    lib.or_pencils_pw.argtypes = pw + [ctypes.c_int, ctypes.c_int]
    lib.or_gauss_seidel2d.restype = ctypes.c_int
    lib.or_gauss_seidel2d.argtypes = [_dp, _i64, _i64, _i64, _i64]
    lib.or_pw_points.restype = ctypes.c_int
    lib.or_pw_points.argtypes = [_dp] * 3 + [_i64] * 4 + [_dbl, _dbl] + [_dp] * 4 + [_dp, _i64, _dp]
    lib.or_stencil2d.restype = ctypes.c_int
    lib.or_stencil2d.argtypes = [_dp, _dp, _i64, _i64, _i64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, _i64,
                                 ctypes.c_int]
    _lib = lib
    return lib


def default_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def _check2d(a: np.ndarray):
    assert a.dtype == np.float64 and a.ndim == 2 and a.flags.c_contiguous
    assert a.shape[0] >= 3 and a.shape[1] >= 3


def jacobi2d(a0: np.ndarray, iters: int, nx: int | None = None, threads: int | None = None) -> np.ndarray:
    """Result of `iters` Jacobi sweeps of the padded field a0 ((ny+2) x ld).

    PAPER.md:98-104 (Listing 1) under stencil.apply value semantics.
    a0 is not modified. nx defaults to ld-2 (no pitch padding)."""
    _check2d(a0)
    ny = a0.shape[0] - 2
    ld = a0.shape[1]
    nx = ld - 2 if nx is None else nx
    a = a0.copy()
    b = np.empty_like(a)
    rc = _load().or_jacobi2d(a.ctypes.data, b.ctypes.data, nx, ny, ld, iters,
                             threads or default_threads())
    if rc < 0:
        raise ValueError("or_jacobi2d: bad arguments")
    return b if rc == 1 else a


def jacobi2d_slabs(a0: np.ndarray, iters: int, p: int, h: int = 1, nx: int | None = None) -> np.ndarray:
    """Decomposed oracle: P row slabs, H-deep ghosts swapped every H sweeps."""
    _check2d(a0)
    ny = a0.shape[0] - 2
    ld = a0.shape[1]
    nx = ld - 2 if nx is None else nx
    out = np.zeros_like(a0)
    rc = _load().or_jacobi2d_slabs(np.ascontiguousarray(a0).ctypes.data, out.ctypes.data,
                                   nx, ny, ld, iters, p, h)
    if rc < 0:
        raise ValueError("or_jacobi2d_slabs: bad arguments")
    return out


def jacobi3d(a0: np.ndarray, iters: int, nx: int | None = None, threads: int | None = None) -> np.ndarray:
    """`iters` sweeps of the 3-D 7-point Jacobi (R20/R21) of a
    padded (nz+2, ny+2, ldx) field; a0 is not modified."""
    assert a0.dtype == np.float64 and a0.ndim == 3 and a0.flags.c_contiguous
    nz, ny, ldx = a0.shape[0] - 2, a0.shape[1] - 2, a0.shape[2]
    nx = ldx - 2 if nx is None else nx
    a = a0.copy()
    b = np.empty_like(a)
    rc = _load().or_jacobi3d(a.ctypes.data, b.ctypes.data, nx, ny, nz, ldx, iters, threads or default_threads())
    if rc < 0:
        raise ValueError("or_jacobi3d: bad arguments")
    return b if rc == 1 else a


def jacobi3d_slabs(a0: np.ndarray, iters: int, p: int, nx: int | None = None) -> np.ndarray:
    """z-slab decomposed 3-D Jacobi (1 ghost plane swapped before every sweep)."""
    nz, ny, ldx = a0.shape[0] - 2, a0.shape[1] - 2, a0.shape[2]
    nx = ldx - 2 if nx is None else nx
    out = np.zeros_like(a0)
    rc = _load().or_jacobi3d_slabs(np.ascontiguousarray(a0).ctypes.data, out.ctypes.data, nx, ny, nz, ldx, iters, p)
    if rc < 0:
        raise ValueError("or_jacobi3d_slabs: bad arguments")
    return out


def _pw_args(u, v, w, co, nx):
    for f in (u, v, w):
        assert f.dtype == np.float64 and f.ndim == 3 and f.flags.c_contiguous
        assert f.shape == u.shape
    nz = u.shape[0] - 2
    ny = u.shape[1] - 2
    ldx = u.shape[2]
    nx = ldx - 2 if nx is None else nx
    tz = [np.ascontiguousarray(co[k], dtype=np.float64) for k in ("tzc1", "tzc2", "tzd1", "tzd2")]
    for t in tz:
        assert t.shape == (nz + 2,)
    return nx, ny, nz, ldx, tz


def pw_advect3d(u, v, w, co: dict, nx: int | None = None, threads: int | None = None,
                out: tuple | None = None):
    """(su, sv, sw) of the Piacsek-Williams advection (R6).

    Output halos are zero (or whatever `out` held: they are never written)."""
    nx, ny, nz, ldx, tz = _pw_args(u, v, w, co, nx)
    su, sv, sw = out if out is not None else tuple(np.zeros_like(u) for _ in range(3))
    rc = _load().or_pw_advect3d(u.ctypes.data, v.ctypes.data, w.ctypes.data, su.ctypes.data,
                                sv.ctypes.data, sw.ctypes.data, nx, ny, nz, ldx, co["tcx"],
                                co["tcy"], *[t.ctypes.data for t in tz],
                                threads or default_threads())
    if rc < 0:
        raise ValueError("or_pw_advect3d: bad arguments")
    return su, sv, sw


def pw_points(u, v, w, co: dict, zyx: np.ndarray, nx: int | None = None) -> np.ndarray:
    """Oracle values at sampled interior points: returns (npts, 3) [su, sv, sw]."""
    nx, ny, nz, ldx, tz = _pw_args(u, v, w, co, nx)
    zyx = np.ascontiguousarray(zyx, dtype=np.int64).reshape(-1, 3)
    out = np.empty((zyx.shape[0], 3), dtype=np.float64)
    rc = _load().or_pw_points(u.ctypes.data, v.ctypes.data, w.ctypes.data, nx, ny, nz, ldx,
                              co["tcx"], co["tcy"], *[t.ctypes.data for t in tz],
                              zyx.ctypes.data, zyx.shape[0], out.ctypes.data)
    if rc < 0:
        raise ValueError("or_pw_points: bad arguments / non-interior point")
    return out


def pw_slabs(u, v, w, co: dict, p: int, nx: int | None = None):
    """Decomposed PW oracle: P z-slabs with 1-plane ghost swap."""
    nx, ny, nz, ldx, tz = _pw_args(u, v, w, co, nx)
    su, sv, sw = (np.zeros_like(u) for _ in range(3))
    rc = _load().or_pw_slabs(u.ctypes.data, v.ctypes.data, w.ctypes.data, su.ctypes.data,
                             sv.ctypes.data, sw.ctypes.data, nx, ny, nz, ldx, co["tcx"], co["tcy"],
                             *[t.ctypes.data for t in tz], p)
    if rc < 0:
        raise ValueError("or_pw_slabs: bad arguments")
    return su, sv, sw


def pencils_jacobi3d(a0: np.ndarray, iters: int, py: int, pz: int, nx: int | None = None) -> np.ndarray:
    """3-D Jacobi on a Py x Pz (y, z) process grid, 1-deep ghosts swapped every sweep."""
    nz, ny, ldx = a0.shape[0] - 2, a0.shape[1] - 2, a0.shape[2]
    nx = ldx - 2 if nx is None else nx
    out = np.zeros_like(a0)
    rc = _load().or_pencils_jacobi3d(np.ascontiguousarray(a0).ctypes.data, out.ctypes.data, nx, ny, nz, ldx, iters,
                                     py, pz)
    if rc < 0:
        raise ValueError("or_pencils_jacobi3d: bad arguments")
    return out


def pencils_pw(u, v, w, co: dict, py: int, pz: int, nx: int | None = None):
    """PW advection on a Py x Pz (y, z) process grid; ghosts (incl. y-z corners) come from the swap."""
    nx, ny, nz, ldx, tz = _pw_args(u, v, w, co, nx)
    su, sv, sw = (np.zeros_like(u) for _ in range(3))
    rc = _load().or_pencils_pw(u.ctypes.data, v.ctypes.data, w.ctypes.data, su.ctypes.data, sv.ctypes.data,
                               sw.ctypes.data, nx, ny, nz, ldx, co["tcx"], co["tcy"], *[t.ctypes.data for t in tz],
                               py, pz)
    if rc < 0:
        raise ValueError("or_pencils_pw: bad arguments")
    return su, sv, sw


def gauss_seidel2d(a0: np.ndarray, iters: int, nx: int | None = None) -> np.ndarray:
    """`iters` in-place lexicographic Gauss-Seidel sweeps (Listing 1 literally)."""
    _check2d(a0)
    ny, ld = a0.shape[0] - 2, a0.shape[1]
    nx = ld - 2 if nx is None else nx
    a = a0.copy()
    if _load().or_gauss_seidel2d(a.ctypes.data, nx, ny, ld, iters) < 0:
        raise ValueError("or_gauss_seidel2d: bad arguments")
    return a


def stencil_halo(offsets) -> int:
    """R = max |offset| (input bounds = output bounds widened by the offsets)."""
    return max(max(abs(int(dy)), abs(int(dx))) for dy, dx in offsets)


def stencil2d(a0: np.ndarray, offsets, coeffs, iters: int, nx: int | None = None,
              threads: int | None = None) -> np.ndarray:
    """`iters` sweeps of the generic linear stencil sum_i c_i a(y+dy_i, x+dx_i), left to right
    (reading R23). a0: (ny + 2R) x ld padded field, R = stencil_halo."""
    assert a0.dtype == np.float64 and a0.ndim == 2 and a0.flags.c_contiguous
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 2))
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64))
    assert len(off) == len(c) >= 1
    R = stencil_halo(off)
    ny, ld = a0.shape[0] - 2 * R, a0.shape[1]
    nx = ld - 2 * R if nx is None else nx
    a = a0.copy()
    b = np.empty_like(a)
    rc = _load().or_stencil2d(a.ctypes.data, b.ctypes.data, nx, ny, ld, off.ctypes.data, c.ctypes.data, len(c),
                              iters, threads or default_threads())
    if rc < 0:
        raise ValueError("or_stencil2d: bad arguments")
    return b if rc == 1 else a
