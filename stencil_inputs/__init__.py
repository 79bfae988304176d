"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO stencil arithmetic: only the counter-based SplitMix64
generator of SURVEY.md §8(d) ("Generator", SPEC.md:486 `seeded:<n>`) and the
input recipes of DESIGN.md §"Input recipe" built on it. Both `oracle/` and
`paper_2310_01882_b200/` consumers receive identical arrays from here; neither
side generates its own values.

The generator is a small C library (`libstinputs.so`, OpenMP) so that
full-size fields (16386^2, 514^3) are produced in well under a second; a pure
NumPy transcription (`u01_numpy`) exists only to cross-check it in tests.
"""
from __future__ import annotations

import ctypes
import os
import pathlib

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libstinputs.so"
_lib = None

GOLDEN_MUL = 0x9E3779B97F4A7C15
STREAM_MUL = 0xD1B54A32D192ED03
MASK64 = (1 << 64) - 1

# Input recipe constants.
SEED = 42
STREAM_JACOBI = 0
STREAM_U, STREAM_V, STREAM_W = 1, 2, 3
STREAM_TZC1, STREAM_TZC2, STREAM_TZD1, STREAM_TZD2 = 4, 5, 6, 7
STREAM_JACOBI3D = 8
PW_TCX = 0.25 / 3.0
PW_TCY = 0.25 / 5.0


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise RuntimeError(
            f"{_LIB_PATH} not built; run `make -C {_HERE.parent}` or __graft_entry__.build()")
    lib = ctypes.CDLL(str(_LIB_PATH))
    lib.sti_raw.restype = ctypes.c_uint64
    lib.sti_raw.argtypes = [ctypes.c_uint64] * 3
    lib.sti_u01.restype = ctypes.c_double
    lib.sti_u01.argtypes = [ctypes.c_uint64] * 3
    lib.sti_fill_affine.restype = ctypes.c_int
    lib.sti_fill_affine.argtypes = [
        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
        ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
        ctypes.c_double, ctypes.c_double]
    _lib = lib
    return lib


def raw(seed: int, stream: int, idx: int) -> int:
    return int(_load().sti_raw(seed, stream, idx))


def u01(seed: int, stream: int, idx: int) -> float:
    return float(_load().sti_u01(seed, stream, idx))


def u01_numpy(seed: int, stream: int, idx) -> np.ndarray:
    """Pure NumPy transcription of the same generator (test cross-check only)."""
    idx = np.asarray(idx, dtype=np.uint64)
    s0 = np.uint64((seed ^ ((stream * STREAM_MUL) & MASK64)) & MASK64)
    with np.errstate(over="ignore"):
        z = s0 + (idx + np.uint64(1)) * np.uint64(GOLDEN_MUL)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def fill_affine(out: np.ndarray, n_outer: int, n_inner: int, out_stride: int,
                idx_base: int, idx_stride: int, seed: int, stream: int,
                scale: float, offset: float) -> None:
    """out.flat[o*out_stride+i] = offset + scale*U01(seed, stream, idx_base+o*idx_stride+i)."""
    assert out.dtype == np.float64 and out.flags.c_contiguous
    assert out.size >= (n_outer - 1) * out_stride + n_inner if n_outer > 0 else True
    rc = _load().sti_fill_affine(out.ctypes.data, n_outer, n_inner, out_stride,
                                 idx_base, idx_stride, seed, stream, scale, offset)
    if rc != 0:
        raise ValueError("sti_fill_affine: bad arguments")


def even_ld(n: int) -> int:
    """Smallest even row pitch >= n (16-byte rows for fp64)."""
    return n + (n & 1)


def jacobi2d_grid(nx: int, ny: int, ld: int | None = None, *, seed: int = SEED,
                  stream: int = STREAM_JACOBI, row0: int = 0, rows: int | None = None,
                  scale: float = 1.0, offset: float = 0.5) -> np.ndarray:
    """Padded 2-D field (rows x ld), value(y, x) = offset + scale*U01(seed, stream, y*(nx+2)+x).

    `y` is the GLOBAL padded row index (0 = lower Dirichlet row, ny+1 = upper);
    rows [row0, row0+rows) are produced, so a rank slab with ghost rows gets
    exactly the global values. Columns x >= nx+2 (pitch padding) are 0.
    Recipe C1/C2/C4: interior and ring = 0.5 + U01.
    """
    ld = even_ld(nx + 2) if ld is None else ld
    if ld < nx + 2:
        raise ValueError(f"ld={ld} < nx+2={nx + 2}")
    rows = (ny + 2 - row0) if rows is None else rows
    out = np.zeros((rows, ld), dtype=np.float64)
    fill_affine(out, rows, nx + 2, ld, row0 * (nx + 2), nx + 2, seed, stream, scale, offset)
    return out


def pw_field(nx: int, ny: int, nz: int, stream: int, ldx: int | None = None, *,
             seed: int = SEED, plane0: int = 0, planes: int | None = None) -> np.ndarray:
    """Padded 3-D field (planes x (ny+2) x ldx), x fastest, z slowest.

    value(z, y, x) = 2*U01(seed, stream, (z*(ny+2)+y)*(nx+2)+x) - 1 (recipe C3/C5).
    Halo cells are seeded too (they are inputs of the advection).
    """
    ldx = even_ld(nx + 2) if ldx is None else ldx
    if ldx < nx + 2:
        raise ValueError(f"ldx={ldx} < nx+2={nx + 2}")
    planes = (nz + 2 - plane0) if planes is None else planes
    out = np.zeros((planes, ny + 2, ldx), dtype=np.float64)
    fill_affine(out, planes * (ny + 2), nx + 2, ldx, plane0 * (ny + 2) * (nx + 2), nx + 2,
                seed, stream, 2.0, -1.0)
    return out


def jacobi3d_grid(nx: int, ny: int, nz: int, ldx: int | None = None, *, seed: int = SEED,
                  stream: int = STREAM_JACOBI3D, plane0: int = 0, planes: int | None = None) -> np.ndarray:
    """Padded 3-D field (planes x (ny+2) x ldx) for the 7-point Jacobi (NEXT #1):
    value(z, y, x) = 0.5 + U01(seed, 8, (z*(ny+2)+y)*(nx+2)+x), ring included."""
    ldx = even_ld(nx + 2) if ldx is None else ldx
    if ldx < nx + 2:
        raise ValueError(f"ldx={ldx} < nx+2={nx + 2}")
    planes = (nz + 2 - plane0) if planes is None else planes
    out = np.zeros((planes, ny + 2, ldx), dtype=np.float64)
    fill_affine(out, planes * (ny + 2), nx + 2, ldx, plane0 * (ny + 2) * (nx + 2), nx + 2,
                seed, stream, 1.0, 0.5)
    return out


def pw_coefficients(nz: int, *, seed: int = SEED, plane0: int = 0,
                    planes: int | None = None) -> dict:
    """tcx, tcy scalars and per-plane tzc1, tzc2, tzd1, tzd2 (recipe C3: 0.25*(1+0.5*U01))."""
    planes = (nz + 2 - plane0) if planes is None else planes
    co = {"tcx": PW_TCX, "tcy": PW_TCY}
    for name, stream in (("tzc1", STREAM_TZC1), ("tzc2", STREAM_TZC2),
                         ("tzd1", STREAM_TZD1), ("tzd2", STREAM_TZD2)):
        arr = np.empty((1, planes), dtype=np.float64)
        fill_affine(arr, 1, planes, planes, plane0, 0, seed, stream, 0.125, 0.25)
        co[name] = arr[0].copy()
    return co


def pw_inputs(nx: int, ny: int, nz: int, ldx: int | None = None, *, seed: int = SEED,
              plane0: int = 0, planes: int | None = None) -> dict:
    d = {name: pw_field(nx, ny, nz, s, ldx, seed=seed, plane0=plane0, planes=planes)
         for name, s in (("u", STREAM_U), ("v", STREAM_V), ("w", STREAM_W))}
    d.update(pw_coefficients(nz, seed=seed, plane0=plane0, planes=planes))
    return d


def omp_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
