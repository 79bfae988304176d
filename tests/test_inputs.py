"""Generator pins (G1) and recipe properties of stencil_inputs (CPU)."""
import json
import pathlib

import numpy as np

import stencil_inputs as si

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "g1_splitmix.json").read_text())


def test_g1_raw_first_output():
    assert si.raw(42, 0, 0) == int(GOLD["raw_42_0_0"], 16)


def test_g1_values():
    assert [si.u01(42, 0, i) for i in range(4)] == GOLD["u01_42_0"]
    assert [si.u01(42, 1, i) for i in range(4)] == GOLD["u01_42_1"]
    assert si.u01(42, 0, 10 ** 9) == GOLD["u01_42_0_1e9"]


def test_numpy_transcription_matches_c():
    idx = np.arange(0, 5000, 7, dtype=np.uint64)
    c = np.array([si.u01(42, 3, int(i)) for i in idx])
    assert np.array_equal(c, si.u01_numpy(42, 3, idx))


def test_slab_equals_global_window():
    # counter based: a rank slab (rows [r0, r0+k)) is bitwise the global window
    nx, ny = 37, 29
    g = si.jacobi2d_grid(nx, ny)
    s = si.jacobi2d_grid(nx, ny, row0=11, rows=7)
    assert np.array_equal(g[11:18], s)
    u = si.pw_field(9, 7, 8, si.STREAM_U)
    us = si.pw_field(9, 7, 8, si.STREAM_U, plane0=3, planes=4)
    assert np.array_equal(u[3:7], us)


def test_pitch_padding_zero_and_independent_of_ld():
    a = si.jacobi2d_grid(5, 4, ld=7)
    b = si.jacobi2d_grid(5, 4, ld=16)
    assert np.array_equal(a[:, :7], b[:, :7])
    assert np.all(b[:, 7:] == 0)


def test_recipe_ranges():
    a = si.jacobi2d_grid(64, 64)
    assert a.min() >= 0.5 and a.max() < 1.5
    d = si.pw_inputs(8, 8, 8)
    for k in "uvw":
        assert d[k].min() >= -1.0 and d[k].max() < 1.0
    for k in ("tzc1", "tzc2", "tzd1", "tzd2"):
        assert d[k].shape == (10,) and d[k].min() >= 0.25 and d[k].max() < 0.375
