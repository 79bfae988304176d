"""CPU tests of the host-side decomposition logic (st_jacobi2d/3d_schedule,
st_halo_plan, st_block_split): the schedule the CUDA path runs, executed with
NumPy ops for simulated ranks, is bitwise the oracle (SURVEY.md §8(c5) D1/D2,
SPEC.md:465 ranks-sim == serial)."""
import numpy as np
import pytest

import oracle
import paper_2310_01882_b200 as st
import stencil_inputs as si
from slab_sim import run_simulated


@pytest.mark.parametrize("nranks,h,iters,tblock", [
    (1, 1, 7, 1), (1, 1, 9, 4), (1, 1, 10, 2),
    (2, 1, 5, 1), (3, 1, 8, 1), (4, 1, 3, 1),
    (2, 2, 7, 1), (3, 3, 10, 1),            # deep ghosts, single sweeps, shrinking ranges
    (2, 4, 13, 4), (3, 4, 9, 4), (4, 2, 11, 2),  # temporal blocking across ranks
    (2, 6, 17, 6), (2, 8, 20, 8), (5, 4, 6, 2),
])
def test_schedule_simulated_equals_oracle(nranks, h, iters, tblock):
    nx, ny = 37, 61
    a = si.jacobi2d_grid(nx, ny)
    got = run_simulated(a, nx, nranks, h, iters, tblock)
    want = oracle.jacobi2d(a, iters, nx=nx)
    assert np.array_equal(got, want)


def test_auto_tblock_choice():
    ops = st.st_jacobi2d_schedule(0, 1, 16384, 16384, 1, 1000, 0)
    sweeps = {o["sweeps"] for o in ops if o["kind"] == st.OP_SWEEP}
    assert max(sweeps) == 10  # auto depth on large single-domain grids (schedule.cu kAutoTblock)
    assert sum(o["sweeps"] for o in ops if o["kind"] == st.OP_SWEEP) == 1000
    small = st.st_jacobi2d_schedule(0, 1, 100, 100, 1, 10, 0)
    assert {o["sweeps"] for o in small if o["kind"] == st.OP_SWEEP} == {1}
    # across ranks the auto depth is capped by the ghost depth
    multi = st.st_jacobi2d_schedule(1, 4, 4096, 4096, 2, 10, 0)
    assert max(o["sweeps"] for o in multi if o["kind"] == st.OP_SWEEP) == 2


@pytest.mark.parametrize("iters", list(range(0, 23)))
@pytest.mark.parametrize("t", [2, 4, 6, 8])
def test_pass_parity_and_count(iters, t):
    ops = st.st_jacobi2d_schedule(0, 1, 500, 500, 1, iters, t)
    sw = [o for o in ops if o["kind"] == st.OP_SWEEP]
    assert sum(o["sweeps"] for o in sw) == iters
    assert len(sw) % 2 == iters % 2  # result in b iff iters odd
    assert all(o["sweeps"] == 1 or (o["sweeps"] % 2 == 0 and o["sweeps"] <= t) for o in sw)


def test_overlap_structure_h1():
    # boundary rows, async swap, interior rows, join — every sweep but the last
    ops = st.st_jacobi2d_schedule(1, 3, 64, 40, 1, 3, 1)
    kinds = [o["kind"] for o in ops]
    S, E, J, W = st.OP_SWEEP, st.OP_EXCHANGE, st.OP_JOIN, st.OP_SWAP
    assert kinds == [E, S, S, E, S, J, W, S, S, E, S, J, W, S, W]
    assert [o["flag"] for o in ops if o["kind"] == E] == [0, 1, 1]
    b1, b2, _, interior = ops[1], ops[2], ops[3], ops[4]
    assert (b1["y_lo"], b1["y_hi"], b2["y_lo"], b2["y_hi"]) == (1, 1, 40, 40)
    assert (interior["y_lo"], interior["y_hi"]) == (2, 39)


def test_schedule_rejects():
    with pytest.raises(st.StencilError):
        st.st_jacobi2d_schedule(0, 2, 64, 3, 4, 5, 1)  # slab thinner than the ghost depth
    with pytest.raises(st.StencilError):
        st.st_jacobi2d_schedule(0, 2, 64, 64, 2, 5, 4)  # T deeper than the ghosts
    with pytest.raises(st.StencilError):
        st.st_jacobi2d_schedule(0, 1, 64, 64, 1, 5, 3)  # odd T


@pytest.mark.parametrize("nranks,h,iters,tblock", [
    (1, 1, 7, 0), (1, 1, 6, 2), (1, 1, 5, 1),
    (2, 1, 5, 0), (3, 1, 4, 1),               # halo 1: one sweep per pass
    (2, 2, 7, 0), (3, 2, 6, 2), (4, 3, 9, 2),  # T = 2 across ranks (auto with halo >= 2)
    (2, 2, 1, 2), (3, 4, 11, 0), (2, 3, 8, 1),
])
def test_schedule3d_simulated_equals_oracle(nranks, h, iters, tblock):
    nx, ny, nz = 9, 7, 23
    a = si.jacobi3d_grid(nx, ny, nz)
    got = run_simulated(a, nx, nranks, h, iters, tblock)
    assert np.array_equal(got, oracle.jacobi3d(a, iters, nx=nx))


def test_schedule3d_tblock_choice():
    def sweeps(ops):  # sweeps per pass (a pass = the sweep ops before a SWAP)
        out, last = [], None
        for o in ops:
            if o["kind"] == st.OP_SWEEP:
                last = o["sweeps"]
            elif o["kind"] == st.OP_SWAP:
                out.append(last)
        return out
    assert set(sweeps(st.st_jacobi3d_schedule(0, 1, 512, 512, 1, 100, 0))) == {2}
    assert set(sweeps(st.st_jacobi3d_schedule(1, 4, 512, 128, 1, 100, 0))) == {1}   # halo 1 -> one sweep
    multi = st.st_jacobi3d_schedule(1, 4, 512, 128, 2, 100, 0)
    assert set(sweeps(multi)) == {2} and sum(sweeps(multi)) == 100
    for it in range(12):
        sw = sweeps(st.st_jacobi3d_schedule(0, 2, 64, 64, 2, it, 2))
        assert sum(sw) == it and len(sw) % 2 == it % 2
    with pytest.raises(st.StencilError):
        st.st_jacobi3d_schedule(0, 2, 64, 64, 1, 5, 2)  # T = 2 needs two ghost planes
    with pytest.raises(st.StencilError):
        st.st_jacobi3d_schedule(0, 1, 64, 64, 1, 5, 4)  # only 1 and 2 in 3-D
