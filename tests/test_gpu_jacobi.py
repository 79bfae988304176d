"""GPU parity of st_jacobi2d_run against the CPU oracle (bitwise).

The CUDA path evaluates ((N+S)+W)+E then *0.25 with one rounding per op and
no contraction, exactly like the oracle, so the bar is bit-exact equality
(stricter than north_star's 1e-12 relative tolerance)."""
import numpy as np
import pytest

import oracle
import stencil_inputs as si

pytestmark = pytest.mark.gpu


def run_gpu(st, a_np, iters, tblock=0, nx=None, which=False):
    import torch
    a = torch.from_numpy(a_np).cuda()
    b = torch.empty_like(a)
    b.fill_(float("nan"))  # the library must copy the ring itself
    r = st.st_jacobi2d_run(a, b, iters, tblock=tblock, nx=nx)
    torch.cuda.synchronize()
    assert (r is b) == bool(iters & 1)  # result in b iff iters odd
    return (r.cpu().numpy(), r is b) if which else r.cpu().numpy()


def assert_bitwise(got, want):
    assert got.shape == want.shape
    bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:5].tolist()}: {got[tuple(bad[0])]} vs {want[tuple(bad[0])]}"


@pytest.mark.parametrize("tblock", [0, 1])
def test_C1_64x64_100_sweeps(cuda_lib, tblock):
    # configs[0]: 64x64 interior + 1-cell Dirichlet ring, 100 iterations
    a = si.jacobi2d_grid(64, 64)
    assert_bitwise(run_gpu(cuda_lib, a, 100, tblock), oracle.jacobi2d(a, 100))


SHAPES = [  # (nx, ny, ld, iters): odd/even nx, nx not a multiple of the 64-col strip, 1-wide, 1-tall, padded pitch
    (1, 1, 4, 3), (1, 37, 4, 5), (37, 1, 40, 4), (2, 2, 4, 7), (62, 9, 64, 2), (63, 9, 66, 3),
    (64, 17, 66, 1), (65, 130, 68, 6), (127, 129, 130, 9), (190, 33, 200, 10), (1000, 300, 1002, 11),
    (4093, 257, 4096, 4),
]


@pytest.mark.parametrize("nx,ny,ld,iters", SHAPES)
@pytest.mark.parametrize("tblock", [0, 1, 2, 4, 6, 8, 10])
def test_ragged_shapes(cuda_lib, nx, ny, ld, iters, tblock):
    a = si.jacobi2d_grid(nx, ny, ld=ld)
    want = oracle.jacobi2d(a, iters, nx=nx)
    got, in_b = run_gpu(cuda_lib, a, iters, tblock, nx=nx, which=True)
    assert_bitwise(got[:, : nx + 2], want[:, : nx + 2])
    # pitch padding of the result buffer is never written (b starts NaN-filled)
    pad = got[:, nx + 2:]
    assert np.all(np.isnan(pad)) if in_b else np.array_equal(pad, a[:, nx + 2:])


@pytest.mark.parametrize("tblock", [2, 4, 6, 8, 10])
@pytest.mark.parametrize("iters", [1, 2, 3, 5, 8, 13, 17, 33])
def test_temporal_blocking_equals_single_sweeps(cuda_lib, tblock, iters):
    # T sweeps per HBM pass is bitwise T single sweeps, for every remainder/parity
    nx, ny = 250, 1100  # several strips and several 512-row chunks
    a = si.jacobi2d_grid(nx, ny, ld=256)
    want = oracle.jacobi2d(a, iters, nx=nx)
    got = run_gpu(cuda_lib, a, iters, tblock, nx=nx)
    assert_bitwise(got[:, : nx + 2], want[:, : nx + 2])


def test_tblock_rejects_unsupported(cuda_lib):
    import torch
    a = torch.zeros(20, 20, dtype=torch.float64, device="cuda")
    with pytest.raises(cuda_lib.StencilError) as e:
        cuda_lib.st_jacobi2d_run(a, a.clone(), 5, tblock=3)
    assert e.value.code == cuda_lib.ST_ENOTSUP


def test_iters_zero_is_identity(cuda_lib):
    a = si.jacobi2d_grid(70, 20)
    assert_bitwise(run_gpu(cuda_lib, a, 0, 1), a)


def test_chunked_calls_equal_one_call(cuda_lib):
    import torch
    a_np = si.jacobi2d_grid(300, 200, ld=304)
    a = torch.from_numpy(a_np).cuda()
    b = torch.empty_like(a)
    r1 = cuda_lib.st_jacobi2d_run(a, b, 40, tblock=1, nx=300)
    o1 = b if r1 is a else a
    r2 = cuda_lib.st_jacobi2d_run(r1, o1, 60, tblock=1, nx=300)
    assert_bitwise(r2.cpu().numpy()[:, :302], oracle.jacobi2d(a_np, 100, nx=300)[:, :302])


def test_linear_field_fixed_point_1000_sweeps(cuda_lib):
    # J3 at a size that spans many strips and row chunks: exact fixed point
    nx, ny = 2050, 1030
    y, x = np.mgrid[0: ny + 2, 0: nx + 2]
    a = (3 * x + 2 * y + 7).astype(np.float64)
    a = np.ascontiguousarray(np.pad(a, ((0, 0), (0, 2))))
    got = run_gpu(cuda_lib, a, 1000, 1, nx=nx)
    assert_bitwise(got, a)


@pytest.fixture(scope="module")
def c2_case():
    a = si.jacobi2d_grid(16384, 16384)
    return a, oracle.jacobi2d(a, 10)


@pytest.mark.slow
@pytest.mark.parametrize("tblock", [1, 0, 4, 8, 10])
def test_C2_full_size_10_sweeps(cuda_lib, c2_case, tblock):
    # configs[1] grid (16384^2 interior), 10 sweeps, every element vs the oracle,
    # in the launch configurations bench.py times (tblock=0 = auto)
    a, want = c2_case
    assert_bitwise(run_gpu(cuda_lib, a, 10, tblock), want)


def test_stream_and_sync_semantics(cuda_lib):
    # work is ordered on the caller's (non-default) stream
    import torch
    a_np = si.jacobi2d_grid(500, 400)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = torch.from_numpy(a_np).cuda()
        b = torch.empty_like(a)
        r = cuda_lib.st_jacobi2d_run(a, b, 13, tblock=1)
        out = r.cpu()
    assert_bitwise(out.numpy(), oracle.jacobi2d(a_np, 13))


def test_rejects_host_tensor_and_wrong_dtype(cuda_lib):
    import torch
    a = torch.zeros(10, 10, dtype=torch.float64)
    with pytest.raises(TypeError):
        cuda_lib.st_jacobi2d_run(a, a.clone(), 1)
    g = torch.zeros(10, 10, dtype=torch.float32, device="cuda")
    with pytest.raises(TypeError):
        cuda_lib.st_jacobi2d_run(g, g.clone(), 1)


def test_launches_counted(cuda_lib):
    import torch
    a = torch.from_numpy(si.jacobi2d_grid(200, 100)).cuda()
    b = torch.empty_like(a)
    n0 = cuda_lib.launch_count()
    cuda_lib.st_jacobi2d_run(a, b, 7, tblock=1)
    torch.cuda.synchronize()
    assert cuda_lib.launch_count() - n0 == 7


def _subprocess_bitwise(cases_code, env_extra):
    """Runs cases in a fresh process with environment knobs (read once per process by the library)."""
    import os
    import pathlib
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle, stencil_inputs as si, paper_2310_01882_b200 as st
def run(a, it, tb, nx=None):
    nx = a.shape[1] - 2 if nx is None else nx
    ta = torch.from_numpy(a).cuda(); tb_ = torch.empty_like(ta)
    return st.st_jacobi2d_run(ta, tb_, it, tblock=tb, nx=nx).cpu().numpy()
res = []
""" % str(pathlib.Path(__file__).resolve().parent.parent) + cases_code + "\nprint('RESULT', res)\n"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")]
    assert line, r.stdout + r.stderr[-3000:]
    return eval(line[0][len("RESULT"):])


# Grids outside the folding's exactness range (every input zero or
# with a biased exponent in [1+2T, 2045-2T]): tiny values whose level sums round
# in the subnormal range, huge values, a single tiny row deep inside a chunk (the
# warp restarts after it already stored rows), and the range edges for T = 8.
FOLD_CASES = r"""
rng = np.random.default_rng(7)
base = si.jacobi2d_grid(300, 2600)
cases = []
cases.append(("tiny", base * 2.0**-1060, 9, 8))                 # subnormal sums: folding must not be used
cases.append(("tiny_t2", base * 2.0**-1070, 5, 2))
cases.append(("huge", base * 2.0**1012, 16, 8))                 # 4^8 x 2^1012 overflows
mid = base.copy(); mid[1500:2000] *= 2.0**-1062; cases.append(("mid_band", mid, 17, 8))  # tiny band deep in the grid
edge = base * 2.0**-1006; cases.append(("edge_lo_safe", edge, 16, 8))   # exponent -1006 (biased 17): folded
edge2 = base * 2.0**-1007; cases.append(("edge_lo_unsafe", edge2, 16, 8))
zero = base.copy(); zero[0, :] = 0.0; zero[:, 0] = 0.0; zero[5:9, 100:200] = 0.0; cases.append(("zeros", zero, 24, 8))
neg = base - 1.0; cases.append(("signs", neg, 24, 8))           # cancellation -> values near zero, sign changes
for name, a, it, tb in cases:
    want = oracle.jacobi2d(a, it)
    got = run(a, it, tb)
    res.append((name, bool(np.array_equal(got.view(np.uint64), want.view(np.uint64)))))
"""


def test_fold_out_of_range_grids_bitwise(cuda_lib):
    # ST_JACOBI_FOLD=1: folded levels with the per-row range check
    res = _subprocess_bitwise(FOLD_CASES, {"ST_JACOBI_FOLD": "1"})
    assert all(ok for _, ok in res), res


def test_fold_exact_path_bitwise(cuda_lib):
    # ST_JACOBI_FOLD=0 (the default): every level multiplies
    res = _subprocess_bitwise(FOLD_CASES, {"ST_JACOBI_FOLD": "0"})
    assert all(ok for _, ok in res), res


def test_fold_check_is_necessary(cuda_lib):
    # ST_JACOBI_FOLD=2 folds without the range check (test-only knob): the tiny and
    # huge grids then differ from the oracle, so the range check is what keeps them exact
    res = dict(_subprocess_bitwise(FOLD_CASES, {"ST_JACOBI_FOLD": "2"}))
    assert not res["tiny"] and not res["huge"] and not res["mid_band"], res
    assert res["edge_lo_safe"] and res["zeros"], res


@pytest.mark.parametrize("tblock", [2, 4, 6, 8, 10])
@pytest.mark.parametrize("nx,ny,ld,iters", [(2301, 700, 2304, 21), (3100, 181, 3102, 13), (1150, 400, 1152, 11)])
def test_wide_grids_equal_single_sweeps(cuda_lib, tblock, nx, ny, ld, iters):
    # wide ragged grids: many interior strips on the rotated path, both ring-column strips
    # on the general path, several row chunks
    a = si.jacobi2d_grid(nx, ny, ld=ld)
    want = oracle.jacobi2d(a, iters, nx=nx)
    got = run_gpu(cuda_lib, a, iters, tblock, nx=nx)
    assert_bitwise(got[:, : nx + 2], want[:, : nx + 2])
