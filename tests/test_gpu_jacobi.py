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


# Extreme magnitudes through the temporally blocked kernels: tiny values whose
# level sums round in the subnormal range, huge values, a tiny band deep inside a
# chunk, zeros, and sign changes (cancellation to values near zero). Every level
# multiplies by 0.25 exactly as Listing 1 does, so these stay bitwise.
EXTREME_CASES = [
    ("tiny", 2.0**-1060, 9, 8),
    ("tiny_t2", 2.0**-1070, 5, 2),
    ("huge", 2.0**1012, 16, 8),
    ("mid_band", None, 17, 8),
    ("edge_lo", 2.0**-1006, 16, 10),
    ("zeros", 0.0, 24, 8),
    ("signs", -1.0, 24, 10),
]


@pytest.mark.parametrize("name,scale,iters,tblock", EXTREME_CASES)
def test_extreme_magnitudes_bitwise(cuda_lib, name, scale, iters, tblock):
    a = si.jacobi2d_grid(300, 2600)
    if name == "mid_band":
        a[1500:2000] *= 2.0**-1062
    elif name == "zeros":
        a[0, :] = 0.0
        a[:, 0] = 0.0
        a[5:9, 100:200] = 0.0
    elif name == "signs":
        a = a - 1.0
    else:
        a = a * scale
    want = oracle.jacobi2d(a, iters)
    got = run_gpu(cuda_lib, a, iters, tblock)
    assert_bitwise(got, want)


@pytest.mark.parametrize("tblock", [2, 4, 6, 8, 10])
@pytest.mark.parametrize("nx,ny,ld,iters", [(2301, 700, 2304, 21), (3100, 181, 3102, 13), (1150, 400, 1152, 11)])
def test_wide_grids_equal_single_sweeps(cuda_lib, tblock, nx, ny, ld, iters):
    # wide ragged grids: many interior strips on the rotated path, both ring-column strips
    # on the general path, several row chunks
    a = si.jacobi2d_grid(nx, ny, ld=ld)
    want = oracle.jacobi2d(a, iters, nx=nx)
    got = run_gpu(cuda_lib, a, iters, tblock, nx=nx)
    assert_bitwise(got[:, : nx + 2], want[:, : nx + 2])


@pytest.mark.parametrize("tblock,iters", [(1, 7), (0, 23), (4, 10)])
def test_cuda_graph_capture_bitwise(cuda_lib, tblock, iters):
    # st_jacobi2d_run does no host synchronisation or allocation, so a whole multi-launch
    # call can be captured in a CUDA graph once and replayed (the C1 bench leg times this)
    import torch
    st = cuda_lib
    grid = si.jacobi2d_grid(1000, 500)
    a0 = torch.from_numpy(grid).cuda()
    a = a0.clone()
    b = torch.empty_like(a)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        st.st_jacobi2d_run(a, b, iters, tblock=tblock)  # warm the launch path outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        r = st.st_jacobi2d_run(a, b, iters, tblock=tblock)
    a.copy_(a0)
    b.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert_bitwise(r.cpu().numpy(), oracle.jacobi2d(grid, iters))
