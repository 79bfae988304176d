"""GPU parity of the generic linear stencil.apply executor (reading R23;
st_stencil2d_run) against the CPU oracle — bitwise: both evaluate the terms
left to right with one rounding per product and per sum."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
rng = np.random.default_rng(185)

STENCILS = {
    "listing1_generic": ([(-1, 0), (1, 0), (0, -1), (0, 1)], [0.25, 0.25, 0.25, 0.25]),
    "nine_point_R2": ([(0, 0), (-2, 0), (2, 0), (0, -2), (0, 2), (-1, -1), (1, 1), (-1, 1), (1, -1)],
                      [0.2, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1]),
    "asymmetric_R3": ([(3, -2), (-1, 3), (0, 0), (0, -1)], [0.7, -0.3, 0.45, 0.15]),
    "identity": ([(0, 0)], [1.0]),
    "shift": ([(0, 1)], [1.0]),
    "max_offset_8": ([(8, 0), (-8, 0), (0, 8), (0, -8), (0, 0)], [0.1, 0.2, 0.3, 0.15, 0.25]),
}


def run(st, a_np, offs, coefs, iters, nx=None):
    import torch
    a = torch.from_numpy(a_np).cuda()
    b = torch.full_like(a, float("nan"))
    r = st.st_stencil2d_run(a, b, offs, coefs, iters, nx=nx)
    torch.cuda.synchronize()
    assert (r is b) == bool(iters & 1)
    return r.cpu().numpy()


@pytest.mark.parametrize("name", list(STENCILS))
@pytest.mark.parametrize("ny,nx,pad,iters", [(1, 1, 0, 3), (7, 33, 3, 2), (40, 65, 0, 5), (97, 130, 2, 4),
                                             (257, 300, 4, 3)])
def test_stencil_bitwise(cuda_lib, name, ny, nx, pad, iters):
    offs, coefs = STENCILS[name]
    R = oracle.stencil_halo(offs)
    a = rng.standard_normal((ny + 2 * R, nx + 2 * R + pad))
    want = oracle.stencil2d(a, offs, coefs, iters, nx=nx)
    got = run(cuda_lib, a, offs, coefs, iters, nx=nx)
    assert np.array_equal(got[:, :nx + 2 * R], want[:, :nx + 2 * R])


@pytest.mark.parametrize("name", list(STENCILS))
@pytest.mark.parametrize("ny,nx,iters", [(1, 1, 3), (3, 2, 2), (40, 65, 5), (97, 130, 4), (57, 301, 3)])
def test_stencil_even_pitch_bitwise(cuda_lib, name, ny, nx, iters):
    # 16-byte rows: the column-pair kernel (even and odd dx terms, pairs straddling the ring)
    offs, coefs = STENCILS[name]
    R = oracle.stencil_halo(offs)
    ld = nx + 2 * R + ((nx + 2 * R) & 1)  # even, no spare column when nx + 2R is even
    a = rng.standard_normal((ny + 2 * R, ld))
    want = oracle.stencil2d(a, offs, coefs, iters, nx=nx)
    got = run(cuda_lib, a, offs, coefs, iters, nx=nx)
    assert np.array_equal(got[:, :nx + 2 * R], want[:, :nx + 2 * R])


def test_random_stencils_bitwise(cuda_lib):
    for _ in range(10):
        n = int(rng.integers(1, 33))
        R = int(rng.integers(1, 5))
        offs = [(int(rng.integers(-R, R + 1)), int(rng.integers(-R, R + 1))) for _ in range(n)]
        coefs = list(rng.standard_normal(n))
        Rr = oracle.stencil_halo(offs)
        ny, nx = int(rng.integers(1, 120)), int(rng.integers(1, 150))
        a = rng.standard_normal((ny + 2 * Rr, nx + 2 * Rr))
        assert np.array_equal(run(cuda_lib, a, offs, coefs, 3), oracle.stencil2d(a, offs, coefs, 3))


def test_rejects_bad_arguments(cuda_lib):
    import torch
    a = torch.zeros(10, 10, dtype=torch.float64, device="cuda")
    b = torch.zeros_like(a)
    with pytest.raises(cuda_lib.StencilError):
        cuda_lib.st_stencil2d_run(a, b, [(0, 9)], [1.0], 1)  # |offset| > 8
    with pytest.raises(cuda_lib.StencilError):
        cuda_lib.st_stencil2d_run(a, b, [(0, 5)], [1.0], 1)  # halo 5 leaves no interior
    with pytest.raises(cuda_lib.StencilError):
        cuda_lib.st_stencil2d_run(a, a, [(0, 1)], [1.0], 1)  # a and b overlap


# ---------------------------------------------------------------- expression stencils (R24, NVRTC)
EXPRS = [
    "(a(-1,0) + a(1,0) + a(0,-1) + a(0,1)) * 0.25",
    "a(0,1)*a(0,-1) - a(1,0)",
    "-(a(3,0) - 2*a(0,0)) / 3 + 0.1*a(-2,2)",
    "(a(0,0) + a(2,0))*(a(0,0) - a(-2,0)) / (1 + a(0,2)*a(0,2))",
    ".5*a(0, 0) + 1e-3 - 0.125*a( -8 , 8 )",
]


@pytest.mark.parametrize("e", EXPRS)
@pytest.mark.parametrize("ny,nx,iters", [(1, 1, 2), (37, 45, 3), (130, 257, 2)])
def test_expression_stencil_bitwise(cuda_lib, e, ny, nx, iters):
    import torch
    from oracle import expr as ox
    R = ox.halo(e)
    a_np = rng.uniform(0.5, 1.5, size=(ny + 2 * R, nx + 2 * R))
    a = torch.from_numpy(a_np).cuda()
    b = torch.full_like(a, float("nan"))
    r = cuda_lib.st_stencil2d_expr_run(a, b, e, iters)
    torch.cuda.synchronize()
    assert np.array_equal(r.cpu().numpy(), ox.stencil2d_expr(a_np, e, iters))


@pytest.mark.parametrize("e", EXPRS)
@pytest.mark.parametrize("ny,nx,iters", [(1, 1, 2), (3, 2, 3), (37, 45, 3), (130, 257, 2), (70, 300, 3)])
def test_expression_stencil_even_pitch_bitwise(cuda_lib, e, ny, nx, iters):
    # 16-byte rows (even pitch, aligned base): the column-pair y-streaming kernel for bodies
    # without a division; odd and even halos and widths exercise its edge clamps and the
    # single-column stores of the pairs that straddle the Dirichlet ring
    import torch
    from oracle import expr as ox
    R = ox.halo(e)
    ld = nx + 2 * R + ((nx + 2 * R) & 1) + 2  # even, with pitch padding
    full = rng.uniform(0.5, 1.5, size=(ny + 2 * R, ld))
    a = torch.from_numpy(full).cuda()
    b = torch.full_like(a, float("nan"))
    r = cuda_lib.st_stencil2d_expr_run(a, b, e, iters, nx=nx)
    torch.cuda.synchronize()
    want = ox.stencil2d_expr(np.ascontiguousarray(full[:, : nx + 2 * R]), e, iters)
    assert np.array_equal(r.cpu().numpy()[:, : nx + 2 * R], want)


def test_listing1_expression_equals_jacobi_kernels(cuda_lib):
    # the NVRTC-compiled Listing 1 and the hand-written Jacobi kernels agree bitwise
    import torch
    import stencil_inputs as si
    a_np = si.jacobi2d_grid(300, 200)
    a = torch.from_numpy(a_np).cuda()
    a2 = a.clone()  # both runs ping-pong through their own buffers
    r1 = cuda_lib.st_stencil2d_expr_run(a, torch.empty_like(a), "(a(-1,0)+a(1,0)+a(0,-1)+a(0,1))*0.25", 9)
    r2 = cuda_lib.st_jacobi2d_run(a2, torch.empty_like(a2), 9)
    assert torch.equal(r1, r2)


EXPRS3 = [
    "(a(-1,0,0) + a(1,0,0) + a(0,-1,0) + a(0,1,0) + a(0,0,-1) + a(0,0,1)) / 6",
    "a(1,0,-1)*a(0,2,0) - 3*a(-1,-1,1) + 0.5",
    "(a(0,0,0) - a(2,-1,1)) / (2 + a(-2,0,0)*a(0,0,2))",
]


@pytest.mark.parametrize("e", EXPRS3)
@pytest.mark.parametrize("nz,ny,nx,iters", [(1, 1, 1, 2), (9, 13, 37, 3), (21, 30, 70, 2)])
def test_expression_stencil_3d_bitwise(cuda_lib, e, nz, ny, nx, iters):
    import torch
    from oracle import expr as ox
    R = ox.halo3(e)
    a_np = rng.uniform(0.5, 1.5, size=(nz + 2 * R, ny + 2 * R, nx + 2 * R))
    a = torch.from_numpy(a_np).cuda()
    r = cuda_lib.st_stencil3d_expr_run(a, torch.full_like(a, float("nan")), e, iters)
    torch.cuda.synchronize()
    assert np.array_equal(r.cpu().numpy(), ox.stencil3d_expr(a_np, e, iters))


@pytest.mark.parametrize("e", ["a(1,0,-1)*a(0,2,0) - 3*a(-1,-1,1) + 0.5",
                               "(a(-1,0,0) + a(1,0,0) + a(0,-1,0) + a(0,1,0)) * 0.25 - a(0,0,-3)*a(0,0,2)"])
@pytest.mark.parametrize("nz,ny,nx,iters", [(3, 4, 1, 2), (5, 6, 9, 2), (17, 9, 70, 3)])
def test_expression_stencil_3d_even_pitch_bitwise(cuda_lib, e, nz, ny, nx, iters):
    # 16-byte rows and a division-free body: the column-pair register-queue kernel
    # (odd and even halos and widths: pairs straddling the ring, clamped pair loads)
    import torch
    from oracle import expr as ox
    R = ox.halo3(e)
    ldx = nx + 2 * R + ((nx + 2 * R) & 1)
    full = rng.uniform(0.5, 1.5, size=(nz + 2 * R, ny + 2 * R, ldx))
    a = torch.from_numpy(full).cuda()
    r = cuda_lib.st_stencil3d_expr_run(a, torch.full_like(a, float("nan")), e, iters, nx=nx)
    torch.cuda.synchronize()
    want = ox.stencil3d_expr(np.ascontiguousarray(full[:, :, : nx + 2 * R]), e, iters)
    assert np.array_equal(r.cpu().numpy()[:, :, : nx + 2 * R], want)


def test_benchmark1_expression_equals_jacobi3d_kernel(cuda_lib):
    # NVRTC-compiled benchmark 1 and the hand-written TMA jacobi3d kernel agree bitwise
    import torch
    import stencil_inputs as si
    g = si.jacobi3d_grid(70, 40, 33)
    a = torch.from_numpy(g).cuda()
    a2 = a.clone()
    e = "(a(-1,0,0)+a(1,0,0)+a(0,-1,0)+a(0,1,0)+a(0,0,-1)+a(0,0,1))/6"
    r1 = cuda_lib.st_stencil3d_expr_run(a, torch.empty_like(a), e, 5, nx=70)
    r2 = cuda_lib.st_jacobi3d_run(a2, torch.empty_like(a2), 5, nx=70)
    assert torch.equal(r1[:, :, :72], r2[:, :, :72])


# ---------------------------------------------------------------- fused regions
@pytest.mark.parametrize("nx,ny,nz", [(1, 1, 1), (23, 17, 11), (130, 33, 20)])
def test_fused_pw_region_equals_pw_kernel_and_oracle(cuda_lib, nx, ny, nz):
    # benchmark 2 written as one fused region of three NVRTC-compiled expressions is bitwise
    # the hand-written TMA PW kernel and the C oracle
    import torch
    import stencil_inputs as si
    d = si.pw_inputs(nx, ny, nz)
    g = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
    exprs = cuda_lib.pw_fused_expressions(d["tcx"], d["tcy"])
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    cuda_lib.st_stencil3d_fused_run([g["u"], g["v"], g["w"]], outs, exprs, [g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"]],
                                    nx=nx)
    ref = [torch.zeros_like(g["u"]) for _ in range(3)]
    cuda_lib.st_pw_advect3d(g["u"], g["v"], g["w"], *ref, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"],
                            g["tzd2"], nx=nx)
    torch.cuda.synchronize()
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx)
    for o, r, w in zip(outs, ref, want):
        o, r = o.cpu().numpy()[:, :, :nx + 2], r.cpu().numpy()[:, :, :nx + 2]
        assert np.array_equal(o[1:-1, 1:-1, 1:-1], w[1:-1, 1:-1, 1:nx + 1])
        assert np.array_equal(o, r)


def test_fused_random_region_bitwise(cuda_lib):
    import torch
    from oracle import expr as ox
    exprs = ["f0(1,0,-1)*k0 - f1(0,-2,1)/(1 + f0(0,0,0)*f0(0,0,0))", "2*f1(0,0,0) + f0(-1,1,-1)*k1 - 0.5*f2(0,0,2)"]
    R = ox.fused_halo(exprs)
    nz, ny, nx = 12, 19, 45
    ins = [rng.uniform(0.5, 1.5, size=(nz + 2 * R, ny + 2 * R, nx + 2 * R)) for _ in range(3)]
    ks = [rng.uniform(0.5, 1.5, size=nz + 2 * R) for _ in range(2)]
    want = ox.fused3d_expr(ins, exprs, ks)
    gi = [torch.from_numpy(a).cuda() for a in ins]
    go = [torch.zeros_like(gi[0]) for _ in exprs]
    cuda_lib.st_stencil3d_fused_run(gi, go, exprs, [torch.from_numpy(k).cuda() for k in ks])
    torch.cuda.synchronize()
    for o, w in zip(go, want):
        assert np.array_equal(o.cpu().numpy(), w)
