"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (tblock=0 = auto temporal blocking; one PW launch over the whole grid),
on samples the oracle can compute independently:

* C4 (configs[3], 32768^2, the N>1 strong-scaling grid) on one GPU: 20 sweeps;
  row bands (top ring, middle, bottom ring) are recomputed by the oracle on
  windows widened by the 20-row influence radius — bitwise.
* C5 (configs[4], 1024x1024x512 PW) on one GPU: sampled planes recomputed by the
  oracle from their 3-plane input windows — bitwise.
* C2 (configs[1], 16384^2) for the FULL 1000 sweeps of one bench step: the
  discrete sine eigenmode (pin J6) must decay as lambda^1000 within the
  accumulated rounding bound; an integer linear field must stay an exact fixed
  point (pin J3).
* The in-place Gauss-Seidel grid of the bench (16384^2, one launch): every point
  vs the sequential oracle after 2 sweeps; a linear field stays fixed for 100.

Inputs are generated band by band straight into device memory (the generator
indexes the global grid, so a band has exactly the full grid's values)."""
import math

import numpy as np
import pytest

import oracle
import stencil_inputs as si

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _fill_jacobi_device(n, ld, band=2048):
    import torch
    a = torch.empty((n + 2, ld), dtype=torch.float64, device="cuda")
    for r0 in range(0, n + 2, band):
        rows = min(band, n + 2 - r0)
        a[r0:r0 + rows] = torch.from_numpy(si.jacobi2d_grid(n, n, ld=ld, row0=r0, rows=rows))
    return a


def test_C4_32768_sampled_bands_20_sweeps(cuda_lib):
    import torch
    n, iters = 32768, 20
    ld = n + 2
    a = _fill_jacobi_device(n, ld)
    b = torch.empty_like(a)
    r = cuda_lib.st_jacobi2d_run(a, b, iters, tblock=0)
    torch.cuda.synchronize()
    for y0, y1 in ((0, 47), (16000, 16047), (n + 2 - 48, n + 1)):  # global padded rows, inclusive
        w0, w1 = max(0, y0 - iters), min(n + 1, y1 + iters)
        win = si.jacobi2d_grid(n, n, ld=ld, row0=w0, rows=w1 - w0 + 1)
        # the window's first/last rows act as a Dirichlet ring for the oracle; they are
        # >= iters rows from the compared band unless they are the true ring
        want = oracle.jacobi2d(win, iters, nx=n)[y0 - w0: y1 - w0 + 1]
        got = r[y0:y1 + 1].cpu().numpy()
        bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
        assert bad.size == 0, f"rows {y0}..{y1}: {len(bad)} mismatches, first {bad[:3].tolist()}"
    del a, b, r
    torch.cuda.empty_cache()


def test_C5_pw_1024x1024x512_sampled_planes(cuda_lib):
    import torch
    nx = ny = 1024
    nz = 512
    ldx = nx + 2
    fields = {}
    for name, stream in (("u", si.STREAM_U), ("v", si.STREAM_V), ("w", si.STREAM_W)):
        t = torch.empty((nz + 2, ny + 2, ldx), dtype=torch.float64, device="cuda")
        for p0 in range(0, nz + 2, 64):
            k = min(64, nz + 2 - p0)
            t[p0:p0 + k] = torch.from_numpy(si.pw_field(nx, ny, nz, stream, ldx, plane0=p0, planes=k))
        fields[name] = t
    co = si.pw_coefficients(nz)
    cod = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in co.items()}
    outs = [torch.empty_like(fields["u"]) for _ in range(3)]
    cuda_lib.st_pw_advect3d(fields["u"], fields["v"], fields["w"], *outs, cod["tcx"], cod["tcy"], cod["tzc1"],
                            cod["tzc2"], cod["tzd1"], cod["tzd2"])
    torch.cuda.synchronize()
    for z in (1, 2, 257, 511, 512):
        win = si.pw_inputs(nx, ny, nz, ldx, plane0=z - 1, planes=3)
        want = oracle.pw_advect3d(win["u"], win["v"], win["w"], win, nx=nx)
        for name, g, wnt in zip(("su", "sv", "sw"), outs, want):
            got = g[z, 1:ny + 1, 1:nx + 1].cpu().numpy()
            w = wnt[1, 1:ny + 1, 1:nx + 1]
            bad = np.argwhere(got.view(np.uint64) != w.view(np.uint64))
            assert bad.size == 0, f"{name} plane {z}: {len(bad)} mismatches, first {bad[:3].tolist()}"
    del fields, outs
    torch.cuda.empty_cache()


def test_C2_1000_sweeps_eigenmode_and_fixed_point(cuda_lib):
    import torch
    n, iters = 16384, 1000
    ld = n + 2
    # J6: u0 = sin(pi x/(n+1)) sin(pi y/(n+1)), zero ring -> u_k = lambda^k u0 exactly in real
    # arithmetic, lambda = cos(pi/(n+1)); each sweep adds <= ~3 ulp of the current magnitude
    s = np.sin(np.pi * np.arange(n + 2) / (n + 1))
    s[0] = s[-1] = 0.0
    u0 = torch.from_numpy(np.outer(s, s)).cuda()
    b = torch.empty_like(u0)
    r = cuda_lib.st_jacobi2d_run(u0.clone(), b, iters, tblock=0)
    lam = math.cos(math.pi / (n + 1))
    want = (lam ** iters) * u0
    err = (r - want).abs().max().item()
    assert err <= iters * 4 * 2.0 ** -53, f"eigenmode drift {err}"
    assert torch.equal(r[0], u0[0]) and torch.equal(r[:, -1], u0[:, -1])  # ring untouched
    del u0, b, r, want
    # J3: an integer-valued linear field (incl. ring) is an exact fixed point
    y = torch.arange(n + 2, dtype=torch.float64, device="cuda")[:, None]
    x = torch.arange(ld, dtype=torch.float64, device="cuda")[None, :]
    a = (3 * x - 2 * y + 7).contiguous()
    out = cuda_lib.st_jacobi2d_run(a.clone(), torch.empty_like(a), iters, tblock=0)
    assert torch.equal(out, a)
    torch.cuda.empty_cache()


def test_gauss_seidel_16384_full_grid_2_sweeps_and_fixed_point(cuda_lib):
    # the bench's GS grid (16384^2, tiled wavefront kernel, one launch): every point vs the
    # sequential oracle after 2 sweeps, and an integer linear field stays fixed for 100 sweeps
    import torch
    n = 16384
    a_np = si.jacobi2d_grid(n, n)
    want = oracle.gauss_seidel2d(a_np, 2)
    a = torch.from_numpy(a_np).cuda()
    cuda_lib.st_gauss_seidel2d_run(a, 2)
    got = a.cpu().numpy()
    bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:3].tolist()}"
    del a, a_np, want, got
    y = torch.arange(n + 2, dtype=torch.float64, device="cuda")[:, None]
    x = torch.arange(n + 2, dtype=torch.float64, device="cuda")[None, :]
    lin = (5 * x - 3 * y + 2).contiguous()
    g = lin.clone()
    cuda_lib.st_gauss_seidel2d_run(g, 100)
    assert torch.equal(g, lin)
    torch.cuda.empty_cache()


@pytest.mark.parametrize("tblock", [0, 1])
def test_C2_recipe_1024_full_1000_sweeps_every_point(cuda_lib, tblock):
    # "full 1000 sweeps on a 1024^2 grid" — every point bitwise
    # against the C oracle, at auto temporal blocking (T = 10: 100 passes) and at T = 1
    import torch
    n, iters = 1024, 1000
    grid = si.jacobi2d_grid(n, n)
    want = oracle.jacobi2d(grid, iters)
    a = torch.from_numpy(grid).cuda()
    b = torch.empty_like(a)
    r = cuda_lib.st_jacobi2d_run(a, b, iters, tblock=tblock)
    torch.cuda.synchronize()
    got = r.cpu().numpy()
    bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:5].tolist()}"


def test_jacobi3d_128_cubed_100_sweeps_every_point(cuda_lib):
    # the 3-D counterpart: 50 two-sweep passes (jacobi3d_t2_kernel) end to end, every point
    import torch
    n, iters = 128, 100
    grid = si.jacobi3d_grid(n, n, n)
    want = oracle.jacobi3d(grid, iters)
    a = torch.from_numpy(grid).cuda()
    b = torch.empty_like(a)
    r = cuda_lib.st_jacobi3d_run(a, b, iters)
    torch.cuda.synchronize()
    got = r.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
