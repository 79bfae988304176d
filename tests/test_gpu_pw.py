"""GPU parity of st_pw_advect3d against the CPU oracle (bitwise)."""
import numpy as np
import pytest

import oracle
import stencil_inputs as si

pytestmark = pytest.mark.gpu


def to_dev(d):
    import torch
    return {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if isinstance(v, np.ndarray) else v)
            for k, v in d.items()}


def run_gpu(st, d, nx=None, fill=float("nan")):
    import torch
    g = to_dev(d)
    outs = [torch.full_like(g["u"], fill) for _ in range(3)]
    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"],
                      g["tzd2"], nx=nx)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


def assert_interior_bitwise(got, want, nx):
    gi = got[1:-1, 1:-1, 1:nx + 1]
    wi = want[1:-1, 1:-1, 1:nx + 1]
    bad = np.argwhere(gi.view(np.uint64) != wi.view(np.uint64))
    assert bad.size == 0, f"{len(bad)} mismatches, first (interior idx) {bad[:5].tolist()}"


SHAPES = [  # (nx, ny, nz, ldx): tiles of 64 x 8, ragged tails in every dim
    (1, 1, 1, 4), (2, 3, 2, 4), (5, 7, 3, 8), (62, 8, 4, 64), (63, 9, 5, 66), (64, 16, 70, 66),
    (65, 17, 9, 68), (130, 23, 11, 132), (200, 40, 130, 204), (257, 33, 67, 260),
]


@pytest.mark.parametrize("nx,ny,nz,ldx", SHAPES)
def test_ragged_shapes_bitwise(cuda_lib, nx, ny, nz, ldx):
    d = si.pw_inputs(nx, ny, nz, ldx=ldx)
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx)
    got = run_gpu(cuda_lib, d, nx=nx)
    for g, w in zip(got, want):
        assert_interior_bitwise(g, w, nx)
        # halos and pitch padding of the outputs are never written
        m = np.ones_like(g, dtype=bool)
        m[1:-1, 1:-1, 1:nx + 1] = False
        assert np.all(np.isnan(g[m]))


def test_constant_fields_exact_zero(cuda_lib):
    # P2 on the GPU: tzc1 == tzc2, tzd1 == tzd2 => exactly +0 (any FMA contraction breaks it)
    nz, ny, nx = 20, 19, 70
    shape = (nz + 2, ny + 2, nx + 2)
    d = si.pw_coefficients(nz)
    d["tzc2"], d["tzd2"] = d["tzc1"].copy(), d["tzd1"].copy()
    d.update(u=np.full(shape, 0.1), v=np.full(shape, 0.3), w=np.full(shape, 0.7))
    for s in run_gpu(cuda_lib, d, fill=0.0):
        assert np.all(s[1:-1, 1:-1, 1:-1] == 0.0) and not np.any(np.signbit(s))


@pytest.mark.slow
def test_C3_full_size_bitwise(cuda_lib):
    # configs[2]: 512^3 interior, every interior point vs the oracle
    n = 512
    d = si.pw_inputs(n, n, n)
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    got = run_gpu(cuda_lib, d)
    for g, w in zip(got, want):
        assert_interior_bitwise(g, w, n)


def test_u_v_w_may_alias_without_comm(cuda_lib):
    import torch
    nz, ny, nx = 6, 10, 66
    d = si.pw_inputs(nx, ny, nz)
    d["v"] = d["u"]
    d["w"] = d["u"]
    want = oracle.pw_advect3d(d["u"], d["u"], d["u"], d)
    g = to_dev(d)
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    cuda_lib.st_pw_advect3d(g["u"], g["u"], g["u"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"],
                            g["tzd1"], g["tzd2"])
    for o, w in zip(outs, want):
        assert_interior_bitwise(o.cpu().numpy(), w, nx)
