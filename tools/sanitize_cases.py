"""Small invocations of every kernel for compute-sanitizer (memcheck/racecheck/synccheck/initcheck)."""
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2310_01882_b200 as st
import stencil_inputs as si

# (500, 400, 16, 8) etc.: interior strips with enough rows for the rotated-register blocks
for nx, ny, iters, tb in ((64, 64, 5, 0), (130, 70, 3, 1), (130, 70, 5, 2), (130, 1100, 9, 4), (61, 37, 8, 8),
                          (500, 400, 16, 8), (400, 300, 12, 6), (300, 200, 8, 4), (300, 200, 6, 2)):
    a = torch.from_numpy(si.jacobi2d_grid(nx, ny)).cuda()
    b = torch.empty_like(a)
    st.st_jacobi2d_run(a, b, iters, tblock=tb)
for nx, ny, nz in ((70, 13, 9), (129, 17, 70)):
    d = si.pw_inputs(nx, ny, nz)
    g = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"])
for nx, ny, nz in ((33, 31, 9), (70, 40, 66)):
    a = torch.from_numpy(si.jacobi3d_grid(nx, ny, nz)).cuda()
    b = torch.empty_like(a)
    st.st_jacobi3d_run(a, b, 3)  # T=1 sweeps (odd pass count)
    st.st_jacobi3d_run(a, b, 4)  # two T=2 passes (jacobi3d_t2_kernel)
# GS: single-sweep tiled (even ld) and register (odd ld) kernels; multi-sweep wavefront (nx >= 382:
# K = 4 passes plus a remainder pass, wide and 8-byte copies)
for nx, ny, ld, iters in ((200, 95, 202, 3), (65, 33, 67, 2), (1000, 130, 1002, 6), (400, 70, 403, 5)):
    a = torch.from_numpy(si.jacobi2d_grid(nx, ny, ld=ld)).cuda()
    st.st_gauss_seidel2d_run(a, iters, nx=nx)
for nx, ny in ((64, 64), (37, 21)):  # register-resident C1 kernel
    a = torch.from_numpy(si.jacobi2d_grid(nx, ny)).cuda()
    st.st_jacobi2d_run(a, torch.empty_like(a), 7)
for offs in ([(-1, 0), (1, 0), (0, -1), (0, 1)], [(3, -2), (-1, 3), (0, 0), (8, 0)]):  # generic stencil
    R = max(max(abs(dy), abs(dx)) for dy, dx in offs)
    a = torch.rand(37 + 2 * R, 45 + 2 * R, dtype=torch.float64, device="cuda")
    st.st_stencil2d_run(a, torch.empty_like(a), offs, [0.5] * len(offs), 3)
a = torch.rand(41, 53, dtype=torch.float64, device="cuda")  # NVRTC expression stencil
st.st_stencil2d_expr_run(a, torch.empty_like(a), "-(a(3,0) - 2*a(0,0)) / 3 + 0.1*a(-2,2)", 3)
torch.cuda.synchronize()
print("sanitize cases done")
