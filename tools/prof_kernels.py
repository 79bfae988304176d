"""Small driver for ncu captures: a few C2 Jacobi sweeps and C3 PW applications
(the same kernels and launch configurations bench.py times)."""
import argparse
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import torch

import paper_2310_01882_b200 as st
import stencil_inputs as si

ap = argparse.ArgumentParser()
ap.add_argument("--sweeps", type=int, default=4)
ap.add_argument("--apps", type=int, default=2)
ap.add_argument("--tblock", type=int, default=1)
ap.add_argument("--gs-sweeps", type=int, default=4)
args = ap.parse_args()

n = 16384
a = torch.from_numpy(si.jacobi2d_grid(n, n)).cuda()
b = torch.empty_like(a)
st.st_jacobi2d_run(a, b, args.sweeps, tblock=args.tblock)
torch.cuda.synchronize()
del a, b
m = 512
d = si.pw_inputs(m, m, m)
g = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in d.items()}
outs = [torch.empty_like(g["u"]) for _ in range(3)]
for _ in range(args.apps):
    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"])
torch.cuda.synchronize()
del g, outs
a3 = torch.from_numpy(si.jacobi3d_grid(m, m, m)).cuda()
b3 = torch.empty_like(a3)
st.st_jacobi3d_run(a3, b3, 4)  # two T=2 passes (jacobi3d_t2_kernel)
st.st_jacobi3d_run(a3, b3, 1)  # one T=1 sweep (jacobi3d_kernel)
torch.cuda.synchronize()
del a3, b3
ag = torch.from_numpy(si.jacobi2d_grid(n, n)).cuda()
st.st_gauss_seidel2d_run(ag, args.gs_sweeps)
torch.cuda.synchronize()
del ag
ag = torch.rand(n + 2, n + 2, dtype=torch.float64, device="cuda")
st.st_stencil2d_run(ag, torch.empty_like(ag), [(-1, 0), (1, 0), (0, -1), (0, 1)], [0.25] * 4, 2)
torch.cuda.synchronize()
print("done")
