"""Gauss-Seidel throughput, 16384^2 (in place), for a few sweep counts: the
linear model t = fill + sweeps * per_sweep separates the pipeline fill."""
import sys, pathlib, argparse
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))
import torch
import paper_2310_01882_b200 as st
import stencil_inputs as si
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--sweeps", type=str, default="4,100,400")
ap.add_argument("--ny", type=int, default=0)
args = ap.parse_args()
n = args.n
ny = args.ny or n
a = torch.from_numpy(si.jacobi2d_grid(n, ny)).cuda()
ws = torch.empty(int(st.lib().st_gauss_seidel2d_workspace_bytes(n, ny)) // 8 + 1, dtype=torch.int64, device="cuda")
st.st_gauss_seidel2d_run(a, 4, workspace=ws)
torch.cuda.synchronize()
res = []
for sw in [int(x) for x in args.sweeps.split(",")]:
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(); st.st_gauss_seidel2d_run(a, sw, workspace=ws); ev1.record(); ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    res.append((sw, ms))
    print(f"n={n} ny={ny} {sw} sweeps: {ms:.3f} ms = {n * ny * sw / ms / 1e6:.1f} Gpts/s", flush=True)
if len(res) >= 2:
    (s0, t0), (s1, t1) = res[-2], res[-1]
    per = (t1 - t0) / (s1 - s0)
    print(f"steady: {per:.4f} ms/sweep = {n * ny / per / 1e6:.1f} Gpts/s; fill {t1 - s1 * per:.2f} ms")
