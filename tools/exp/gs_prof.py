"""ncu driver: one in-place Gauss-Seidel launch (16384^2, --sweeps sweeps)."""
import sys, pathlib, argparse
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))
import torch
import paper_2310_01882_b200 as st
import stencil_inputs as si
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--ny", type=int, default=0)
args = ap.parse_args()
a = torch.from_numpy(si.jacobi2d_grid(args.n, args.ny or args.n)).cuda()
for sw in (1, args.sweeps):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(); st.st_gauss_seidel2d_run(a, sw); ev1.record(); ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(f"nx={args.n} ny={args.ny or args.n} {sw} sweeps: {ms:.3f} ms = {ms * 1e3 / (sw * (args.n + 31)):.3f} us/step", flush=True)
