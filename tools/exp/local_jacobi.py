"""Debug: LOCAL group jacobi2d, 2 ranks on device 0, poll instead of sync."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import numpy as np
import torch
import paper_2310_01882_b200 as st
import stencil_inputs as si

iters = int(sys.argv[1]); h = int(sys.argv[2]); tb = int(sys.argv[3])
nx, ny, P = 130, 200, 2
g = si.jacobi2d_grid(nx, ny)
comms = st.Comm.local_group(P)
streams = [torch.cuda.Stream() for _ in range(P)]
bufs = []
for r in range(P):
    start, n = st.st_block_split(ny, P, r)
    loc = np.zeros((n + 2 * h, g.shape[1]))
    for l in range(n + 2 * h):
        gr = start + 1 + (l - h)
        if 0 <= gr <= ny + 1:
            loc[l] = g[gr]
    a = torch.from_numpy(loc).cuda(); b = torch.empty_like(a)
    comms[r].bind([a, b], n)
    bufs.append((a, b, n))
torch.cuda.synchronize()
print("ops rank0:", [(o["kind"], o["buf"], o["flag"]) for o in st.st_jacobi2d_schedule(0, P, nx, bufs[0][2], h, iters, tb)][:12], flush=True)
for r in range(P):
    a, b, n = bufs[r]
    with torch.cuda.stream(streams[r]):
        st.st_jacobi2d_run(a, b, iters, tblock=tb, halo=h, comm=comms[r], nx=nx)
    print("issued rank", r, flush=True)
t0 = time.time()
while time.time() - t0 < 8 and not all(s.query() for s in streams):
    time.sleep(0.2)
print("iters", iters, "streams done:", [s.query() for s in streams], "comm streams?", flush=True)
