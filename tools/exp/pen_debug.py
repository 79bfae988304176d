import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2] / "tests"))
import numpy as np, torch
import oracle, stencil_inputs as si, paper_2310_01882_b200 as st
py, pz, nx, ny, nz = 3, 2, 40, 33, 17
P = py * pz
d = si.pw_inputs(nx, ny, nz)
want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
comms = st.Comm.local_group(P)
streams = [torch.cuda.Stream() for _ in range(P)]
parts = []
for r in range(P):
    y0, nyl, z0, nzl = st.st_pencil_split(ny, nz, py, pz, r)
    g = {k: torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2, y0:y0 + nyl + 2])).cuda() for k in "uvw"}
    for k in ("tzc1", "tzc2", "tzd1", "tzd2"):
        g[k] = torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2])).cuda()
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    comms[r].set_grid(py, nyl); comms[r].bind([g["u"], g["v"], g["w"]], nzl)
    parts.append((g, outs, y0, nyl, z0, nzl))
torch.cuda.synchronize()
for r in range(P):
    g, outs = parts[r][:2]
    with torch.cuda.stream(streams[r]):
        st.st_pw_advect3d_pencils(g["u"], g["v"], g["w"], *outs, d["tcx"], d["tcy"], g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"], comm=comms[r])
torch.cuda.synchronize()
for r, (g, outs, y0, nyl, z0, nzl) in enumerate(parts):
    # ghosts after the swap vs the global field
    for k in "uvw":
        loc = g[k].cpu().numpy(); ref = d[k][z0:z0 + nzl + 2, y0:y0 + nyl + 2]
        bad = np.argwhere(loc[:, :, :nx + 2] != ref[:, :, :nx + 2])
        if len(bad): print("rank", r, "field", k, "ghost mismatches", len(bad), bad[:4].tolist())
    for c, (o, w) in enumerate(zip(outs, want)):
        bad = np.argwhere(o.cpu().numpy()[1:nzl + 1, 1:nyl + 1, 1:nx + 1] != w[z0 + 1:z0 + 1 + nzl, y0 + 1:y0 + 1 + nyl, 1:nx + 1])
        if len(bad): print("rank", r, "out", c, "mismatches", len(bad), bad[:4].tolist())
print("done")
