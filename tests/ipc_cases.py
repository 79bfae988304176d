"""Multi-process IPC-transport cases (spawned by tests/test_gpu_ipc.py): every
rank is its own process; all ranks may share one GPU (the IPC transport allows
it, NCCL does not). Bitwise vs the oracle."""
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np
import torch
import torch.distributed as dist

import oracle
import paper_2310_01882_b200 as st
import stencil_inputs as si


def jacobi2d(rank, world, dev, h, iters, tblock):
    nx, ny = 300, 260
    g = si.jacobi2d_grid(nx, ny)
    start, n = st.st_block_split(ny, world, rank)
    loc = np.zeros((n + 2 * h, g.shape[1]))
    for l in range(n + 2 * h):
        gr = start + 1 + (l - h)
        if 0 <= gr <= ny + 1:
            loc[l] = g[gr]
    a = torch.from_numpy(loc).to(dev)
    if rank > 0:
        a[:h] = float("nan")
    if rank < world - 1:
        a[h + n:] = float("nan")
    b = torch.full_like(a, float("nan"))
    comm = st.Comm.ipc_from_process_group(dev.index)
    comm.bind_ipc([a, b], n)
    r = st.st_jacobi2d_run(a, b, iters, tblock=tblock, halo=h, comm=comm, nx=nx)
    torch.cuda.synchronize()
    rows = [None] * world
    dist.all_gather_object(rows, (start, r.cpu().numpy()[h:h + n, :nx + 2]))
    comm.close()
    if rank == 0:
        want = oracle.jacobi2d(g, iters, nx=nx)
        return all(np.array_equal(blk, want[s0 + 1:s0 + 1 + blk.shape[0], :nx + 2]) for s0, blk in rows)
    return True


def jacobi3d(rank, world, dev, h, iters, tblock, nx=70, ny=33, nz=29):
    # z slabs; h >= 2 runs two sweeps per pass (jacobi3d_t2_kernel) across ranks
    g = si.jacobi3d_grid(nx, ny, nz)
    start, n = st.st_block_split(nz, world, rank)
    loc = np.zeros((n + 2 * h, ny + 2, g.shape[2]))
    for l in range(n + 2 * h):
        gz = start + 1 + (l - h)
        if 0 <= gz <= nz + 1:
            loc[l] = g[gz]
    a = torch.from_numpy(loc).to(dev)
    if rank > 0:
        a[:h] = float("nan")
    if rank < world - 1:
        a[h + n:] = float("nan")
    b = torch.full_like(a, float("nan"))
    comm = st.Comm.ipc_from_process_group(dev.index)
    comm.bind_ipc([a, b], n)
    r = st.st_jacobi3d_run(a, b, iters, tblock=tblock, halo=h, comm=comm, nx=nx)
    torch.cuda.synchronize()
    blocks = [None] * world
    dist.all_gather_object(blocks, (start, r.cpu().numpy()[h:h + n, :, :nx + 2]))
    comm.close()
    if rank == 0:
        want = oracle.jacobi3d(g, iters, nx=nx)
        ok = True
        for r, (s0, blk) in enumerate(blocks):
            w = want[s0 + 1:s0 + 1 + blk.shape[0], :, :nx + 2]
            if not np.array_equal(blk, w):
                bad = np.argwhere(blk.view(np.uint64) != w.view(np.uint64))
                print(f"rank {r}: {len(bad)} mismatches, planes {sorted(set(bad[:, 0].tolist()))[:10]}, "
                      f"first {bad[:3].tolist()}", flush=True)
                ok = False
        return ok
    return True


def pw(rank, world, dev):
    nx, ny, nz = 140, 20, 41
    d = si.pw_inputs(nx, ny, nz)
    z0, n = st.st_block_split(nz, world, rank)
    dl = si.pw_inputs(nx, ny, nz, plane0=z0, planes=n + 2)
    g = {k: (torch.from_numpy(v).to(dev) if isinstance(v, np.ndarray) else v) for k, v in dl.items()}
    for k in "uvw":
        if rank > 0:
            g[k][0] = float("nan")
        if rank < world - 1:
            g[k][-1] = float("nan")
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    comm = st.Comm.ipc_from_process_group(dev.index)
    comm.bind_ipc([g["u"], g["v"], g["w"]], n)
    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"],
                      comm=comm)
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, (z0, [o.cpu().numpy()[1:n + 1] for o in outs]))
    comm.close()
    if rank == 0:
        want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
        return all(np.array_equal(blk, w[s0 + 1:s0 + 1 + blk.shape[0]]) for s0, blks in parts
                   for blk, w in zip(blks, want))
    return True


def pencils(rank, world, dev, which):
    py = 2 if world % 2 == 0 else world
    pz = world // py
    nx, ny, nz = 70, 37, 29
    y0, nyl, z0, nzl = st.st_pencil_split(ny, nz, py, pz, rank)
    iy, iz = rank % py, rank // py
    comm = st.Comm.ipc_from_process_group(dev.index)
    comm.set_grid(py, nyl)

    def block(f):
        t = torch.from_numpy(np.ascontiguousarray(f[z0:z0 + nzl + 2, y0:y0 + nyl + 2])).to(dev)
        if iy > 0:
            t[:, 0] = float("nan")
        if iy < py - 1:
            t[:, -1] = float("nan")
        if iz > 0:
            t[0] = float("nan")
        if iz < pz - 1:
            t[-1] = float("nan")
        return t

    if which in ("j3", "j3t2"):
        h = 2 if which == "j3t2" else 1
        g = si.jacobi3d_grid(nx, ny, nz)
        if h == 1:
            a = block(g)
        else:  # two ghost layers (beyond the global grid: NaN), two sweeps per pass
            gp = np.pad(g, ((1, 1), (1, 1), (0, 0)), constant_values=np.nan)
            a = torch.from_numpy(np.ascontiguousarray(gp[z0:z0 + nzl + 4, y0:y0 + nyl + 4])).to(dev)
            if iy > 0:
                a[:, :2] = float("nan")
            if iy < py - 1:
                a[:, -2:] = float("nan")
            if iz > 0:
                a[:2] = float("nan")
            if iz < pz - 1:
                a[-2:] = float("nan")
        b = torch.full_like(a, float("nan"))
        comm.bind_ipc([a, b], nzl)
        r = st.st_jacobi3d_run_pencils(a, b, 7, comm=comm, nx=nx, halo=h, tblock=h)
        torch.cuda.synchronize()
        got = [r.cpu().numpy()[h:nzl + h, h:nyl + h, :nx + 2]]
        want_full = [oracle.jacobi3d(g, 7, nx=nx)]
        sl = (slice(z0 + 1, z0 + 1 + nzl), slice(y0 + 1, y0 + 1 + nyl), slice(0, nx + 2))
    else:
        d = si.pw_inputs(nx, ny, nz)
        u, v, w = block(d["u"]), block(d["v"]), block(d["w"])
        tz = [torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2])).to(dev)
              for k in ("tzc1", "tzc2", "tzd1", "tzd2")]
        outs = [torch.zeros_like(u) for _ in range(3)]
        comm.bind_ipc([u, v, w], nzl)
        st.st_pw_advect3d_pencils(u, v, w, *outs, d["tcx"], d["tcy"], *tz, comm=comm, nx=nx)
        torch.cuda.synchronize()
        got = [o.cpu().numpy()[1:nzl + 1, 1:nyl + 1, 1:nx + 1] for o in outs]
        want_full = list(oracle.pw_advect3d(d["u"], d["v"], d["w"], d, nx=nx))
        sl = (slice(z0 + 1, z0 + 1 + nzl), slice(y0 + 1, y0 + 1 + nyl), slice(1, nx + 1))
    ok = all(np.array_equal(gg, ww[sl]) for gg, ww in zip(got, want_full))
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    comm.close()
    return all(oks)


def c4_bands(rank, world, dev, iters=24, h=8, ny_rank=4096):
    """Pre-flight of the N = 8 launch shapes: C4's full width (32768
    interior columns), slabs of 4096 rows as at N = 8, H = 8 ghost rows, T = 8
    across ranks, fused neighbour stores. Bands around every slab boundary and the
    ring rows are compared bitwise with the oracle run on windows widened by the
    influence radius (`iters` rows)."""
    nx = 32768
    ny = ny_rank * world
    ld = nx + 2
    start, n = st.st_block_split(ny, world, rank)
    lo, hi = max(0, start + 1 - h), min(ny + 1, start + n + h)  # global padded rows present in the slab
    loc = np.zeros((n + 2 * h, ld))
    loc[lo - (start + 1 - h): hi - (start + 1 - h) + 1] = si.jacobi2d_grid(nx, ny, ld=ld, row0=lo, rows=hi - lo + 1)
    a = torch.from_numpy(loc).to(dev)
    del loc
    if rank > 0:
        a[:h] = float("nan")
    if rank < world - 1:
        a[h + n:] = float("nan")
    b = torch.full_like(a, float("nan"))
    comm = st.Comm.ipc_from_process_group(dev.index)
    comm.bind_ipc([a, b], n)
    r = st.st_jacobi2d_run(a, b, iters, tblock=0, halo=h, comm=comm)
    torch.cuda.synchronize()
    band = 40
    mine = {}
    for g0 in (start + 1, start + n - band + 1):  # first / last `band` owned rows (global padded index)
        l0 = g0 - (start + 1) + h
        mine[g0] = r[l0:l0 + band].cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    comm.close()
    if rank != 0:
        return True
    ok = True
    for part in parts:
        for g0, got in part.items():
            w0, w1 = max(0, g0 - iters), min(ny + 1, g0 + band - 1 + iters)
            win = si.jacobi2d_grid(nx, ny, ld=ld, row0=w0, rows=w1 - w0 + 1)
            want = oracle.jacobi2d(win, iters, nx=nx)[g0 - w0: g0 - w0 + band]
            bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
            if bad.size:
                print(f"rows {g0}..{g0 + band - 1}: {len(bad)} mismatches, first {bad[:3].tolist()}", flush=True)
                ok = False
    return ok


def c5_planes(rank, world, dev):
    """Pre-flight of C5's slab shapes: PW 1024 x 1024 x 512 in z-slabs (128 planes at
    P = 4), ghost planes swapped by the transport; the first/last owned planes of
    every slab (the ones that read swapped ghosts) and one interior plane are
    compared bitwise with the oracle on their 3-plane input windows."""
    nx = ny = 1024
    nz = 512
    z0, n = st.st_block_split(nz, world, rank)
    dl = si.pw_inputs(nx, ny, nz, plane0=z0, planes=n + 2)
    g = {k: (torch.from_numpy(v).to(dev) if isinstance(v, np.ndarray) else v) for k, v in dl.items()}
    del dl
    for k in "uvw":
        if rank > 0:
            g[k][0] = float("nan")
        if rank < world - 1:
            g[k][-1] = float("nan")
    outs = [torch.zeros_like(g["u"]) for _ in range(3)]
    comm = st.Comm.ipc_from_process_group(dev.index)
    comm.bind_ipc([g["u"], g["v"], g["w"]], n)
    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"],
                      comm=comm)
    torch.cuda.synchronize()
    mine = {z0 + l: [o[l].cpu().numpy() for o in outs] for l in (1, n // 2, n)}  # local plane l = global z0 + l
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    comm.close()
    if rank != 0:
        return True
    ok = True
    for part in parts:
        for z, got in part.items():
            win = si.pw_inputs(nx, ny, nz, plane0=z - 1, planes=3)
            want = oracle.pw_advect3d(win["u"], win["v"], win["w"], win, nx=nx)
            for name, gg, ww in zip(("su", "sv", "sw"), got, want):
                if not np.array_equal(gg[1:ny + 1, 1:nx + 1], ww[1, 1:ny + 1, 1:nx + 1]):
                    print(f"plane {z} {name} mismatch", flush=True)
                    ok = False
    return ok


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ngpu)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    case = sys.argv[1]
    ok = {"j2_h1": lambda: jacobi2d(rank, world, dev, 1, 9, 1),
          "j2_h4_t4": lambda: jacobi2d(rank, world, dev, 4, 13, 4),
          "pw": lambda: pw(rank, world, dev),
          "j3_h2_t2": lambda: jacobi3d(rank, world, dev, 2, 9, 0),
          "j3_h2_t1": lambda: jacobi3d(rank, world, dev, 2, 9, 1),
          "j3_h1": lambda: jacobi3d(rank, world, dev, 1, 5, 1),
          "j3_dbg": lambda: jacobi3d(rank, world, dev, int(os.environ["J3_H"]), int(os.environ["J3_IT"]),
                                     int(os.environ["J3_TB"]), *[int(v) for v in os.environ["J3_DIMS"].split(",")]),
          "j3_h3_t2": lambda: jacobi3d(rank, world, dev, 3, 8, 2),
          "pen_j3": lambda: pencils(rank, world, dev, "j3"),
          "pen_pw": lambda: pencils(rank, world, dev, "pw"),
          "pen_j3t2": lambda: pencils(rank, world, dev, "j3t2"),
          "c4_bands": lambda: c4_bands(rank, world, dev),
          "c5_planes": lambda: c5_planes(rank, world, dev)}[case]()
    if rank == 0:
        print("IPC CASE", case, "OK" if ok else "FAILED", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
