"""Runs the decomposed CUDA path with a LOCAL rank group on one GPU (P ranks in
this process) and checks the gathered result against the oracle, bitwise.
Executed as a subprocess by tests/test_gpu_local_group.py so that
CUDA_DEVICE_MAX_CONNECTIONS is set before CUDA initialises (each rank uses its
own main + comm stream; the ranks' calls are issued one after another and
ordered on the device)."""
import pathlib
import os
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import oracle
import paper_2310_01882_b200 as st
import stencil_inputs as si


def slab2d(g, nranks, r, h):
    ny = g.shape[0] - 2
    start, n = st.st_block_split(ny, nranks, r)
    buf = np.zeros((n + 2 * h, g.shape[1]))
    for l in range(n + 2 * h):
        gr = start + 1 + (l - h)
        if 0 <= gr <= ny + 1:
            buf[l] = g[gr]
    return buf, start, n


def jacobi2d_case(P, nx, ny, h, iters, tblock, poison=True):
    g = si.jacobi2d_grid(nx, ny)
    comms = st.Comm.local_group(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ranks = []
    for r in range(P):
        buf, start, n = slab2d(g, P, r, h)
        a = torch.from_numpy(buf).cuda()
        if poison:  # ghosts of middle ranks must come from the swap
            if r > 0:
                a[:h] = float("nan")
            if r < P - 1:
                a[h + n:] = float("nan")
        b = torch.full_like(a, float("nan"))
        comms[r].bind([a, b], n)
        ranks.append((a, b, start, n))
    torch.cuda.synchronize()
    outs = []
    for r in range(P):
        a, b, start, n = ranks[r]
        with torch.cuda.stream(streams[r]):
            outs.append(st.st_jacobi2d_run(a, b, iters, tblock=tblock, halo=h, comm=comms[r], nx=nx))
    torch.cuda.synchronize()
    want = oracle.jacobi2d(g, iters, nx=nx)
    ok = True
    for r in range(P):
        _, _, start, n = ranks[r]
        got = outs[r].cpu().numpy()[h:h + n, :nx + 2]
        ok &= bool(np.array_equal(got, want[start + 1:start + 1 + n, :nx + 2]))
    for c in comms:
        c.close()
    return ok


def jacobi3d_case(P, nx, ny, nz, h, iters, tblock=0):
    g = si.jacobi3d_grid(nx, ny, nz)
    comms = st.Comm.local_group(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ranks = []
    for r in range(P):
        start, n = st.st_block_split(nz, P, r)
        loc = np.zeros((n + 2 * h, ny + 2, g.shape[2]))
        for l in range(n + 2 * h):
            gz = start + 1 + (l - h)
            if 0 <= gz <= nz + 1:
                loc[l] = g[gz]
        if r > 0:
            loc[:h] = np.nan  # ghost planes must come from the swap (incl. their side faces)
        if r < P - 1:
            loc[h + n:] = np.nan
        a = torch.from_numpy(loc).cuda()
        b = torch.full_like(a, float("nan"))
        comms[r].bind([a, b], n)
        ranks.append((a, b, start, n))
    torch.cuda.synchronize()
    outs = []
    for r in range(P):
        a, b, start, n = ranks[r]
        with torch.cuda.stream(streams[r]):
            outs.append(st.st_jacobi3d_run(a, b, iters, tblock=tblock, halo=h, comm=comms[r], nx=nx))
    torch.cuda.synchronize()
    want = oracle.jacobi3d(g, iters, nx=nx)
    ok = True
    for r in range(P):
        _, _, start, n = ranks[r]
        ok &= bool(np.array_equal(outs[r].cpu().numpy()[h:h + n], want[start + 1:start + 1 + n]))
    for c in comms:
        c.close()
    return ok


def pw_case(P, nx, ny, nz):
    d = si.pw_inputs(nx, ny, nz)
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    comms = st.Comm.local_group(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = []
    for r in range(P):
        z0, n = st.st_block_split(nz, P, r)
        dl = si.pw_inputs(nx, ny, nz, plane0=z0, planes=n + 2)
        g = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in dl.items()}
        for k in "uvw":
            if r > 0:
                g[k][0] = float("nan")
            if r < P - 1:
                g[k][-1] = float("nan")
        outs = [torch.zeros_like(g["u"]) for _ in range(3)]
        comms[r].bind([g["u"], g["v"], g["w"]], n)
        parts.append((g, outs, z0, n))
    torch.cuda.synchronize()
    for r in range(P):
        g, outs, _, _ = parts[r]
        with torch.cuda.stream(streams[r]):
            st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"],
                              g["tzd2"], comm=comms[r])
    torch.cuda.synchronize()
    ok = True
    for g, outs, z0, n in parts:
        for o, w in zip(outs, want):
            ok &= bool(np.array_equal(o.cpu().numpy()[1:n + 1], w[z0 + 1:z0 + 1 + n]))
    for c in comms:
        c.close()
    return ok


def pencil_block(g, ny, nz, py, pz, r):
    y0, nyl, z0, nzl = st.st_pencil_split(ny, nz, py, pz, r)
    return np.ascontiguousarray(g[z0:z0 + nzl + 2, y0:y0 + nyl + 2]), y0, nyl, z0, nzl


def pencil_block_h(g, ny, nz, py, pz, r, h):
    """Rank r's block with h ghost layers in y and z (layers beyond the global grid: NaN)."""
    y0, nyl, z0, nzl = st.st_pencil_split(ny, nz, py, pz, r)
    p = h - 1
    gp = np.pad(g, ((p, p), (p, p), (0, 0)), constant_values=np.nan) if p else g
    # global row y0 + 1 (the first owned) sits at buffer row h, i.e. gp row y0 + 1 + p
    return np.ascontiguousarray(gp[z0:z0 + nzl + 2 * h, y0:y0 + nyl + 2 * h]), y0, nyl, z0, nzl


def pencils_j3_case(py, pz, nx, ny, nz, iters, halo=1, tblock=0):
    P = py * pz
    h = halo
    g = si.jacobi3d_grid(nx, ny, nz)
    comms = st.Comm.local_group(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ranks = []
    for r in range(P):
        loc, y0, nyl, z0, nzl = pencil_block_h(g, ny, nz, py, pz, r, h)
        a = torch.from_numpy(loc).cuda()
        iy, iz = r % py, r // py
        if iy > 0:
            a[:, :h] = float("nan")
        if iy < py - 1:
            a[:, -h:] = float("nan")
        if iz > 0:
            a[:h] = float("nan")
        if iz < pz - 1:
            a[-h:] = float("nan")
        b = torch.full_like(a, float("nan"))
        comms[r].set_grid(py, nyl)
        comms[r].bind([a, b], nzl)
        ranks.append((a, b, y0, nyl, z0, nzl))
    torch.cuda.synchronize()
    outs = []
    for r in range(P):
        a, b = ranks[r][:2]
        with torch.cuda.stream(streams[r]):
            outs.append(st.st_jacobi3d_run_pencils(a, b, iters, comm=comms[r], nx=nx, halo=h, tblock=tblock))
    torch.cuda.synchronize()
    want = oracle.jacobi3d(g, iters, nx=nx)
    ok = True
    for r in range(P):
        _, _, y0, nyl, z0, nzl = ranks[r]
        got = outs[r].cpu().numpy()[h:nzl + h, h:nyl + h, :nx + 2]
        ok &= bool(np.array_equal(got, want[z0 + 1:z0 + 1 + nzl, y0 + 1:y0 + 1 + nyl, :nx + 2]))
    for c in comms:
        c.close()
    return ok


def pencils_pw_case(py, pz, nx, ny, nz):
    P = py * pz
    d = si.pw_inputs(nx, ny, nz)
    want = oracle.pw_advect3d(d["u"], d["v"], d["w"], d)
    comms = st.Comm.local_group(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = []
    for r in range(P):
        y0, nyl, z0, nzl = st.st_pencil_split(ny, nz, py, pz, r)
        iy, iz = r % py, r // py
        g = {}
        for k in "uvw":
            blk = torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2, y0:y0 + nyl + 2])).cuda()
            if iy > 0:
                blk[:, 0] = float("nan")
            if iy < py - 1:
                blk[:, -1] = float("nan")
            if iz > 0:
                blk[0] = float("nan")
            if iz < pz - 1:
                blk[-1] = float("nan")
            g[k] = blk
        for k in ("tzc1", "tzc2", "tzd1", "tzd2"):
            g[k] = torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2])).cuda()
        outs = [torch.zeros_like(g["u"]) for _ in range(3)]
        comms[r].set_grid(py, nyl)
        comms[r].bind([g["u"], g["v"], g["w"]], nzl)
        parts.append((g, outs, y0, nyl, z0, nzl))
    torch.cuda.synchronize()
    for r in range(P):
        g, outs = parts[r][:2]
        with torch.cuda.stream(streams[r]):
            st.st_pw_advect3d_pencils(g["u"], g["v"], g["w"], *outs, d["tcx"], d["tcy"], g["tzc1"], g["tzc2"],
                                      g["tzd1"], g["tzd2"], comm=comms[r])
    torch.cuda.synchronize()
    ok = True
    for g, outs, y0, nyl, z0, nzl in parts:
        for o, w in zip(outs, want):
            ok &= bool(np.array_equal(o.cpu().numpy()[1:nzl + 1, 1:nyl + 1, 1:nx + 1],
                                      w[z0 + 1:z0 + 1 + nzl, y0 + 1:y0 + 1 + nyl, 1:nx + 1]))
    for c in comms:
        c.close()
    return ok


def late_rank_case():
    """Failure detection: rank 1 does not join the swap; rank 0's
    st_comm_wait reports ST_ETIMEDOUT instead of hanging or returning wrong data.
    Then rank 1 joins late and the swap completes with the right ghost rows."""
    P, nx, n, w = 2, 64, 16, 1
    comms = st.Comm.local_group(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    bufs = []
    for r in range(P):
        t = torch.full((n + 2 * w, nx + 2), float(r + 1), dtype=torch.float64, device="cuda")
        comms[r].bind([t], n)
        bufs.append(t)
    torch.cuda.synchronize()
    with torch.cuda.stream(streams[0]):
        st.st_halo_exchange(comms[0], [bufs[0]], n, nx + 2, w)
    timed_out = False
    try:
        comms[0].wait(streams[0], timeout_ms=300)
    except st.StencilError as e:
        timed_out = e.code == st.ST_ETIMEDOUT
    # the timed-out comm is broken: a new swap fails fast instead of queueing behind the wait
    refused = False
    try:
        st.st_halo_exchange(comms[0], [bufs[0]], n, nx + 2, w)
    except st.StencilError as e:
        refused = e.code == st.ST_ENCCL
    with torch.cuda.stream(streams[1]):
        st.halo_exchange(comms[1], [bufs[1]], w)  # SURVEY §8(b) convention (shape-derived slabs)
    comms[0].wait(streams[0], timeout_ms=10000)
    comms[1].wait(streams[1], timeout_ms=10000)
    torch.cuda.synchronize()
    ok = timed_out and refused and bool((bufs[0][n + w:] == 2.0).all()) and bool((bufs[1][:w] == 1.0).all())
    for c in comms:
        c.close()
    return ok


def connections_case():
    """Ranks sharing a device need CUDA_DEVICE_MAX_CONNECTIONS >= 2k+1 (run with it unset:
    the default 8 admits 3 ranks per device, not 4)."""
    assert "CUDA_DEVICE_MAX_CONNECTIONS" not in os.environ
    three = st.Comm.local_group(3)
    for c in three:
        c.close()
    try:
        st.Comm.local_group(4)
    except st.StencilError as e:
        return e.code == st.ST_ENOTSUP and "CUDA_DEVICE_MAX_CONNECTIONS" in str(e)
    return False


CASES = {
    "late_rank": late_rank_case,
    "connections": connections_case,
    "pen_j3_2x1": lambda: pencils_j3_case(2, 1, 70, 40, 33, 6),
    "pen_j3_1x2": lambda: pencils_j3_case(1, 2, 70, 40, 33, 6),
    "pen_j3_2x2": lambda: pencils_j3_case(2, 2, 66, 37, 31, 7),
    "pen_j3_3x2": lambda: pencils_j3_case(3, 2, 40, 50, 21, 5),
    # two sweeps per pass on pencils (ghost depth 2): odd/even sweep counts, blocks thin
    # enough that the ghost-free interior is empty, ragged tiles in y
    "pen_j3t2_2x1": lambda: pencils_j3_case(2, 1, 70, 40, 33, 6, halo=2, tblock=2),
    "pen_j3t2_1x2": lambda: pencils_j3_case(1, 2, 70, 40, 33, 7, halo=2, tblock=2),
    "pen_j3t2_2x2": lambda: pencils_j3_case(2, 2, 130, 37, 31, 9, halo=2),
    "pen_j3t2_3x2": lambda: pencils_j3_case(3, 2, 40, 50, 21, 4, halo=2, tblock=2),
    "pen_j3t2_2x3_thin": lambda: pencils_j3_case(2, 3, 33, 7, 9, 5, halo=2, tblock=2),
    "pen_j3h2_t1_2x2": lambda: pencils_j3_case(2, 2, 66, 37, 31, 5, halo=2, tblock=1),
    "pen_pw_2x2": lambda: pencils_pw_case(2, 2, 70, 30, 22),
    "pen_pw_3x2": lambda: pencils_pw_case(3, 2, 40, 33, 17),
    "pen_pw_1x3": lambda: pencils_pw_case(1, 3, 40, 20, 25),
    "j2_h1": lambda: jacobi2d_case(2, 130, 200, 1, 9, 1),
    "j2_p3_h1": lambda: jacobi2d_case(3, 70, 101, 1, 7, 1),
    "j2_h4_t4": lambda: jacobi2d_case(2, 300, 260, 4, 13, 4),
    "j2_p4_h6_t6": lambda: jacobi2d_case(4, 260, 520, 6, 25, 6),
    "j2_p3_h3_t1": lambda: jacobi2d_case(3, 90, 99, 3, 10, 1),
    "j3_h1": lambda: jacobi3d_case(2, 70, 40, 33, 1, 7),
    "j3_p3_h2": lambda: jacobi3d_case(3, 40, 30, 31, 2, 6),          # auto: two sweeps per pass
    "j3_p3_h2_t1": lambda: jacobi3d_case(3, 40, 30, 31, 2, 6, 1),
    "j3_p2_h2_t2": lambda: jacobi3d_case(2, 140, 37, 40, 2, 9, 2),   # odd iters: a 1-sweep pass
    "j3_p4_h3_t2": lambda: jacobi3d_case(4, 70, 20, 23, 3, 11, 2),   # slabs of 5-6 planes < 2*halo
    "j3_p2_h4_t2": lambda: jacobi3d_case(2, 33, 17, 300, 4, 12, 2),  # several T=2 chunks per slab
    "j3_p2_h2_t2_b": lambda: jacobi3d_case(2, 70, 33, 29, 2, 9, 0),
    "pw_p2": lambda: pw_case(2, 140, 20, 41),
    "pw_p4": lambda: pw_case(4, 70, 17, 40),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    bad = [n for n in names if not CASES[n]()]
    print("LOCAL-GROUP CASES", "FAILED: " + ",".join(bad) if bad else "OK", flush=True)
    sys.exit(1 if bad else 0)
