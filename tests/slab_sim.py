"""Test-side executor of libstencil's Jacobi schedules (st_jacobi2d_schedule,
st_jacobi3d_schedule: the same logic with z planes for rows).

Runs the exact op sequence the CUDA path runs, with a plain NumPy definition
of each op, so the host logic of the decomposition (slab split, ghost depth,
halo-swap placement, redundant ghost rows, temporal-blocking passes, parity)
is checked on CPU against the oracle — either for P simulated ranks in one
process (exchange = array copies) or for real gloo ranks (exchange =
torch.distributed send/recv). Test infrastructure only.
"""
from __future__ import annotations

import numpy as np

import paper_2310_01882_b200 as st


def sweep_pass(src: np.ndarray, dst: np.ndarray, nx: int, y_lo: int, y_hi: int, b: int,
               ring_lo: int, ring_hi: int) -> None:
    """dst rows [y_lo, y_hi] := the state b Jacobi sweeps after src (definition of ST_OP_SWEEP):
    rows <= ring_lo / >= ring_hi are Dirichlet; level l is valid on rows
    [y_lo-(b-l), y_hi+(b-l)], which is all that level b needs."""
    nrows = src.shape[0]
    cur = src.copy()
    for lvl in range(1, b + 1):
        lo = max(y_lo - (b - lvl), ring_lo + 1, 1)
        hi = min(y_hi + (b - lvl), ring_hi - 1, nrows - 2)
        nxt = cur.copy()
        if hi >= lo:
            nxt[lo:hi + 1, 1:nx + 1] = (((cur[lo - 1:hi, 1:nx + 1] + cur[lo + 1:hi + 2, 1:nx + 1])
                                         + cur[lo:hi + 1, 0:nx]) + cur[lo:hi + 1, 2:nx + 2]) * 0.25
        cur = nxt
    dst[y_lo:y_hi + 1, :nx + 2] = cur[y_lo:y_hi + 1, :nx + 2]


def sweep_pass3d(src: np.ndarray, dst: np.ndarray, nx: int, z_lo: int, z_hi: int, b: int,
                 ring_lo: int, ring_hi: int) -> None:
    """3-D ST_OP_SWEEP: dst planes [z_lo, z_hi] := b 7-point sweeps after src (sum order z-, z+,
    y-, y+, x-, x+, then / 6; R20/R21); planes <= ring_lo / >= ring_hi are Dirichlet."""
    nplanes, ny = src.shape[0], src.shape[1] - 2
    cur = src.copy()
    for lvl in range(1, b + 1):
        lo = max(z_lo - (b - lvl), ring_lo + 1, 1)
        hi = min(z_hi + (b - lvl), ring_hi - 1, nplanes - 2)
        nxt = cur.copy()
        if hi >= lo:
            c = lambda dz, dy, dx: cur[lo + dz:hi + 1 + dz, 1 + dy:ny + 1 + dy, 1 + dx:nx + 1 + dx]
            nxt[lo:hi + 1, 1:ny + 1, 1:nx + 1] = (((((c(-1, 0, 0) + c(1, 0, 0)) + c(0, -1, 0)) + c(0, 1, 0))
                                                    + c(0, 0, -1)) + c(0, 0, 1)) / 6.0
        cur = nxt
    dst[z_lo:z_hi + 1, :, :nx + 2] = cur[z_lo:z_hi + 1, :, :nx + 2]


def slab_arrays(a_glob: np.ndarray, nranks: int, rank: int, h: int):
    """Rank slab of the global padded grid with h ghost rows per side (zeros where no row exists)."""
    ny = a_glob.shape[0] - 2
    start, n = st.st_block_split(ny, nranks, rank)
    buf = np.zeros((n + 2 * h,) + a_glob.shape[1:])
    for l in range(n + 2 * h):
        g = start + 1 + (l - h)
        if 0 <= g <= ny + 1:
            buf[l] = a_glob[g]
    return buf, start, n


def run_simulated(a_glob: np.ndarray, nx: int, nranks: int, h: int, iters: int, tblock: int) -> np.ndarray:
    """All ranks in one process; returns the gathered global result. A 3-D a_glob
    (planes, ny+2, ldx) runs st_jacobi3d_schedule with 3-D sweeps."""
    ny = a_glob.shape[0] - 2
    dims = a_glob.ndim
    schedule = st.st_jacobi3d_schedule if dims == 3 else st.st_jacobi2d_schedule
    sweep = sweep_pass3d if dims == 3 else sweep_pass
    ranks = []
    for r in range(nranks):
        a, start, n = slab_arrays(a_glob, nranks, r, h)
        b = a.copy()  # the library copies ghost/Dirichlet rows a -> b
        ops = schedule(r, nranks, nx, n, h, iters, tblock)
        ranks.append({"buf": [a, b], "start": start, "n": n, "ops": ops})
    # ranks run independently between swaps (a slab thinner than 2*halo has no boundary/interior
    # split, so op lists may differ); every rank has the same number of swaps, executed together
    nex = {sum(o["kind"] == st.OP_EXCHANGE for o in x["ops"]) for x in ranks}
    assert len(nex) == 1, "every rank takes part in every swap"
    pos = [0] * nranks
    pitch = int(np.prod(a_glob.shape[1:]))
    for _ in range(nex.pop() + 1):
        ex = []
        for r, x in enumerate(ranks):
            while pos[r] < len(x["ops"]) and x["ops"][pos[r]]["kind"] != st.OP_EXCHANGE:
                o = x["ops"][pos[r]]
                if o["kind"] == st.OP_SWEEP:
                    sweep(x["buf"][o["buf"]], x["buf"][1 - o["buf"]], nx, o["y_lo"], o["y_hi"], o["sweeps"],
                          o["ring_lo"], o["ring_hi"])
                pos[r] += 1
            ex.append(x["ops"][pos[r]] if pos[r] < len(x["ops"]) else None)
            pos[r] += 1
        if ex[0] is None:
            break
        assert len({o["sweeps"] for o in ex}) == 1
        flat = [x["buf"][o["buf"]].reshape(-1) for x, o in zip(ranks, ex)]
        snap = [f.copy() for f in flat]
        for r, x in enumerate(ranks):
            w = ex[r]["sweeps"]
            sends, recvs = st.st_halo_plan(r, nranks, x["n"], pitch, w)
            for peer, off, cnt in recvs:
                # what peer sends to r
                ps, _ = st.st_halo_plan(peer, nranks, ranks[peer]["n"], pitch, w)
                src = [s for s in ps if s[0] == r][0]
                assert src[2] == cnt
                flat[r][off:off + cnt] = snap[peer][src[1]:src[1] + cnt]
    out = np.zeros_like(a_glob)
    for r, x in enumerate(ranks):
        fin = x["buf"][iters & 1]
        out[x["start"] + 1: x["start"] + 1 + x["n"]] = fin[h:h + x["n"]]
        if r == 0:
            out[0] = fin[h - 1]
        if r == nranks - 1:
            out[ny + 1] = fin[h + x["n"]]
    return out


def run_gloo_rank(a_glob: np.ndarray, nx: int, h: int, iters: int, tblock: int) -> np.ndarray | None:
    """One real rank (torch.distributed, gloo): executes its schedule with send/recv
    halo swaps per st_halo_plan; returns the gathered result on rank 0."""
    import torch
    import torch.distributed as dist
    rank, nranks = dist.get_rank(), dist.get_world_size()
    ny = a_glob.shape[0] - 2
    a, start, n = slab_arrays(a_glob, nranks, rank, h)
    buf = [a, a.copy()]
    pitch = int(np.prod(a_glob.shape[1:]))
    schedule = st.st_jacobi3d_schedule if a_glob.ndim == 3 else st.st_jacobi2d_schedule
    sweep = sweep_pass3d if a_glob.ndim == 3 else sweep_pass
    for o in schedule(rank, nranks, nx, n, h, iters, tblock):
        if o["kind"] == st.OP_SWEEP:
            sweep(buf[o["buf"]], buf[1 - o["buf"]], nx, o["y_lo"], o["y_hi"], o["sweeps"], o["ring_lo"],
                  o["ring_hi"])
        elif o["kind"] == st.OP_EXCHANGE:
            flat = torch.from_numpy(buf[o["buf"]].reshape(-1))  # shares memory with the slab
            sends, recvs = st.st_halo_plan(rank, nranks, n, pitch, o["sweeps"])
            reqs = [dist.isend(flat[off:off + cnt].clone(), peer) for peer, off, cnt in sends]
            tmp = [(off, cnt, torch.empty(cnt, dtype=torch.float64)) for _, off, cnt in recvs]
            reqs += [dist.irecv(t, peer) for (peer, _, _), (_, _, t) in zip(recvs, tmp)]
            for q in reqs:
                q.wait()
            for off, cnt, t in tmp:
                flat[off:off + cnt] = t
    fin = buf[iters & 1]
    owned = torch.from_numpy(np.ascontiguousarray(fin[h:h + n]))
    pieces = [None] * nranks
    dist.all_gather_object(pieces, (start, owned.numpy(), fin[h - 1].copy(), fin[h + n].copy()))
    if rank != 0:
        return None
    out = np.zeros_like(a_glob)
    for r, (s0, rows, lo_row, hi_row) in enumerate(pieces):
        out[s0 + 1:s0 + 1 + rows.shape[0]] = rows
        if r == 0:
            out[0] = lo_row
        if r == nranks - 1:
            out[ny + 1] = hi_row
    return out
