"""Decomposition overhead on ONE GPU: the C2 Jacobi grid (16384^2) and the C3 PW
grid (512^3) split into P = 1, 2, 4 slab ranks of a LOCAL group (all ranks in
this process, all on cuda:0, each on its own stream, halo swaps by fused
kernel stores + device-side flags). Total work is fixed, so Gpts/s(P) /
Gpts/s(1) is the fraction of throughput the decomposition (ghost rows, swaps,
flag waits, boundary/interior launch split) leaves — not multi-GPU scaling,
which needs several GPUs. Device-timed: one event on the default stream before
all ranks, one after all ranks joined."""
import json
import os
import pathlib
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))

import numpy as np
import torch

import paper_2310_01882_b200 as st
import stencil_inputs as si


def timed(ranks_fn, streams, reps):
    main = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ranks_fn()  # warm-up
    torch.cuda.synchronize()
    ev0.record(main)
    for s in streams:
        s.wait_event(ev0)
    for _ in range(reps):
        ranks_fn()
    for s in streams:
        main.wait_stream(s)
    ev1.record(main)
    ev1.synchronize()
    return ev0.elapsed_time(ev1) / reps


def jacobi(P, n=16384, sweeps=200, h=8):
    comms = st.Comm.local_group(P) if P > 1 else [None]
    streams = [torch.cuda.Stream() for _ in range(P)]
    bufs = []
    for r in range(P):
        start, cnt = st.st_block_split(n, P, r)
        hh = h if P > 1 else 1
        lo = max(0, start + 1 - hh)
        hi = min(n + 1, start + cnt + hh)
        a_np = np.zeros((cnt + 2 * hh, n + 2))
        a_np[lo - (start + 1 - hh): hi - (start + 1 - hh) + 1] = si.jacobi2d_grid(n, n, row0=lo, rows=hi - lo + 1)
        a = torch.from_numpy(a_np).cuda()
        b = torch.empty_like(a)
        if comms[r] is not None:
            comms[r].bind([a, b], cnt)
        bufs.append((a, b, hh))
    torch.cuda.synchronize()

    def run():
        for r in range(P):
            a, b, hh = bufs[r]
            with torch.cuda.stream(streams[r]):
                st.st_jacobi2d_run(a, b, sweeps, tblock=0, halo=hh, comm=comms[r])

    ms = timed(run, streams, 2)
    for c in comms:
        if c is not None:
            c.close()
    return n * n * sweeps / (ms / 1e3) / 1e9, ms


def pw(P, n=512, apps=20):
    comms = st.Comm.local_group(P) if P > 1 else [None]
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = []
    for r in range(P):
        z0, cnt = st.st_block_split(n, P, r)
        d = si.pw_inputs(n, n, n, plane0=z0, planes=cnt + 2)
        g = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
        outs = [torch.empty_like(g["u"]) for _ in range(3)]
        if comms[r] is not None:
            comms[r].bind([g["u"], g["v"], g["w"]], cnt)
        parts.append((g, outs))
    torch.cuda.synchronize()

    def run():
        for r in range(P):
            g, outs = parts[r]
            with torch.cuda.stream(streams[r]):
                st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"],
                                  g["tzd1"], g["tzd2"], comm=comms[r])

    ms = timed(run, streams, apps)
    for c in comms:
        if c is not None:
            c.close()
    return n ** 3 / (ms / 1e3) / 1e9, ms


_G3 = {}


def jacobi3d(P, n=512, sweeps=100, h=2):
    # z slabs; h = 2 ghost planes run two sweeps per pass across ranks (T = 2), h = 1 one
    if n not in _G3:
        _G3[n] = torch.from_numpy(si.jacobi3d_grid(n, n, n)).cuda()  # generated once, sliced per rank
    g = _G3[n]
    comms = st.Comm.local_group(P) if P > 1 else [None]
    streams = [torch.cuda.Stream() for _ in range(P)]
    bufs = []
    for r in range(P):
        z0, cnt = st.st_block_split(n, P, r)
        hh = h if P > 1 else 1
        a = torch.zeros((cnt + 2 * hh, n + 2, n + 2), dtype=torch.float64, device="cuda")
        lo = max(0, z0 + 1 - hh)
        hi = min(n + 1, z0 + cnt + hh)
        a[lo - (z0 + 1 - hh): hi - (z0 + 1 - hh) + 1] = g[lo:hi + 1]
        b = torch.empty_like(a)
        if comms[r] is not None:
            comms[r].bind([a, b], cnt)
        bufs.append((a, b, hh))
    torch.cuda.synchronize()

    def run():
        for r in range(P):
            a, b, hh = bufs[r]
            with torch.cuda.stream(streams[r]):
                st.st_jacobi3d_run(a, b, sweeps, halo=hh, comm=comms[r])

    ms = timed(run, streams, 2)
    for c in comms:
        if c is not None:
            c.close()
    return n ** 3 * sweeps / (ms / 1e3) / 1e9, ms


def pencils_j3(py, pz, n=512, sweeps=50, tblock=1):
    """3-D Jacobi on a py x pz (y, z) pencil grid of LOCAL ranks (swap overlapped with the interior block;
    tblock 2: two sweeps per pass on ghost depth 2). py = pz = 1: the single domain at the same tblock
    (same sweep kernel, no decomposition)."""
    if n not in _G3:
        _G3[n] = torch.from_numpy(si.jacobi3d_grid(n, n, n)).cuda()
    g = _G3[n]
    P = py * pz
    h = 2 if tblock == 2 and P > 1 else 1
    gp = torch.nn.functional.pad(g, (0, 0, h - 1, h - 1, h - 1, h - 1)) if h > 1 else g
    comms = st.Comm.local_group(P) if P > 1 else [None]
    streams = [torch.cuda.Stream() for _ in range(P)]
    bufs = []
    for r in range(P):
        y0, nyl, z0, nzl = st.st_pencil_split(n, n, py, pz, r) if P > 1 else (0, n, 0, n)
        a = gp[z0:z0 + nzl + 2 * h, y0:y0 + nyl + 2 * h].contiguous()
        b = torch.empty_like(a)
        if comms[r] is not None:
            comms[r].set_grid(py, nyl)
            comms[r].bind([a, b], nzl)
        bufs.append((a, b))
    torch.cuda.synchronize()

    def run():
        for r in range(P):
            a, b = bufs[r]
            with torch.cuda.stream(streams[r]):
                if comms[r] is None:
                    st.st_jacobi3d_run(a, b, sweeps, tblock=tblock)
                else:
                    st.st_jacobi3d_run_pencils(a, b, sweeps, comm=comms[r], nx=n, halo=h, tblock=tblock)

    ms = timed(run, streams, 2)
    for c in comms:
        if c is not None:
            c.close()
    return n ** 3 * sweeps / (ms / 1e3) / 1e9, ms


def pencils_pw(py, pz, n=512, apps=20):
    d = si.pw_inputs(n, n, n)
    P = py * pz
    comms = st.Comm.local_group(P) if P > 1 else [None]
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = []
    for r in range(P):
        y0, nyl, z0, nzl = st.st_pencil_split(n, n, py, pz, r) if P > 1 else (0, n, 0, n)
        g = {k: torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2, y0:y0 + nyl + 2])).cuda() for k in "uvw"}
        for k in ("tzc1", "tzc2", "tzd1", "tzd2"):
            g[k] = torch.from_numpy(np.ascontiguousarray(d[k][z0:z0 + nzl + 2])).cuda()
        outs = [torch.empty_like(g["u"]) for _ in range(3)]
        if comms[r] is not None:
            comms[r].set_grid(py, nyl)
            comms[r].bind([g["u"], g["v"], g["w"]], nzl)
        parts.append((g, outs))
    del d
    torch.cuda.synchronize()

    def run():
        for r in range(P):
            g, outs = parts[r]
            with torch.cuda.stream(streams[r]):
                if comms[r] is None:
                    st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, 0.25 / 3, 0.05, g["tzc1"], g["tzc2"],
                                      g["tzd1"], g["tzd2"])
                else:
                    st.st_pw_advect3d_pencils(g["u"], g["v"], g["w"], *outs, 0.25 / 3, 0.05, g["tzc1"],
                                              g["tzc2"], g["tzd1"], g["tzd2"], comm=comms[r])

    ms = timed(run, streams, apps)
    for c in comms:
        if c is not None:
            c.close()
    return n ** 3 / (ms / 1e3) / 1e9, ms


if __name__ == "__main__":
    if sys.argv[1:] == ["pencils"]:  # the (y, z) pencil decomposition (NEXT #2) on one GPU
        out = {"what": "LOCAL pencil grids (py x pz) on one B200: throughput at fixed total work vs the single "
                       "domain with the same sweep kernel (T = 1; t2: two sweeps per pass, ghost depth 2)",
               "jacobi3d_512^3_50sw": {}, "jacobi3d_t2_512^3_50sw": {}, "pw_512^3": {}}
        for py, pz in ((1, 1), (2, 1), (1, 2), (2, 2), (4, 2)):
            v, ms = pencils_j3(py, pz)
            out["jacobi3d_512^3_50sw"][f"{py}x{pz}"] = {"gpts": round(v, 1), "ms": round(ms, 2)}
            print(f"pencils j3 {py}x{pz}: {v:.1f} Gpts/s", file=sys.stderr, flush=True)
            v, ms = pencils_j3(py, pz, tblock=2)
            out["jacobi3d_t2_512^3_50sw"][f"{py}x{pz}"] = {"gpts": round(v, 1), "ms": round(ms, 2)}
            print(f"pencils j3 t2 {py}x{pz}: {v:.1f} Gpts/s", file=sys.stderr, flush=True)
            v, ms = pencils_pw(py, pz)
            out["pw_512^3"][f"{py}x{pz}"] = {"gpts": round(v, 2), "ms_per_app": round(ms, 4)}
            print(f"pencils pw {py}x{pz}: {v:.2f} Gpts/s", file=sys.stderr, flush=True)
        for k in ("jacobi3d_512^3_50sw", "jacobi3d_t2_512^3_50sw", "pw_512^3"):
            base = out[k]["1x1"]["gpts"]
            for g in out[k]:
                out[k][g]["vs_1x1"] = round(out[k][g]["gpts"] / base, 3)
        print(json.dumps(out))
        sys.exit(0)
    only3d = sys.argv[1:] == ["3d"]  # just the 3-D Jacobi legs
    out = {"what": "LOCAL rank group on one B200: throughput at fixed total work vs P=1", "jacobi2d_16384^2_200sw": {},
           "pw_512^3": {}, "jacobi3d_512^3_100sw_h2": {}, "jacobi3d_512^3_100sw_h1": {}}
    for P in (1, 2, 4):
        for h in (2, 1):
            v, ms = jacobi3d(P, h=h)
            out[f"jacobi3d_512^3_100sw_h{h}"][P] = {"gpts": round(v, 1), "ms": round(ms, 2)}
            print(f"jacobi3d P={P} h={h}: {v:.1f} Gpts/s", file=sys.stderr, flush=True)
        if only3d:
            continue
        v, ms = jacobi(P)
        out["jacobi2d_16384^2_200sw"][P] = {"gpts": round(v, 1), "ms": round(ms, 2)}
        v, ms = pw(P)
        out["pw_512^3"][P] = {"gpts": round(v, 2), "ms_per_app": round(ms, 4)}
    for k in ("jacobi2d_16384^2_200sw", "pw_512^3", "jacobi3d_512^3_100sw_h2", "jacobi3d_512^3_100sw_h1"):
        if not out[k]:
            del out[k]
            continue
        base = out[k][1]["gpts"]
        for P in out[k]:
            out[k][P]["vs_P1"] = round(out[k][P]["gpts"] / base, 3)
    print(json.dumps(out))
