#!/usr/bin/env python
"""Benchmark of the B200 stencil hot path (contract: README/DESIGN.md §8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {cuda,reference}]

N=1 workload = BASELINE.json configs[1]: Jacobi-2D 5-point, 16384x16384
interior fp64, 1000 sweeps per step (one st_jacobi2d_run call). The PW
advection (configs[2], 512^3) is measured in the same run and reported under
"pw_advect3d" with its own roofline. N>1 (torchrun, one rank per GPU):
configs[3], Jacobi-2D 32768^2 strong scaling over row slabs with NCCL halo
exchange, plus configs[4] PW 1024x1024x512 z-slabs.

Metric: Gpts/s = 1e9 grid-point updates per second (the paper's MCells/s /
1000), whole job over all ranks. Inputs are synthetic, from
stencil_inputs (seed 42, SURVEY.md §8(d) recipe). Every buffer is larger than
the 126 MB L2, so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gpts/s per GPU and % of B200 HBM BW; 1/2/4/8-GPU scaling eff."
UNIT = "Gpts/s"
JACOBI_BYTES_PER_PT = 16  # one 8-byte read + one 8-byte write per point per sweep
PW_BYTES_PER_PT = 48      # u,v,w read + su,sv,sw written
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
FP64_PEAK_TFLOPS = 18.5    # measured non-FMA fp64 rate (tools/exp/fp64_pipe.cu)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key: str):
    """DRAM bytes per launch from the committed ncu --set full summary, or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    v = d.get(kernel_key)
    return None if v is None else v.get("dram_bytes_per_launch")


def gs_traffic_per_sweep():
    """The GS launch runs all sweeps; tools/prof_kernels.py profiles a 4-sweep launch."""
    v = ncu_traffic("gauss_seidel2d_tiled_kernel")
    return None if v is None else v / 4


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def pitch(n: int, align: int) -> int:
    """Row pitch in doubles: n rounded up to a multiple of `align` (even)."""
    align = max(2, align + (align & 1))
    return (n + align - 1) // align * align


def host_info():
    model = ""
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return model, os.cpu_count() or 1


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The CPU oracle, as it stands, on the host cores (bench.py --impl reference)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np  # noqa: F401
    import oracle
    import stencil_inputs as si
    model, cores = host_info()
    n, sweeps = 16384, args.ref_sweeps
    a = si.jacobi2d_grid(n, n)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.jacobi2d(a, sweeps, threads=cores)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    mean = sum(times) / len(times)
    value = n * n * sweeps / mean / 1e9
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "jacobi2d_16384x16384_fp64 (configs[1]); step = bounded sample of "
                               f"{sweeps} sweeps of the full grid", "sweeps_per_step": sweeps},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{sweeps} Jacobi sweeps of the 16384^2 grid per step, C oracle "
                                   f"(-O2 -ffp-contract=off, OpenMP {cores} threads) on {model}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def cpu_baseline_jacobi(sweeps: int):
    import oracle
    import stencil_inputs as si
    model, cores = host_info()
    n = 16384
    a = si.jacobi2d_grid(n, n)
    oracle.jacobi2d(a, 1, threads=cores)  # warm (page-in)
    t0 = time.perf_counter()
    oracle.jacobi2d(a, sweeps, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": round(n * n * sweeps / dt / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{sweeps} sweeps of the configs[1] 16384^2 grid (of 1000 per step), C oracle "
                      f"-O2 -ffp-contract=off, OpenMP {cores} threads, {model}; {dt:.2f} s"}


def cpu_baseline_pw():
    import oracle
    import stencil_inputs as si
    _, cores = host_info()
    n = 512
    d = si.pw_inputs(n, n, n)
    t0 = time.perf_counter()
    oracle.pw_advect3d(d["u"], d["v"], d["w"], d, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": round(n ** 3 / dt / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 application on the configs[2] 512^3 grid; {dt:.2f} s"}


# --------------------------------------------------------------------------- CUDA arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["cuda", "reference"], default="cuda")
    ap.add_argument("--sweeps", type=int, default=1000, help="Jacobi sweeps per step (configs[1]: 1000)")
    ap.add_argument("--tblock", type=int, default=0)
    ap.add_argument("--halo", type=int, default=8, help="ghost rows per side across ranks (N>1)")
    ap.add_argument("--transport", choices=["ipc", "nccl"], default="ipc",
                    help="N>1 halo transport: ipc = fused stores / copy engines over CUDA-IPC (default), nccl")
    ap.add_argument("--same-gpu", action="store_true", help="all ranks on cuda:0 (functional check only)")
    ap.add_argument("--align", type=int, default=2, help="row pitch multiple in doubles (2 = 16-byte rows)")
    ap.add_argument("--pw-apps", type=int, default=20, help="PW applications timed")
    ap.add_argument("--no-pw", action="store_true")
    ap.add_argument("--no-j3", action="store_true")
    ap.add_argument("--j3-sweeps", type=int, default=100, help="3-D 7-point Jacobi sweeps timed (512^3)")
    ap.add_argument("--no-gs", action="store_true")
    ap.add_argument("--no-generic", action="store_true")
    ap.add_argument("--gs-sweeps", type=int, default=100, help="in-place Gauss-Seidel sweeps timed (16384^2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-pipeline", action="store_true", help="e2e: copies and compute strictly serial")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-sweeps", type=int, default=20)
    ap.add_argument("--cpu-sweeps", type=int, default=40)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import paper_2310_01882_b200 as st
    import stencil_inputs as si

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_gpu:  # functional check of the N>1 path on a 1-GPU box (numbers meaningless)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        if args.transport == "nccl":
            dist.init_process_group("nccl", device_id=dev)
            comm = st.Comm.from_process_group(local)
        else:  # IPC transport: gloo carries only the control plane (blobs, barriers, max)
            dist.init_process_group("gloo")
            # probe: map the neighbours, run one real swap on a side stream and check the
            # ghosts; every rank falls back together (the NCCL transport is the other GPU
            # path, not a CPU fallback) if any rank failed
            ok, err = 1, ""
            try:
                comm = st.Comm.ipc_from_process_group(local)
                probe = torch.full((8, 4), float(rank), dtype=torch.float64, device=dev)
                comm.bind_ipc([probe], 2)
                ps = torch.cuda.Stream()
                st.st_halo_exchange(comm, [probe], 2, 4, 1, stream=ps)
                comm.wait(ps, timeout_ms=30000)
                if rank > 0:
                    ok &= int(bool((probe[0] == rank - 1).all()))
                if rank < world - 1:
                    ok &= int(bool((probe[3] == rank + 1).all()))
            except Exception as e:
                ok, err = 0, str(e)
            flag = torch.tensor([ok], dtype=torch.int32)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                print(f"[bench] IPC transport unavailable ({err or 'a rank failed the probe swap'}); using NCCL",
                      file=sys.stderr)
                comm = st.Comm.from_process_group(local)
                args.transport = "nccl"
    assert world == args.gpus or world == 1, "--gpus must match the torchrun world size"

    def bind(buffers, n_slow):
        """Register the buffers the next phase swaps (collective for the IPC transport)."""
        if comm is not None and getattr(comm, "kind", "nccl") == "ipc":
            comm.bind_ipc(buffers, n_slow)

    stream = torch.cuda.current_stream()
    hbm_peak, peak_src = peaks()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ------------------------------------------------------------------ Jacobi
    n_glob = 16384 if world == 1 else 32768
    halo = 1 if world == 1 else args.halo  # ghost depth across ranks (>= the temporal-blocking depth)
    ny0, ny_loc = st.st_block_split(n_glob, world, rank)
    ld = pitch(n_glob + 2, args.align)
    rows = ny_loc + 2 * halo
    # rank slab: buffer row l <-> global padded row ny0 + 1 + (l - halo); rows beyond the grid stay 0
    g_lo = max(0, ny0 + 1 - halo)
    g_hi = min(n_glob + 1, ny0 + ny_loc + halo)
    a_np = np.zeros((rows, ld))
    a_np[g_lo - (ny0 + 1 - halo): g_hi - (ny0 + 1 - halo) + 1] = si.jacobi2d_grid(
        n_glob, n_glob, ld=ld, row0=g_lo, rows=g_hi - g_lo + 1)
    a_host = torch.from_numpy(a_np)
    a0 = a_host.to(dev)
    A = torch.empty_like(a0)
    B = torch.empty_like(a0)
    sweeps = args.sweeps

    A.copy_(a0)
    bind([A, B], ny_loc)

    def jacobi_step():
        # `sweeps` more sweeps of the resident grid; with an even count the state stays in A
        r = st.st_jacobi2d_run(A, B, sweeps, tblock=args.tblock, halo=halo, comm=comm)
        if r is not A:
            A.copy_(r)

    for _ in range(args.warmup):
        jacobi_step()
    barrier()
    l0 = st.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        times = []
        for _ in range(args.steps):
            barrier()
            ev0.record(stream)
            jacobi_step()
            ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
        barrier()
    launches = st.launch_count() - l0
    step_ms = max_over_ranks(sum(times) / len(times))
    launches_per_step = launches / args.steps
    ops = st.st_jacobi2d_schedule(rank, world, n_glob, ny_loc, halo, sweeps, args.tblock)
    pass_sweeps = sorted({o["sweeps"] for o in ops if o["kind"] == st.OP_SWEEP})
    # one pass = one read + one write of the rank's grid (a pass may be split into boundary and
    # interior launches across ranks); its average duration is the roofline's launch time
    passes_per_step = sum(1 for o in ops if o["kind"] == st.OP_SWAP)
    launch_ms = step_ms / passes_per_step
    pts_total = n_glob * n_glob * sweeps
    value = pts_total / (step_ms / 1e3) / 1e9
    pts_rank = ny_loc * n_glob
    # algorithmic bytes of ONE launch: every pass reads the grid once and writes it once,
    # whatever its temporal-blocking depth (16 B per point per launch)
    achieved_gbs = JACOBI_BYTES_PER_PT * pts_rank / (launch_ms / 1e3) / 1e9
    effective_gbs = JACOBI_BYTES_PER_PT * pts_rank * sweeps / (step_ms / 1e3) / 1e9
    kname = "jacobi2d_tb4_kernel" if max(pass_sweeps) > 1 else "jacobi2d_stream_kernel"
    clocks = clk.summary()

    # ------------------------------------------------------------------ e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        h_in = a_host.pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        Ae, Be = A, B

        def e2e_step():
            Ae.copy_(h_in, non_blocking=True)
            r = st.st_jacobi2d_run(Ae, Be, sweeps, tblock=args.tblock, halo=halo, comm=comm)
            h_out.copy_(r, non_blocking=True)

        e2e_step()
        barrier()
        e_times = []
        for _ in range(max(1, min(args.steps, 3))):
            barrier()
            ev0.record(stream)
            e2e_step()
            ev1.record(stream)
            ev1.synchronize()
            e_times.append(ev0.elapsed_time(ev1))
        e_ms = max_over_ranks(sum(e_times) / len(e_times))
        e2e = {"value": round(pts_total / (e_ms / 1e3) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": h_in.numel() * 8, "d2h_bytes_per_step": h_out.numel() * 8,
               "ms_per_step": round(e_ms, 3), "pipelined": False}
        if world == 1 and not args.no_e2e_pipeline:
            # Pipelined over independent steps: step i's H2D, compute and D2H each run on their
            # own stream; two device buffer sets let step i+1's H2D and step i-1's D2H overlap
            # step i's compute. Every step still copies its whole input in and its result out.
            sets = [(A, B), (torch.empty_like(A), torch.empty_like(B))]
            s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
            in_done = [torch.cuda.Event() for _ in sets]
            comp_done = [torch.cuda.Event() for _ in sets]
            freed = [torch.cuda.Event() for _ in sets]

            def pipelined(nsteps):
                for i in range(nsteps):
                    k = i % 2
                    Ak, Bk = sets[k]
                    if i >= 2:
                        s_in.wait_event(freed[k])
                    with torch.cuda.stream(s_in):
                        Ak.copy_(h_in, non_blocking=True)
                        in_done[k].record(s_in)
                    stream.wait_event(in_done[k])
                    r = st.st_jacobi2d_run(Ak, Bk, sweeps, tblock=args.tblock, halo=halo, comm=comm)
                    comp_done[k].record(stream)
                    s_out.wait_event(comp_done[k])
                    with torch.cuda.stream(s_out):
                        h_out.copy_(r, non_blocking=True)
                        freed[k].record(s_out)

            pipelined(2)
            torch.cuda.synchronize()
            kp = max(3, args.steps)
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(s_in)
            stream.wait_event(p0)
            s_out.wait_event(p0)
            pipelined(kp)
            s_out.wait_stream(stream)
            p1.record(s_out)
            p1.synchronize()
            pe_ms = p0.elapsed_time(p1) / kp
            e2e.update({"value": round(pts_total / (pe_ms / 1e3) / 1e9, 3), "ms_per_step": round(pe_ms, 3),
                        "pipelined": True, "steps_pipelined": kp, "ms_per_step_serial": round(e_ms, 3),
                        "value_serial": round(pts_total / (e_ms / 1e3) / 1e9, 3)})
            del sets
        del h_in, h_out
    del A, B, a0

    # ------------------------------------------------------------------ PW advection
    pw = None
    if not args.no_pw:
        nxy = 512 if world == 1 else 1024
        nz_glob = 512
        z0, nz_loc = st.st_block_split(nz_glob, world, rank)
        d = si.pw_inputs(nxy, nxy, nz_glob, ldx=pitch(nxy + 2, args.align), plane0=z0, planes=nz_loc + 2)
        g = {k: (torch.from_numpy(v).to(dev) if hasattr(v, "shape") else v) for k, v in d.items()}
        outs = [torch.empty_like(g["u"]) for _ in range(3)]
        bind([g["u"], g["v"], g["w"]], nz_loc)

        def pw_app():
            st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"],
                              g["tzd1"], g["tzd2"], comm=comm)

        for _ in range(args.warmup):
            pw_app()
        barrier()
        pl0 = st.launch_count()
        ev0.record(stream)
        for _ in range(args.pw_apps):
            pw_app()
        ev1.record(stream)
        ev1.synchronize()
        pw_launches = st.launch_count() - pl0
        app_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.pw_apps)
        pts = nxy * nxy * nz_glob
        pw_gbs = PW_BYTES_PER_PT * nxy * nxy * nz_loc / (app_ms / 1e3) / 1e9
        pw = {"workload": f"pw_advect3d_{nxy}x{nxy}x{nz_glob}_fp64" + ("" if world == 1 else f"_zslabs{world}"),
              "ldx": pitch(nxy + 2, args.align),
              "value": round(pts / (app_ms / 1e3) / 1e9, 3), "unit": UNIT, "ms_per_app": round(app_ms, 4),
              "apps": args.pw_apps, "gpu_launches": pw_launches,
              "roofline": {"bound": "hbm", "achieved": round(pw_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                           "frac": round(pw_gbs / hbm_peak, 4), "traffic": ncu_traffic("pw_advect3d_kernel"),
                           "bytes_per_pt": PW_BYTES_PER_PT, "peak_source": peak_src}}
        if world == 1 and not args.no_cpu:
            pw["cpu_baseline"] = cpu_baseline_pw()
        del g, outs

    # ------------------------------------------------------------------ 3-D 7-point Jacobi (NEXT #1)
    j3 = None
    if not args.no_j3:
        n3 = 512
        z0, nz3 = st.st_block_split(n3, world, rank)
        h3 = 1 if world == 1 else 2  # two ghost planes: slabs also run two sweeps per pass
        ldx3 = pitch(n3 + 2, args.align)
        # slab buffer: nz3 + 2*h3 planes, buffer plane l = global padded plane z0 + 1 + l - h3
        # (planes beyond the grid stay zero; they are never read)
        g3 = np.zeros((nz3 + 2 * h3, n3 + 2, ldx3))
        zlo, zhi = max(0, z0 + 1 - h3), min(n3 + 1, z0 + nz3 + h3)
        g3[zlo - (z0 + 1 - h3): zhi - (z0 + 1 - h3) + 1] = si.jacobi3d_grid(n3, n3, n3, ldx=ldx3, plane0=zlo,
                                                                        planes=zhi - zlo + 1)
        A3 = torch.from_numpy(g3).to(dev)
        B3 = torch.empty_like(A3)
        bind([A3, B3], nz3)
        j3_sweeps = args.j3_sweeps

        def j3_step():
            r3 = st.st_jacobi3d_run(A3, B3, j3_sweeps, halo=h3, comm=comm)
            if r3 is not A3:
                A3.copy_(r3)

        for _ in range(args.warmup):
            j3_step()
        barrier()
        jl0 = st.launch_count()
        ev0.record(stream)
        j3_step()
        ev1.record(stream)
        ev1.synchronize()
        j3_launches = st.launch_count() - jl0
        j3_ms = max_over_ranks(ev0.elapsed_time(ev1))
        # two sweeps per pass (jacobi3d_t2_kernel; slabs too, with their 2 ghost planes): a pass
        # reads and writes the grid once (16 B/pt); one launch per pass on a single domain, three
        # (boundary planes, boundary planes, interior) on a slab whose swap overlaps the interior
        t2 = j3_sweeps >= 2
        j3_kernel = "jacobi3d_t2_kernel" if t2 else "jacobi3d_kernel"
        j3_passes = (j3_sweeps + 1) // 2 if t2 else j3_sweeps
        j3_launch_ms = j3_ms / max(1, j3_passes)
        j3_gbs = JACOBI_BYTES_PER_PT * n3 * n3 * nz3 / (j3_launch_ms / 1e3) / 1e9
        j3 = {"workload": f"jacobi3d_{n3}^3_fp64_{j3_sweeps}sweeps" + ("" if world == 1 else f"_zslabs{world}"),
              "value": round(n3 ** 3 * j3_sweeps / (j3_ms / 1e3) / 1e9, 3), "unit": UNIT,
              "ms_per_step": round(j3_ms, 3), "gpu_launches": j3_launches,
              "roofline": {"bound": "hbm", "kernel": j3_kernel, "achieved": round(j3_gbs, 1),
                           "peak": hbm_peak, "unit": "GB/s", "frac": round(j3_gbs / hbm_peak, 4),
                           "traffic": ncu_traffic(j3_kernel), "bytes_per_pt_per_launch": JACOBI_BYTES_PER_PT,
                           "sweeps_per_pass": 2 if t2 else 1, "passes": j3_passes,
                           "effective_gbs_16B_per_update": round(
                               JACOBI_BYTES_PER_PT * n3 * n3 * nz3 * j3_sweeps / (j3_ms / 1e3) / 1e9, 1),
                           "peak_source": peak_src}}
        if world == 1 and not args.no_cpu:
            import oracle
            _, cores = host_info()
            t0 = time.perf_counter()
            oracle.jacobi3d(g3, 2, threads=cores)
            dt = time.perf_counter() - t0
            j3["cpu_baseline"] = {"value": round(n3 ** 3 * 2 / dt / 1e9, 4), "unit": UNIT, "cores": cores,
                                  "kind": "oracle", "sample": f"2 sweeps of the 512^3 grid; {dt:.2f} s"}
        del A3, B3

    # ------------------------------------------------------------------ in-place Gauss-Seidel (NEXT #4)
    gs = None
    if world == 1 and not args.no_gs:
        ngs = 16384
        ags = torch.from_numpy(si.jacobi2d_grid(ngs, ngs)).to(dev)
        ws = torch.empty(int(st.lib().st_gauss_seidel2d_workspace_bytes(ngs)) // 8 + 1, dtype=torch.int64, device=dev)
        st.st_gauss_seidel2d_run(ags, 1, workspace=ws)  # warm-up (module load)
        torch.cuda.synchronize()
        gl0 = st.launch_count()
        ev0.record(stream)
        st.st_gauss_seidel2d_run(ags, args.gs_sweeps, workspace=ws)
        ev1.record(stream)
        ev1.synchronize()
        gs_launches = st.launch_count() - gl0
        gs_ms = ev0.elapsed_time(ev1)
        gs_gbs = JACOBI_BYTES_PER_PT * ngs * ngs * args.gs_sweeps / (gs_ms / 1e3) / 1e9
        gs = {"workload": f"gauss_seidel2d_{ngs}x{ngs}_fp64_{args.gs_sweeps}sweeps_inplace_lexicographic",
              "value": round(ngs * ngs * args.gs_sweeps / (gs_ms / 1e3) / 1e9, 3), "unit": UNIT,
              "ms_per_step": round(gs_ms, 3), "sweeps_per_launch": args.gs_sweeps, "gpu_launches": gs_launches,
              "roofline": {"bound": "hbm", "kernel": "gauss_seidel2d_tiled_kernel", "achieved": round(gs_gbs, 1),
                           "peak": hbm_peak, "unit": "GB/s", "frac": round(gs_gbs / hbm_peak, 4),
                           "traffic": gs_traffic_per_sweep(), "traffic_unit": "DRAM bytes per sweep (ncu of a "
                           "4-sweep launch / 4)", "bytes_per_pt_per_sweep": JACOBI_BYTES_PER_PT,
                           "peak_source": peak_src}}
        if not args.no_cpu:
            import oracle
            a_small = si.jacobi2d_grid(ngs, 2048)  # a 2048-row band of the same grid recipe
            t0 = time.perf_counter()
            oracle.gauss_seidel2d(a_small, 1)
            dt = time.perf_counter() - t0
            gs["cpu_baseline"] = {"value": round(ngs * 2048 / dt / 1e9, 4), "unit": UNIT, "cores": 1,
                                  "kind": "oracle", "sample": f"1 sweep of a 16384x2048 grid (sequential by "
                                  f"definition); {dt:.2f} s"}
        del ags, ws

    # ------------------------------------------------------------------ generic stencil.apply executor (R23)
    gen = None
    if world == 1 and not args.no_generic:
        ng, gsw = 16384, 20
        offs, coefs = [(-1, 0), (1, 0), (0, -1), (0, 1)], [0.25, 0.25, 0.25, 0.25]  # Listing 1, generic form
        ag = torch.from_numpy(si.jacobi2d_grid(ng, ng)).to(dev)
        bg = torch.empty_like(ag)
        st.st_stencil2d_run(ag, bg, offs, coefs, 2)
        torch.cuda.synchronize()
        sl0 = st.launch_count()
        ev0.record(stream)
        st.st_stencil2d_run(ag, bg, offs, coefs, gsw)
        ev1.record(stream)
        ev1.synchronize()
        g_ms = ev0.elapsed_time(ev1)
        g_gbs = JACOBI_BYTES_PER_PT * ng * ng * gsw / (g_ms / 1e3) / 1e9
        gen = {"workload": f"stencil2d_generic_5pt_{ng}x{ng}_fp64_{gsw}sweeps",
               "value": round(ng * ng * gsw / (g_ms / 1e3) / 1e9, 3), "unit": UNIT, "ms_per_step": round(g_ms, 3),
               "gpu_launches": st.launch_count() - sl0,
               "roofline": {"bound": "hbm", "kernel": "stencil2d_kernel", "achieved": round(g_gbs, 1),
                            "peak": hbm_peak, "unit": "GB/s", "frac": round(g_gbs / hbm_peak, 4),
                            "traffic": ncu_traffic("stencil2d_kernel"), "bytes_per_pt": JACOBI_BYTES_PER_PT,
                            "peak_source": peak_src}}
        if not args.no_cpu:
            import oracle
            _, cores = host_info()
            a_np = si.jacobi2d_grid(ng, ng)
            t0 = time.perf_counter()
            oracle.stencil2d(a_np, offs, coefs, 1, threads=cores)
            dt = time.perf_counter() - t0
            gen["cpu_baseline"] = {"value": round(ng * ng / dt / 1e9, 4), "unit": UNIT, "cores": cores,
                                   "kind": "oracle", "sample": f"1 sweep of the 16384^2 grid; {dt:.2f} s"}
        del ag, bg

    # ------------------------------------------------------------------ C1: 64^2 + ring, 100 sweeps (latency-bound)
    c1 = None
    if world == 1:
        a1 = torch.from_numpy(si.jacobi2d_grid(64, 64)).to(dev)
        b1 = torch.empty_like(a1)
        c1 = {"workload": "jacobi2d_64x64_fp64_100sweeps (configs[0])", "unit": "us per 100 sweeps"}
        for label, tb in (("resident_single_cta", 0), ("one_launch_per_sweep", 1)):
            for _ in range(3):
                st.st_jacobi2d_run(a1, b1, 100, tblock=tb)
            torch.cuda.synchronize()
            reps = 20
            ev0.record(stream)
            for _ in range(reps):
                st.st_jacobi2d_run(a1, b1, 100, tblock=tb)
            ev1.record(stream)
            ev1.synchronize()
            c1[label] = round(ev0.elapsed_time(ev1) * 1e3 / reps, 2)
        c1["value_resident_gpts"] = round(64 * 64 * 100 / (c1["resident_single_cta"] * 1e-6) / 1e9, 3)
        del a1, b1

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_jacobi(args.cpu_sweeps)

    if comm is not None:
        comm.close()
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "ms_per_step_runs": [round(t, 3) for t in times], "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SplitMix64 seed 42, SURVEY.md §8(d) recipe)",
            "config": {"workload": f"jacobi2d_{n_glob}x{n_glob}_fp64_{sweeps}sweeps"
                                   + ("" if world == 1 else f"_rowslabs{world}"),
                       "sweeps_per_step": sweeps, "tblock": args.tblock, "ld": ld,
                       "l2": "no flush needed: each buffer is %.2f GB > 126 MB L2" % (rows * ld * 8 / 1e9),
                       "step": "st_jacobi2d_run(iters=%d) continuing from the resident state" % sweeps,
                       "transport": None if world == 1 else args.transport, "halo": halo},
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved_gbs, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(achieved_gbs / hbm_peak, 4), "traffic": ncu_traffic(kname),
                         "bytes_per_pt_per_launch": JACOBI_BYTES_PER_PT, "sweeps_per_launch": pass_sweeps,
                         "launches_per_step": launches_per_step, "passes_per_step": passes_per_step,
                         "ms_per_pass": round(launch_ms, 5),
                         "frac_of_nominal_8tbs": round(achieved_gbs / 8000.0, 4),
                         "effective_gbs_16B_per_update": round(effective_gbs, 1), "peak_source": peak_src},
            # the same kernel against the fp64 pipe (temporal blocking lifts it off the HBM roof):
            # 4 flops per update (3 DADD + 1 DMUL, never contracted), peak = the measured DADD rate
            "roofline_fp64": {"bound": "alu", "achieved": round(4 * value / world / 1e3, 3), "peak": FP64_PEAK_TFLOPS,
                              "unit": "TFLOP/s (per GPU)", "frac": round(4 * value / world / 1e3 / FP64_PEAK_TFLOPS, 4),
                              "peak_source": "tools/exp/fp64_pipe.cu: 63.6 DADD/clk/SM x 148 SMs (18.5 T/s); "
                                             "no FMA (DESIGN.md R11)"},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "pw_advect3d": pw,
            "jacobi3d": j3,
            "gauss_seidel2d": gs,
            "stencil2d_generic": gen,
            "c1": c1,
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
