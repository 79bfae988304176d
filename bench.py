#!/usr/bin/env python
"""Benchmark of the B200 stencil hot path (contract: DESIGN.md §7).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {cuda,reference}]

N = 1 (headline): BASELINE.json configs[1], Jacobi-2D 5-point, 16384^2 interior
fp64, 1000 sweeps per step (one st_jacobi2d_run call). In the same run, each
with its own roofline: the single-sweep kernel on the same grid (`jacobi2d_t1`),
the strong-scaling workloads on ONE GPU (`c4`: configs[3] Jacobi 32768^2, 1000
sweeps; `c5`: configs[4] PW 1024x1024x512), configs[2] PW 512^3
(`pw_advect3d`), and the NEXT rows (3-D Jacobi, Gauss-Seidel, generic stencil,
configs[0]).

N > 1 (torchrun, one rank per GPU): strong scaling of configs[3] (C4, row
slabs, 10 ghost rows, T = 10 across ranks) and configs[4] (C5, z-slabs). Halo
transport: fused neighbour stores + device flags over CUDA-IPC mappings
(NVLink peer memory), or NCCL send/recv (--transport nccl, and the loud
fallback if the IPC probe fails). Rank 0 also times the same C4/C5 step on
its GPU alone, so every N > 1 line carries its own efficiency T1 / (N * TN).
A profiled extra step reports per-rank phase times (boundary rows, interior,
blocked join wait) that show whether the swap is hidden behind the interior.

Metric: Gpts/s = 1e9 grid-point updates per second (the paper's MCells/s /
1000). `value` is the whole-job aggregate over all ranks (the
harness contract); `per_gpu` = value / N. Inputs are synthetic, from
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
JACOBI_BYTES_PER_PT = 16  # one 8-byte read + one 8-byte write per point per pass
PW_BYTES_PER_PT = 48      # u,v,w read + su,sv,sw written
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
FP64_PEAK_TFLOPS = 18.5    # measured non-FMA fp64 rate (tools/exp/fp64_pipe.cu)
C2_N, C4_N = 16384, 32768
C5_NXY, C5_NZ = 1024, 512


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
    v = json.loads(p.read_text()).get(kernel_key)
    return None if v is None else v.get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks, power and throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
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
        sm, pw, mx, reasons = [], [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                pw.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


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
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import oracle
    import stencil_inputs as si
    model, cores = host_info()
    n, sweeps = C2_N, args.ref_sweeps
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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "jacobi2d_16384x16384_fp64 (configs[1]); step = bounded sample of "
                               f"{sweeps} sweeps of the full grid", "sweeps_per_step": sweeps},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{sweeps} Jacobi sweeps of the 16384^2 grid per step, C oracle "
                                   f"(-O2 -ffp-contract=off, OpenMP {cores} threads) on {model}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def cpu_baselines(sweeps_all: int, sweeps_one: int):
    """The oracle on all host cores and on one core, C2 grid."""
    import oracle
    import stencil_inputs as si
    model, cores = host_info()
    a = si.jacobi2d_grid(C2_N, C2_N)
    oracle.jacobi2d(a, 1, threads=cores)  # warm (page-in)
    out = {}
    for label, thr, sw in (("all", cores, sweeps_all), ("one", 1, sweeps_one)):
        t0 = time.perf_counter()
        oracle.jacobi2d(a, sw, threads=thr)
        dt = time.perf_counter() - t0
        out[label] = (C2_N * C2_N * sw / dt / 1e9, dt, sw, thr)
    v, dt, sw, thr = out["all"]
    v1, dt1, sw1, _ = out["one"]
    return {"value": round(v, 4), "unit": UNIT, "cores": thr, "kind": "oracle",
            "sample": f"{sw} sweeps of the configs[1] 16384^2 grid (of 1000 per step), C oracle -O2 "
                      f"-ffp-contract=off, OpenMP {thr} threads, {model}; {dt:.2f} s",
            "one_core": {"value": round(v1, 4), "unit": UNIT, "cores": 1,
                         "sample": f"{sw1} sweeps of the same grid on 1 thread; {dt1:.2f} s"}}


def cpu_baseline_pw():
    import oracle
    import stencil_inputs as si
    _, cores = host_info()
    n = 512
    d = si.pw_inputs(n, n, n)
    t0 = time.perf_counter()
    oracle.pw_advect3d(d["u"], d["v"], d["w"], d, threads=cores)
    dt = time.perf_counter() - t0
    planes = 32  # one core: a 32-plane band of the same fields
    db = si.pw_inputs(n, n, planes)
    t1 = time.perf_counter()
    oracle.pw_advect3d(db["u"], db["v"], db["w"], db, threads=1)
    dt1 = time.perf_counter() - t1
    return {"value": round(n ** 3 / dt / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 application on the configs[2] 512^3 grid; {dt:.2f} s",
            "one_core": {"value": round(n * n * planes / dt1 / 1e9, 4), "unit": UNIT, "cores": 1,
                         "sample": f"1 application on a 512x512x{planes} band; {dt1:.2f} s"}}


# --------------------------------------------------------------------------- CUDA arm
class Ctx:
    """Process-group plumbing shared by the legs."""

    def __init__(self, args):
        import torch
        import paper_2310_01882_b200 as st
        self.torch, self.st, self.args = torch, st, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = 0 if args.same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.dist = None
        self.comm = None
        self.transport = None
        self.probe = None
        if self.world > 1:
            import torch.distributed as dist
            self.dist = dist
            if args.transport == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
                self.comm = st.Comm.from_process_group(self.local)
                self.transport = "nccl"
            else:
                self._init_ipc()
        self.stream = torch.cuda.current_stream()
        self.hbm_peak, self.peak_src = peaks()

    def _init_ipc(self):
        # IPC transport: gloo carries only the control plane (blobs, barriers, max). Probe:
        # map the neighbours, run one real swap on a side stream and check the ghosts; every
        # rank falls back together (to the NCCL transport, the other GPU path) if any failed
        torch, st, dist = self.torch, self.st, self.dist
        dist.init_process_group("gloo")
        ok, err = 1, ""
        try:
            self.comm = st.Comm.ipc_from_process_group(self.local)
            probe = torch.full((8, 4), float(self.rank), dtype=torch.float64, device=self.dev)
            self.comm.bind_ipc([probe], 2)
            ps = torch.cuda.Stream()
            st.st_halo_exchange(self.comm, [probe], 2, 4, 1, stream=ps)
            self.comm.wait(ps, timeout_ms=30000)
            if self.rank > 0:
                ok &= int(bool((probe[0] == self.rank - 1).all()))
            if self.rank < self.world - 1:
                ok &= int(bool((probe[3] == self.rank + 1).all()))
            if not ok:
                err = "ghost rows wrong after the probe swap"
        except Exception as e:  # noqa: BLE001 - any failure means: fall back loudly
            ok, err = 0, str(e)
        flag = torch.tensor([ok], dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            msg = err or "another rank failed the probe swap"
            print(f"[bench] rank {self.rank}: IPC transport UNAVAILABLE ({msg}); FALLING BACK to NCCL send/recv",
                  file=sys.stderr, flush=True)
            self.probe = "failed: " + msg
            self.comm = st.Comm.from_process_group(self.local)
            self.transport = "nccl (fallback)"
        else:
            self.probe = "ok"
            fused = os.environ.get("ST_FUSED_HALO", "1") != "0"
            self.transport = "ipc-fused" if fused else "ipc-copy-engine"

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, obj):
        if self.dist is None:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def bind(self, buffers, n_slow):
        """Register the buffers the next phase swaps (collective for the IPC transport)."""
        if self.comm is not None and getattr(self.comm, "kind", "nccl") == "ipc":
            self.comm.bind_ipc(buffers, n_slow)

    def events(self):
        t = self.torch
        return t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)

    def time_steps(self, step, steps, warmup):
        """W untimed steps, then K steps each bracketed by a barrier and CUDA events on the
        launching stream; returns the per-step times (ms) of this rank."""
        for _ in range(warmup):
            step()
        self.barrier()
        ev0, ev1 = self.events()
        times = []
        for _ in range(steps):
            self.barrier()
            ev0.record(self.stream)
            step()
            ev1.record(self.stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
        self.barrier()
        return times


def jacobi_slab(ctx, n, world, rank, halo, align, with_host=False):
    """A rank's row slab of the n x n Jacobi grid (global values; rows beyond the grid 0)."""
    import numpy as np
    import stencil_inputs as si
    torch, st = ctx.torch, ctx.st
    ny0, ny_loc = st.st_block_split(n, world, rank)
    ld = pitch(n + 2, align)
    rows = ny_loc + 2 * halo
    # buffer row l <-> global padded row ny0 + 1 + (l - halo)
    g_lo = max(0, ny0 + 1 - halo)
    g_hi = min(n + 1, ny0 + ny_loc + halo)
    a_np = np.zeros((rows, ld))
    a_np[g_lo - (ny0 + 1 - halo): g_hi - (ny0 + 1 - halo) + 1] = si.jacobi2d_grid(
        n, n, ld=ld, row0=g_lo, rows=g_hi - g_lo + 1)
    a_host = torch.from_numpy(a_np)
    a = a_host.to(ctx.dev)
    return (a, torch.empty_like(a), ld, ny_loc, (a_host if with_host else None))


def jacobi_roofline(ctx, kname, ops, step_ms, pts_rank, sweeps, extra=None):
    """Dominant-kernel roofline: 16 algorithmic bytes per point per pass (a pass reads and
    writes the rank's grid once, whatever its temporal-blocking depth) / average pass time."""
    st = ctx.st
    pass_sweeps = sorted({o["sweeps"] for o in ops if o["kind"] == st.OP_SWEEP})
    passes = sum(1 for o in ops if o["kind"] == st.OP_SWAP)
    pass_ms = step_ms / passes
    gbs = JACOBI_BYTES_PER_PT * pts_rank / (pass_ms / 1e3) / 1e9
    r = {"bound": "hbm", "kernel": kname, "achieved": round(gbs, 1), "peak": ctx.hbm_peak, "unit": "GB/s",
         "frac": round(gbs / ctx.hbm_peak, 4), "traffic": ncu_traffic(kname),
         "bytes_per_pt_per_launch": JACOBI_BYTES_PER_PT, "sweeps_per_launch": pass_sweeps,
         "passes_per_step": passes, "ms_per_pass": round(pass_ms, 5),
         "frac_of_nominal_8tbs": round(gbs / 8000.0, 4),
         "effective_gbs_16B_per_update": round(JACOBI_BYTES_PER_PT * pts_rank * sweeps / (step_ms / 1e3) / 1e9, 1),
         "peak_source": ctx.peak_src}
    if extra:
        r.update(extra)
    return r


def jacobi_leg(ctx, n, world, rank, comm, sweeps, steps, warmup, tblock=0, halo=1):
    """`steps` timed steps of `sweeps` sweeps of the n x n grid on this rank's slab."""
    st, torch = ctx.st, ctx.torch
    A, B, ld, ny_loc, _ = jacobi_slab(ctx, n, world, rank, halo, ctx.args.align)
    if comm is not None:
        ctx.bind([A, B], ny_loc)

    def step():
        r = st.st_jacobi2d_run(A, B, sweeps, tblock=tblock, halo=halo, comm=comm)
        if r is not A:
            A.copy_(r)

    l0 = st.launch_count()
    times = ctx.time_steps(step, steps, warmup)
    launches = (st.launch_count() - l0) // (steps + warmup) * steps
    ops = st.st_jacobi2d_schedule(rank, world, n, ny_loc, halo, sweeps, tblock)
    del A, B
    torch.cuda.empty_cache()
    return times, launches, ops, ny_loc


def pw_leg(ctx, world, rank, comm, nxy, nz, apps, warmup):
    """`apps` timed PW applications on this rank's z-slab of an nxy x nxy x nz grid."""
    import stencil_inputs as si
    st, torch = ctx.st, ctx.torch
    z0, nz_loc = st.st_block_split(nz, world, rank)
    ldx = pitch(nxy + 2, ctx.args.align)
    d = si.pw_inputs(nxy, nxy, nz, ldx=ldx, plane0=z0, planes=nz_loc + 2)
    g = {k: (torch.from_numpy(v).to(ctx.dev) if hasattr(v, "shape") else v) for k, v in d.items()}
    del d
    outs = [torch.empty_like(g["u"]) for _ in range(3)]
    if comm is not None:
        ctx.bind([g["u"], g["v"], g["w"]], nz_loc)

    def app():
        st.st_pw_advect3d(g["u"], g["v"], g["w"], *outs, g["tcx"], g["tcy"], g["tzc1"], g["tzc2"], g["tzd1"],
                          g["tzd2"], comm=comm)

    def step():
        for _ in range(apps):
            app()

    l0 = st.launch_count()
    times = ctx.time_steps(step, 1, warmup)
    launches = st.launch_count() - l0
    prof = None
    if comm is not None and world > 1:
        ctx.barrier()
        comm.profile(True)
        app()
        ctx.barrier()
        comm.profile(False)
        prof = comm.profile_read()
    del g, outs
    torch.cuda.empty_cache()
    return times[0] / apps, launches, nz_loc, prof


def pw_roofline(ctx, pts_rank, app_ms):
    gbs = PW_BYTES_PER_PT * pts_rank / (app_ms / 1e3) / 1e9
    return {"bound": "hbm", "kernel": "pw_advect3d_kernel", "achieved": round(gbs, 1), "peak": ctx.hbm_peak,
            "unit": "GB/s", "frac": round(gbs / ctx.hbm_peak, 4), "traffic": ncu_traffic("pw_advect3d_kernel"),
            "bytes_per_pt": PW_BYTES_PER_PT, "peak_source": ctx.peak_src}


def phase_summary(per_rank):
    """Per-rank phase times (ms) of one profiled step, and the fraction of the step the
    ranks' streams sat blocked waiting for ghosts (0 = the swap is fully hidden)."""
    rows = []
    for r, p in enumerate(per_rank):
        if p is None:
            continue
        rows.append({"rank": r, **{k: round(v[0], 4) for k, v in p.items()}})
    if not rows:
        return None
    keys = ("boundary", "interior", "join_wait", "ready_wait")
    blocked = max((x["join_wait"] + x["ready_wait"]) / max(1e-9, sum(x[k] for k in keys)) for x in rows)
    return {"unit": "ms per profiled step", "ranks": rows, "max_blocked_frac": round(blocked, 4)}


# --------------------------------------------------------------------------- N = 1
def run_single(ctx):
    import numpy as np
    import stencil_inputs as si
    args, st, torch = ctx.args, ctx.st, ctx.torch
    out = {}
    sweeps = args.sweeps

    # ---------------------------------------------------------------- headline: C2
    A, B, ld, ny_loc, a_host = jacobi_slab(ctx, C2_N, 1, 0, 1, args.align, with_host=True)

    def step():
        r = st.st_jacobi2d_run(A, B, sweeps, tblock=args.tblock)
        if r is not A:
            A.copy_(r)

    for _ in range(args.warmup):
        step()
    ctx.barrier()
    l0 = st.launch_count()
    with ClockSampler(ctx.local) as clk:
        times = ctx.time_steps(step, args.steps, 0)
    launches = st.launch_count() - l0
    step_ms = sum(times) / len(times)
    ops = st.st_jacobi2d_schedule(0, 1, C2_N, C2_N, 1, sweeps, args.tblock)
    kname = "jacobi2d_tb4_kernel" if any(o["sweeps"] > 1 for o in ops if o["kind"] == st.OP_SWEEP) \
        else "jacobi2d_stream_kernel"
    value = C2_N * C2_N * sweeps / (step_ms / 1e3) / 1e9
    out.update({
        "value": round(value, 3), "ms_per_step": round(step_ms, 3), "ms_per_step_runs": [round(t, 3) for t in times],
        "config": {"workload": f"jacobi2d_{C2_N}x{C2_N}_fp64_{sweeps}sweeps (configs[1])", "sweeps_per_step": sweeps,
                   "tblock": args.tblock, "ld": ld,
                   "l2": "no flush needed: each buffer is %.2f GB > 126 MB L2" % (A.numel() * 8 / 1e9),
                   "step": "st_jacobi2d_run(iters=%d) continuing from the resident state" % sweeps},
        "roofline": jacobi_roofline(ctx, kname, ops, step_ms, C2_N * C2_N, sweeps),
        "roofline_fp64": {"bound": "alu", "achieved": round(4 * value / 1e3, 3), "peak": FP64_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "frac": round(4 * value / 1e3 / FP64_PEAK_TFLOPS, 4),
                          "peak_source": "tools/exp/fp64_pipe.cu: 63.6 DADD/clk/SM x 148 SMs (18.5 T/s); "
                                         "no FMA (DESIGN.md R11)"},
        "gpu_launches": launches, "clocks": clk.summary()})

    # ---------------------------------------------------------------- e2e (host buffers)
    if not args.no_e2e:
        out["e2e"] = e2e_single(ctx, A, B, a_host, sweeps)
    del A, B, a_host
    torch.cuda.empty_cache()

    # ---------------------------------------------------------------- T = 1 sweep kernel
    t1_sweeps = max(20, args.t1_sweeps)
    t1_times, t1_l, t1_ops, _ = jacobi_leg(ctx, C2_N, 1, 0, None, t1_sweeps, 3, 2, tblock=1)
    t1_ms = sum(t1_times) / len(t1_times)
    out["jacobi2d_t1"] = {
        "workload": f"jacobi2d_{C2_N}x{C2_N}_fp64_{t1_sweeps}sweeps_tblock1 (configs[1] grid, one sweep per pass)",
        "value": round(C2_N * C2_N * t1_sweeps / (t1_ms / 1e3) / 1e9, 3), "unit": UNIT,
        "ms_per_step": round(t1_ms, 3), "gpu_launches": t1_l,
        "roofline": jacobi_roofline(ctx, "jacobi2d_stream_kernel", t1_ops, t1_ms, C2_N * C2_N, t1_sweeps)}

    # ---------------------------------------------------------------- C4 / C5 on one GPU (scaling base)
    if not args.no_scaling:
        c4_times, c4_l, c4_ops, _ = jacobi_leg(ctx, C4_N, 1, 0, None, sweeps, args.scale_steps, 2)
        c4_ms = sum(c4_times) / len(c4_times)
        out["c4"] = {"workload": f"jacobi2d_{C4_N}x{C4_N}_fp64_{sweeps}sweeps (configs[3]) on 1 GPU",
                     "value": round(C4_N * C4_N * sweeps / (c4_ms / 1e3) / 1e9, 3), "unit": UNIT,
                     "per_gpu": round(C4_N * C4_N * sweeps / (c4_ms / 1e3) / 1e9, 3),
                     "ms_per_step": round(c4_ms, 3), "steps": args.scale_steps, "gpu_launches": c4_l,
                     "roofline": jacobi_roofline(ctx, "jacobi2d_tb4_kernel", c4_ops, c4_ms, C4_N * C4_N, sweeps)}
        c5_ms, c5_l, _, _ = pw_leg(ctx, 1, 0, None, C5_NXY, C5_NZ, args.pw_apps, 2)
        c5_pts = C5_NXY * C5_NXY * C5_NZ
        out["c5"] = {"workload": f"pw_advect3d_{C5_NXY}x{C5_NXY}x{C5_NZ}_fp64 (configs[4]) on 1 GPU",
                     "value": round(c5_pts / (c5_ms / 1e3) / 1e9, 3), "unit": UNIT,
                     "per_gpu": round(c5_pts / (c5_ms / 1e3) / 1e9, 3), "ms_per_app": round(c5_ms, 4),
                     "apps": args.pw_apps, "gpu_launches": c5_l, "roofline": pw_roofline(ctx, c5_pts, c5_ms)}

    # ---------------------------------------------------------------- PW advection, configs[2]
    if not args.no_pw:
        n = 512
        app_ms, pw_l, _, _ = pw_leg(ctx, 1, 0, None, n, n, args.pw_apps, args.warmup)
        out["pw_advect3d"] = {"workload": f"pw_advect3d_{n}x{n}x{n}_fp64 (configs[2])", "ldx": pitch(n + 2, args.align),
                              "value": round(n ** 3 / (app_ms / 1e3) / 1e9, 3), "unit": UNIT,
                              "ms_per_app": round(app_ms, 4), "apps": args.pw_apps, "gpu_launches": pw_l,
                              "roofline": pw_roofline(ctx, n ** 3, app_ms)}
        if not args.no_cpu:
            out["pw_advect3d"]["cpu_baseline"] = cpu_baseline_pw()

    if not args.no_j3:
        out["jacobi3d"] = jacobi3d_leg(ctx)
    if not args.no_gs:
        out["gauss_seidel2d"] = gs_leg(ctx)
    if not args.no_generic:
        out["stencil2d_generic"] = generic_leg(ctx)
    out["c1"] = c1_leg(ctx)
    if not args.no_cpu:
        out["cpu_baseline"] = cpu_baselines(args.cpu_sweeps, 2)
    return out


def e2e_single(ctx, A, B, a_host, sweeps):
    """The same call through the C-ABI with the grid copied from pinned host memory and the
    result copied back every step (pipelined over independent steps, and strictly serial)."""
    torch, st = ctx.torch, ctx.st
    args = ctx.args
    h_in = a_host.pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    stream = ctx.stream
    pts = C2_N * C2_N * sweeps

    def serial_step():
        A.copy_(h_in, non_blocking=True)
        r = st.st_jacobi2d_run(A, B, sweeps, tblock=args.tblock)
        h_out.copy_(r, non_blocking=True)

    e_times = ctx.time_steps(serial_step, max(1, min(args.steps, 3)), 1)
    e_ms = sum(e_times) / len(e_times)
    # Pipelined: step i's H2D, compute and D2H each on their own stream; two device buffer sets
    # let step i+1's upload and step i-1's download overlap step i's sweeps. Every step still
    # copies its whole input in and its result out.
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
            r = st.st_jacobi2d_run(Ak, Bk, sweeps, tblock=args.tblock)
            comp_done[k].record(stream)
            s_out.wait_event(comp_done[k])
            with torch.cuda.stream(s_out):
                h_out.copy_(r, non_blocking=True)
                freed[k].record(s_out)

    pipelined(2)
    torch.cuda.synchronize()
    kp = max(3, args.steps)
    p0, p1 = ctx.events()
    p0.record(s_in)
    stream.wait_event(p0)
    s_out.wait_event(p0)
    pipelined(kp)
    s_out.wait_stream(stream)
    p1.record(s_out)
    p1.synchronize()
    pe_ms = p0.elapsed_time(p1) / kp
    del sets
    return {"value": round(pts / (pe_ms / 1e3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h_in.numel() * 8,
            "d2h_bytes_per_step": h_out.numel() * 8, "ms_per_step": round(pe_ms, 3), "pipelined": True,
            "steps_pipelined": kp, "ms_per_step_serial": round(e_ms, 3),
            "value_serial": round(pts / (e_ms / 1e3) / 1e9, 3)}


def jacobi3d_leg(ctx):
    """NEXT #1: the paper's benchmark 1 as a 3-D 7-point Jacobi, 512^3 (z-slabs at N > 1)."""
    import numpy as np
    import stencil_inputs as si
    args, st, torch = ctx.args, ctx.st, ctx.torch
    world, rank, comm = ctx.world, ctx.rank, ctx.comm
    n3 = 512
    z0, nz3 = st.st_block_split(n3, world, rank)
    h3 = 1 if world == 1 else 2  # two ghost planes: slabs also run two sweeps per pass
    ldx3 = pitch(n3 + 2, args.align)
    g3 = np.zeros((nz3 + 2 * h3, n3 + 2, ldx3))
    zlo, zhi = max(0, z0 + 1 - h3), min(n3 + 1, z0 + nz3 + h3)
    g3[zlo - (z0 + 1 - h3): zhi - (z0 + 1 - h3) + 1] = si.jacobi3d_grid(n3, n3, n3, ldx=ldx3, plane0=zlo,
                                                                    planes=zhi - zlo + 1)
    A3 = torch.from_numpy(g3).to(ctx.dev)
    B3 = torch.empty_like(A3)
    if comm is not None:
        ctx.bind([A3, B3], nz3)
    sw = args.j3_sweeps

    def step():
        r3 = st.st_jacobi3d_run(A3, B3, sw, halo=h3, comm=comm)
        if r3 is not A3:
            A3.copy_(r3)

    l0 = st.launch_count()
    times = ctx.time_steps(step, 1, args.warmup)
    launches = (st.launch_count() - l0) // (1 + args.warmup)
    j3_ms = ctx.max_over_ranks(times[0])
    t2 = sw >= 2
    kname = "jacobi3d_t2_kernel" if t2 else "jacobi3d_kernel"
    passes = (sw + 1) // 2 if t2 else sw
    gbs = JACOBI_BYTES_PER_PT * n3 * n3 * nz3 / (j3_ms / max(1, passes) / 1e3) / 1e9
    res = {"workload": f"jacobi3d_{n3}^3_fp64_{sw}sweeps" + ("" if world == 1 else f"_zslabs{world}"),
           "value": round(n3 ** 3 * sw / (j3_ms / 1e3) / 1e9, 3), "unit": UNIT, "ms_per_step": round(j3_ms, 3),
           "gpu_launches": launches,
           "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(gbs, 1), "peak": ctx.hbm_peak,
                        "unit": "GB/s", "frac": round(gbs / ctx.hbm_peak, 4), "traffic": ncu_traffic(kname),
                        "bytes_per_pt_per_launch": JACOBI_BYTES_PER_PT, "sweeps_per_pass": 2 if t2 else 1,
                        "passes": passes, "effective_gbs_16B_per_update": round(
                            JACOBI_BYTES_PER_PT * n3 * n3 * nz3 * sw / (j3_ms / 1e3) / 1e9, 1),
                        "peak_source": ctx.peak_src}}
    if world == 1 and not args.no_cpu:
        import oracle
        _, cores = host_info()
        t0 = time.perf_counter()
        oracle.jacobi3d(g3, 2, threads=cores)
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": round(n3 ** 3 * 2 / dt / 1e9, 4), "unit": UNIT, "cores": cores,
                               "kind": "oracle", "sample": f"2 sweeps of the 512^3 grid; {dt:.2f} s"}
    del A3, B3
    torch.cuda.empty_cache()
    return res


def gs_leg(ctx):
    """NEXT #4: Listing 1 literally (in-place lexicographic Gauss-Seidel), 16384^2."""
    import stencil_inputs as si
    args, st, torch = ctx.args, ctx.st, ctx.torch
    ngs = C2_N
    ags = torch.from_numpy(si.jacobi2d_grid(ngs, ngs)).to(ctx.dev)
    ws = torch.empty(int(st.lib().st_gauss_seidel2d_workspace_bytes(ngs, ngs)) // 8 + 1, dtype=torch.int64,
                     device=ctx.dev)
    st.st_gauss_seidel2d_run(ags, 1, workspace=ws)  # warm-up (module load)
    l0 = st.launch_count()
    times = ctx.time_steps(lambda: st.st_gauss_seidel2d_run(ags, args.gs_sweeps, workspace=ws), 1, 0)
    gs_ms = times[0]
    # multi-sweep wavefront: K sweeps per pass over the grid (ST_GS_MS_K, default 4); one pass
    # reads and writes the grid once, so the algorithmic HBM bytes are 16 B x points per pass
    k = int(os.environ.get("ST_GS_MS_K", "4"))
    passes = -(-args.gs_sweeps // k)
    gbs = JACOBI_BYTES_PER_PT * ngs * ngs * passes / (gs_ms / 1e3) / 1e9
    t = ncu_traffic("gauss_seidel2d_ms_kernel")
    res = {"workload": f"gauss_seidel2d_{ngs}x{ngs}_fp64_{args.gs_sweeps}sweeps_inplace_lexicographic",
           "value": round(ngs * ngs * args.gs_sweeps / (gs_ms / 1e3) / 1e9, 3), "unit": UNIT,
           "ms_per_step": round(gs_ms, 3), "sweeps_per_launch": args.gs_sweeps, "sweeps_per_pass": k,
           "gpu_launches": st.launch_count() - l0,
           "roofline": {"bound": "hbm", "kernel": "gauss_seidel2d_ms_kernel", "achieved": round(gbs, 1),
                        "peak": ctx.hbm_peak, "unit": "GB/s", "frac": round(gbs / ctx.hbm_peak, 4),
                        "traffic": t, "traffic_unit": "DRAM bytes per pass (ncu of a one-pass launch)",
                        "bytes_per_pt_per_pass": JACOBI_BYTES_PER_PT, "passes": passes,
                        "effective_gbs_16B_per_update": round(gbs * args.gs_sweeps / passes, 1),
                        "peak_source": ctx.peak_src}}
    if not args.no_cpu:
        import oracle
        a_small = si.jacobi2d_grid(ngs, 2048)  # a 2048-row band of the same grid recipe
        t0 = time.perf_counter()
        oracle.gauss_seidel2d(a_small, 1)
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": round(ngs * 2048 / dt / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"1 sweep of a 16384x2048 grid (sequential by definition); {dt:.2f} s"}
    del ags, ws
    return res


def generic_leg(ctx):
    """NEXT #4: the generic linear stencil.apply executor on Listing 1 written generically."""
    import stencil_inputs as si
    args, st, torch = ctx.args, ctx.st, ctx.torch
    ng, gsw = C2_N, 20
    offs, coefs = [(-1, 0), (1, 0), (0, -1), (0, 1)], [0.25, 0.25, 0.25, 0.25]
    ag = torch.from_numpy(si.jacobi2d_grid(ng, ng)).to(ctx.dev)
    bg = torch.empty_like(ag)
    st.st_stencil2d_run(ag, bg, offs, coefs, 2)
    l0 = st.launch_count()
    times = ctx.time_steps(lambda: st.st_stencil2d_run(ag, bg, offs, coefs, gsw), 1, 0)
    g_ms = times[0]
    gbs = JACOBI_BYTES_PER_PT * ng * ng * gsw / (g_ms / 1e3) / 1e9
    res = {"workload": f"stencil2d_generic_5pt_{ng}x{ng}_fp64_{gsw}sweeps",
           "value": round(ng * ng * gsw / (g_ms / 1e3) / 1e9, 3), "unit": UNIT, "ms_per_step": round(g_ms, 3),
           "gpu_launches": st.launch_count() - l0,
           # st_stencil2d_run specialises 16-byte-row grids through NVRTC (st_expr_kernel)
           "roofline": {"bound": "hbm", "kernel": "st_expr_kernel", "achieved": round(gbs, 1),
                        "peak": ctx.hbm_peak, "unit": "GB/s", "frac": round(gbs / ctx.hbm_peak, 4),
                        "traffic": ncu_traffic("st_expr_kernel"), "bytes_per_pt": JACOBI_BYTES_PER_PT,
                        "peak_source": ctx.peak_src}}
    if not args.no_cpu:
        import oracle
        _, cores = host_info()
        a_np = si.jacobi2d_grid(ng, ng)
        t0 = time.perf_counter()
        oracle.stencil2d(a_np, offs, coefs, 1, threads=cores)
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": round(ng * ng / dt / 1e9, 4), "unit": UNIT, "cores": cores,
                               "kind": "oracle", "sample": f"1 sweep of the 16384^2 grid; {dt:.2f} s"}
    del ag, bg
    return res


def c1_leg(ctx):
    """configs[0]: 64^2 + ring, 100 sweeps (latency-bound)."""
    import stencil_inputs as si
    st, torch = ctx.st, ctx.torch
    a1 = torch.from_numpy(si.jacobi2d_grid(64, 64)).to(ctx.dev)
    b1 = torch.empty_like(a1)
    res = {"workload": "jacobi2d_64x64_fp64_100sweeps (configs[0])", "unit": "us per 100 sweeps"}
    ev0, ev1 = ctx.events()
    for label, tb in (("resident_single_cta", 0), ("one_launch_per_sweep", 1)):
        for _ in range(3):
            st.st_jacobi2d_run(a1, b1, 100, tblock=tb)
        torch.cuda.synchronize()
        reps = 20
        ev0.record(ctx.stream)
        for _ in range(reps):
            st.st_jacobi2d_run(a1, b1, 100, tblock=tb)
        ev1.record(ctx.stream)
        ev1.synchronize()
        res[label] = round(ev0.elapsed_time(ev1) * 1e3 / reps, 2)
    # the same 100 one-sweep launches captured once in a CUDA graph and replayed (the C-ABI
    # call does no host synchronisation or allocation, so it is capturable as it stands)
    try:
        cap = torch.cuda.Stream()
        cap.wait_stream(ctx.stream)
        with torch.cuda.stream(cap):
            st.st_jacobi2d_run(a1, b1, 100, tblock=1)  # warm the launch path outside capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            st.st_jacobi2d_run(a1, b1, 100, tblock=1)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        reps = 20
        ev0.record(torch.cuda.current_stream())
        for _ in range(reps):
            graph.replay()
        ev1.record(torch.cuda.current_stream())
        ev1.synchronize()
        res["cuda_graph_100_launches"] = round(ev0.elapsed_time(ev1) * 1e3 / reps, 2)
    except Exception as exc:  # reported, never silently dropped
        res["cuda_graph_100_launches"] = f"failed: {type(exc).__name__}: {exc}"[:200]
    res["value_resident_gpts"] = round(64 * 64 * 100 / (res["resident_single_cta"] * 1e-6) / 1e9, 3)
    return res


# --------------------------------------------------------------------------- N > 1
def run_multi(ctx):
    """Strong scaling of C4 (Jacobi 32768^2, row slabs) and C5 (PW 1024^2 x 512, z-slabs)."""
    args, st, torch = ctx.args, ctx.st, ctx.torch
    world, rank, comm = ctx.world, ctx.rank, ctx.comm
    sweeps, halo = args.sweeps, args.halo
    out = {}

    # ---- the same C4 / C5 steps on rank 0's GPU alone (the N = 1 point of this curve)
    t1 = {}
    if rank == 0 and not args.no_scaling:
        c4_1, _, _, _ = jacobi_leg(ctx_local(ctx), C4_N, 1, 0, None, sweeps, args.scale_steps, 2)
        t1["c4"] = sum(c4_1) / len(c4_1)
        t1["c5"], _, _, _ = pw_leg(ctx_local(ctx), 1, 0, None, C5_NXY, C5_NZ, args.pw_apps, 2)
    ctx.barrier()
    t1 = ctx.gather(t1)[0]

    # ---- C4 across ranks
    A, B, ld, ny_loc, a_host = jacobi_slab(ctx, C4_N, world, rank, halo, args.align, with_host=True)
    ctx.bind([A, B], ny_loc)

    def step():
        r = st.st_jacobi2d_run(A, B, sweeps, tblock=args.tblock, halo=halo, comm=comm)
        if r is not A:
            A.copy_(r)

    for _ in range(args.warmup):
        step()
    ctx.barrier()
    l0 = st.launch_count()
    with ClockSampler(ctx.local) as clk:
        times = ctx.time_steps(step, args.steps, 0)
    launches = st.launch_count() - l0
    step_ms = ctx.max_over_ranks(sum(times) / len(times))
    ops = st.st_jacobi2d_schedule(rank, world, C4_N, ny_loc, halo, sweeps, args.tblock)
    agg = C4_N * C4_N * sweeps / (step_ms / 1e3) / 1e9
    # one profiled step (100 sweeps): per-rank phase times
    comm.profile(True)
    prof_sweeps = min(sweeps, 96)
    r = st.st_jacobi2d_run(A, B, prof_sweeps, tblock=args.tblock, halo=halo, comm=comm)
    if r is not A:
        A.copy_(r)
    ctx.barrier()
    comm.profile(False)
    phases = phase_summary(ctx.gather(comm.profile_read()))
    if phases:
        phases["sweeps"] = prof_sweeps
    out.update({
        "value": round(agg, 3), "ms_per_step": round(step_ms, 3), "ms_per_step_runs": [round(t, 3) for t in times],
        "aggregate": round(agg, 3), "per_gpu": round(agg / world, 3),
        "t1_ms_per_step": None if "c4" not in t1 else round(t1["c4"], 3),
        "efficiency": None if "c4" not in t1 else round(t1["c4"] / (world * step_ms), 4),
        "config": {"workload": f"jacobi2d_{C4_N}x{C4_N}_fp64_{sweeps}sweeps_rowslabs{world} (configs[3])",
                   "sweeps_per_step": sweeps, "tblock": args.tblock, "ld": ld, "halo": halo,
                   "transport": ctx.transport, "ipc_probe": ctx.probe,
                   "l2": "no flush needed: each rank buffer is %.2f GB > 126 MB L2" % (A.numel() * 8 / 1e9),
                   "step": "st_jacobi2d_run(iters=%d) on every rank's row slab" % sweeps},
        "roofline": jacobi_roofline(ctx, "jacobi2d_tb4_kernel", ops, step_ms, ny_loc * C4_N, sweeps,
                                    {"note": "per rank (its slab), pass time incl. boundary/interior split"}),
        "phases": phases, "gpu_launches": launches, "clocks": clk.summary()})

    # ---- e2e: the rank's slab from pinned host memory and back, every step (serial)
    if not args.no_e2e:
        h_in = a_host.pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()

        def e2e_step():
            A.copy_(h_in, non_blocking=True)
            rr = st.st_jacobi2d_run(A, B, sweeps, tblock=args.tblock, halo=halo, comm=comm)
            h_out.copy_(rr, non_blocking=True)

        e_times = ctx.time_steps(e2e_step, max(1, min(args.steps, 3)), 1)
        e_ms = ctx.max_over_ranks(sum(e_times) / len(e_times))
        nbytes = sum(ctx.gather(h_in.numel() * 8))  # all ranks' slabs, in and out
        out["e2e"] = {"value": round(C4_N * C4_N * sweeps / (e_ms / 1e3) / 1e9, 3), "unit": UNIT,
                      "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                      "ms_per_step": round(e_ms, 3), "pipelined": False}
        del h_in, h_out
    del A, B, a_host
    torch.cuda.empty_cache()

    # ---- C5 across ranks
    if not args.no_pw:
        c5_ms, c5_l, nz_loc, prof = pw_leg(ctx, world, rank, comm, C5_NXY, C5_NZ, args.pw_apps, args.warmup)
        c5_ms = ctx.max_over_ranks(c5_ms)
        pts = C5_NXY * C5_NXY * C5_NZ
        c5_agg = pts / (c5_ms / 1e3) / 1e9
        out["c5"] = {"workload": f"pw_advect3d_{C5_NXY}x{C5_NXY}x{C5_NZ}_fp64_zslabs{world} (configs[4])",
                     "value": round(c5_agg, 3), "aggregate": round(c5_agg, 3), "per_gpu": round(c5_agg / world, 3),
                     "unit": UNIT, "ms_per_app": round(c5_ms, 4), "apps": args.pw_apps, "gpu_launches": c5_l,
                     "t1_ms_per_app": None if "c5" not in t1 else round(t1["c5"], 4),
                     "efficiency": None if "c5" not in t1 else round(t1["c5"] / (world * c5_ms), 4),
                     "roofline": pw_roofline(ctx, C5_NXY * C5_NXY * nz_loc, c5_ms),
                     "phases": phase_summary(ctx.gather(prof))}
    if not args.no_j3:
        out["jacobi3d"] = jacobi3d_leg(ctx)
    return out


def ctx_local(ctx):
    """A view of ctx for single-GPU legs inside a multi-rank job (no barriers with other ranks)."""
    class _Solo:
        pass
    s = _Solo()
    s.__dict__.update(ctx.__dict__)
    s.dist = None
    s.barrier = lambda: ctx.torch.cuda.synchronize()
    s.max_over_ranks = lambda x: x
    s.gather = lambda obj: [obj]
    s.bind = lambda buffers, n_slow: None
    s.events = ctx.events
    s.time_steps = lambda step, steps, warmup: Ctx.time_steps(s, step, steps, warmup)
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["cuda", "reference"], default="cuda")
    ap.add_argument("--sweeps", type=int, default=1000, help="Jacobi sweeps per step (configs[1], [3]: 1000)")
    ap.add_argument("--tblock", type=int, default=0)
    ap.add_argument("--halo", type=int, default=10, help="ghost rows per side across ranks (N>1; = the auto T)")
    ap.add_argument("--transport", choices=["ipc", "nccl"], default="ipc",
                    help="N>1 halo transport: ipc = fused neighbour stores over CUDA-IPC (default), nccl")
    ap.add_argument("--same-gpu", action="store_true", help="all ranks on cuda:0 (functional check only)")
    ap.add_argument("--align", type=int, default=2, help="row pitch multiple in doubles (2 = 16-byte rows)")
    ap.add_argument("--pw-apps", type=int, default=20, help="PW applications per timed step")
    ap.add_argument("--scale-steps", type=int, default=3, help="timed steps of the 1-GPU C4 scaling base")
    ap.add_argument("--t1-sweeps", type=int, default=20, help="sweeps of the tblock=1 leg (>= 20)")
    ap.add_argument("--no-scaling", action="store_true", help="skip the 1-GPU C4/C5 legs")
    ap.add_argument("--no-pw", action="store_true")
    ap.add_argument("--no-j3", action="store_true")
    ap.add_argument("--j3-sweeps", type=int, default=100, help="3-D 7-point Jacobi sweeps timed (512^3)")
    ap.add_argument("--no-gs", action="store_true")
    ap.add_argument("--no-generic", action="store_true")
    ap.add_argument("--gs-sweeps", type=int, default=1000,
                    help="in-place Gauss-Seidel sweeps timed (16384^2; 1000 = the configs[1] iteration count)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-sweeps", type=int, default=20)
    ap.add_argument("--cpu-sweeps", type=int, default=40)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    ctx = Ctx(args)
    assert ctx.world == args.gpus or ctx.world == 1, "--gpus must match the torchrun world size"
    res = run_single(ctx) if ctx.world == 1 else run_multi(ctx)
    if ctx.comm is not None:
        ctx.comm.close()
    if ctx.rank == 0:
        out = {"metric": METRIC, "value": res.pop("value"), "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": res.pop("ms_per_step"), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (SplitMix64 seed 42, SURVEY.md §8(d) recipe)"}
        out.update(res)
        print(json.dumps(out), flush=True)
    if ctx.dist is not None:
        ctx.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
