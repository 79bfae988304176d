"""Throughput of NVRTC-compiled expression stencils on 16384^2 (and first-call compile time)."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))
import torch
import paper_2310_01882_b200 as st
n = 16384
for e in ("(a(-1,0)+a(1,0)+a(0,-1)+a(0,1))*0.25", "(a(0,0) + a(2,0))*(a(0,0) - a(-2,0)) / (1 + a(0,2)*a(0,2))"):
    R = st.st_stencil2d_expr_halo(e)
    a = torch.rand(n + 2 * R, n + 2 * R, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    t0 = time.perf_counter(); st.st_stencil2d_expr_run(a, b, e, 2); torch.cuda.synchronize(); tc = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record(); st.st_stencil2d_expr_run(a, b, e, it); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{e}: first call (compile) {tc:.2f} s; {n * n * it / (ms / 1e3) / 1e9:.1f} Gpts/s, "
          f"{16 * n * n * it / (ms / 1e3) / 1e9:.0f} GB/s (16 B/pt)")
m = 512
e = "(a(-1,0,0)+a(1,0,0)+a(0,-1,0)+a(0,1,0)+a(0,0,-1)+a(0,0,1))/6"
a = torch.rand(m + 2, m + 2, m + 2, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
st.st_stencil3d_expr_run(a, b, e, 2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); st.st_stencil3d_expr_run(a, b, e, 20); e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1)
print(f"3-D benchmark 1 expression 512^3: {m ** 3 * 20 / (ms / 1e3) / 1e9:.1f} Gpts/s, "
      f"{16 * m ** 3 * 20 / (ms / 1e3) / 1e9:.0f} GB/s (16 B/pt)")
import stencil_inputs as si
m = 512
d = si.pw_inputs(m, m, m)
g = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in d.items()}
outs = [torch.empty_like(g["u"]) for _ in range(3)]
ex = st.pw_fused_expressions(d["tcx"], d["tcy"])
args = ([g["u"], g["v"], g["w"]], outs, ex, [g["tzc1"], g["tzc2"], g["tzd1"], g["tzd2"]])
st.st_stencil3d_fused_run(*args)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    st.st_stencil3d_fused_run(*args)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"PW as a fused expression region 512^3: {m ** 3 / (ms / 1e3) / 1e9:.1f} Gpts/s, "
      f"{48 * m ** 3 / (ms / 1e3) / 1e9:.0f} GB/s (48 B/pt)")
