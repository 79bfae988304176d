"""Throughput of the generic stencil executor on 16384^2 (5-point Listing 1 form, 9-point R=2)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))
import torch
import paper_2310_01882_b200 as st
n = 16384
for name, offs, coefs in (("5pt", [(-1, 0), (1, 0), (0, -1), (0, 1)], [0.25] * 4),
                          ("9pt_R2", [(0, 0), (-2, 0), (2, 0), (0, -2), (0, 2), (-1, -1), (1, 1), (-1, 1), (1, -1)],
                           [0.2] + [0.1] * 8)):
    R = max(max(abs(a), abs(b)) for a, b in offs)
    a = torch.rand(n + 2 * R, n + 2 * R, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    st.st_stencil2d_run(a, b, offs, coefs, 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record(); st.st_stencil2d_run(a, b, offs, coefs, it); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name}: {n * n * it / (ms / 1e3) / 1e9:.1f} Gpts/s, {16 * n * n * it / (ms / 1e3) / 1e9:.0f} GB/s (16 B/pt)")
