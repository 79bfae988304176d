"""Subprocess driver for the multi-sweep Gauss-Seidel wavefront: the sweep depth
K (ST_GS_MS_K) is read once per process, so each K runs in its own process.
usage: python tests/gs_ms_cases.py K  -> exit 0 when every case is bitwise equal
to the sequential oracle (Listing 1 literally, R22)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2310_01882_b200 as st  # noqa: E402
import stencil_inputs as si  # noqa: E402

# (nx, ny, ld, iters): >= 382 columns (24 tiles of 16) takes the multi-sweep schedule;
# one strip (ny <= 32), a 4-row last strip, partial CTAs, odd pitch, every remainder
CASES = [
    (382, 1, 384, 5), (390, 32, 392, 6), (390, 33, 392, 7), (400, 60, 402, 9),
    (410, 257, 412, 7), (433, 130, 435, 9), (1000, 300, 1002, 13), (395, 1000, 398, 5),
    (480, 95, 482, 1), (480, 95, 482, 2), (480, 95, 482, 3), (480, 95, 482, 4), (480, 95, 482, 8),
    (481, 95, 484, 11),
]


def main(k: int) -> int:
    bad = 0
    for nx, ny, ld, iters in CASES:
        a_np = si.jacobi2d_grid(nx, ny, ld=ld)
        want = oracle.gauss_seidel2d(a_np, iters, nx=nx)
        a = torch.from_numpy(a_np).cuda()
        st.st_gauss_seidel2d_run(a, iters, nx=nx)
        torch.cuda.synchronize()
        got = a.cpu().numpy()
        ok = np.array_equal(got, want)
        if not ok:
            diff = np.argwhere(got != want)
            print(f"K={k} {nx}x{ny} ld={ld} iters={iters}: {len(diff)} mismatches, first {diff[:5].tolist()}")
            bad += 1
    print(f"K={k}: {len(CASES) - bad}/{len(CASES)} cases bitwise")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1])))
