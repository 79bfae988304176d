"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/libstencil.h declares, and the host-only entry points (block split,
halo plan, argument validation) behave as documented."""
import ctypes
import pathlib
import re

import pytest

import paper_2310_01882_b200 as st

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "libstencil.h").read_text()


def declared_functions():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z0-9_]+)\s*\(", body)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = st.lib()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(st.EXPORTS)
    assert lib.st_abi_version() == 1


def test_library_is_sm100a_only():
    # the fatbin carries sm_100a SASS and no PTX to JIT
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", "--list-ptx", str(st.LIB_PATH)],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout
    assert ".ptx" not in out.stdout


@pytest.mark.parametrize("n,p", [(16384, 1), (32768, 8), (37, 4), (512, 3), (7, 7), (5, 8)])
def test_block_split_partitions(n, p):
    pieces = [st.st_block_split(n, p, r) for r in range(p)]
    assert pieces[0][0] == 0
    for (s0, c0), (s1, _) in zip(pieces, pieces[1:]):
        assert s0 + c0 == s1
    assert sum(c for _, c in pieces) == n
    counts = [c for _, c in pieces]
    assert max(counts) - min(counts) <= 1
    assert counts == sorted(counts)  # remainder to the high ranks


def test_halo_plan_shapes():
    # middle rank of 4, 10 owned slabs of pitch 7, width 2
    sends, recvs = st.st_halo_plan(1, 4, 10, 7, 2)
    assert sends == [(0, 2 * 7, 14), (2, 10 * 7, 14)]
    assert recvs == [(0, 0, 14), (2, 12 * 7, 14)]
    s0, r0 = st.st_halo_plan(0, 4, 10, 7, 2)
    assert [x[0] for x in s0] == [1] and [x[0] for x in r0] == [1]
    s3, r3 = st.st_halo_plan(3, 4, 10, 7, 2)
    assert [x[0] for x in s3] == [2] and r3 == [(2, 0, 14)]
    assert st.st_halo_plan(0, 1, 10, 7, 1) == ([], [])


def test_halo_plan_matches_between_neighbours():
    # what r sends to r+1 has the size r+1 expects from r
    for p in (2, 3, 8):
        for r in range(p - 1):
            s, _ = st.st_halo_plan(r, p, 9, 5, 3)
            _, rr = st.st_halo_plan(r + 1, p, 11, 5, 3)
            up = [x for x in s if x[0] == r + 1][0]
            down = [x for x in rr if x[0] == r][0]
            assert up[2] == down[2]


@pytest.mark.parametrize("args", [(4, 4, 1, 7, 1), (0, 2, 1, 7, 2), (0, 2, 5, 0, 1), (-1, 2, 5, 3, 1)])
def test_halo_plan_rejects(args):
    with pytest.raises(st.StencilError) as e:
        st.st_halo_plan(*args)
    assert e.value.code == st.ST_EINVAL


def test_jacobi_validation_is_synchronous_and_needs_no_device():
    lib = st.lib()
    rib = ctypes.c_int32()
    # null pointers
    assert lib.st_jacobi2d_run(None, None, 4, 4, 6, 1, 1, 0, None, None, ctypes.byref(rib)) == st.ST_EINVAL
    assert "null" in st.last_error()
    # odd pitch / misaligned / halo without comm: all rejected before touching CUDA
    assert lib.st_jacobi2d_run(16, 4096, 4, 4, 7, 1, 1, 0, None, None, None) == st.ST_EINVAL
    assert lib.st_jacobi2d_run(8, 4096, 4, 4, 6, 1, 1, 0, None, None, None) == st.ST_EINVAL
    assert lib.st_jacobi2d_run(16, 4096, 4, 4, 6, 2, 1, 0, None, None, None) == st.ST_EINVAL
    assert lib.st_jacobi2d_run(16, 4096, 0, 4, 6, 1, 1, 0, None, None, None) == st.ST_EINVAL
    # overlapping buffers
    assert lib.st_jacobi2d_run(16, 32, 4, 4, 6, 1, 1, 0, None, None, None) == st.ST_EINVAL
    assert "overlap" in st.last_error()


def test_pw_validation():
    lib = st.lib()
    z = [16 * (1 << 20) * (i + 1) for i in range(6)]
    tz = [16] * 4
    assert lib.st_pw_advect3d(*z, 4, 4, 4, 7, 0.1, 0.1, *tz, None, None) == st.ST_EINVAL  # odd ldx
    assert lib.st_pw_advect3d(*z[:5], z[0], 4, 4, 4, 6, 0.1, 0.1, *tz, None, None) == st.ST_EINVAL  # alias
    assert lib.st_pw_advect3d(*z, 4, 4, 4, 6, 0.1, 0.1, None, *tz[1:], None, None) == st.ST_EINVAL


def test_product_never_imports_or_links_oracle():
    pkg = ROOT / "paper_2310_01882_b200"
    for f in pkg.rglob("*"):
        if f.suffix in (".py",):
            assert not re.search(r"^\s*(import|from)\s+oracle", f.read_text(), flags=re.M), f
        if f.suffix in (".cu", ".cuh", ".h", ".cpp"):
            assert not re.search(r"#include\s*[<\"][^>\"]*oracle", f.read_text()), f
    import subprocess
    deps = subprocess.run(["ldd", str(st.LIB_PATH)], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "stinputs" not in deps
